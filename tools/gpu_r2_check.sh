#!/bin/bash
# round 2: full GPU suite + short bench (+ timings)
mkdir -p gpurun_out
rm -f gpurun_out/parity_counts.jsonl
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?" >> gpurun_out/r2_bench.err
