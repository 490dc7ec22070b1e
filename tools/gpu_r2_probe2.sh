#!/bin/bash
mkdir -p gpurun_out/probe2
python -m paper_1803_03383_b200.build > gpurun_out/probe2/build.log 2>&1
timeout 600 python tools/e2e_overlap_probe.py > gpurun_out/probe2/probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_lm.py tests/test_gpu_batch.py -x -q > gpurun_out/probe2/tests.log 2>&1; echo "rc=$?" >> gpurun_out/probe2/tests.log
echo done
