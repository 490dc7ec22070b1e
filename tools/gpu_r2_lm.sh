#!/bin/bash
mkdir -p gpurun_out
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lm.py tests/test_gpu_batch.py tests/test_gpu_grid.py tests/test_gpu_harness.py -x -q --durations=10 > gpurun_out/r2_lm.log 2>&1
echo "rc=$?" >> gpurun_out/r2_lm.log
for w in 1 4; do
HALP_K5_WARPS=$w timeout 300 python - >> gpurun_out/r2_k5bench.log 2>&1 <<'PY'
import sys, json, os; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
ms, nd, st = bench.c5_batch(H, 0, 0, reps=3); print("warps", os.environ["HALP_K5_WARPS"], "C5 ms_per_batch", ms, "diverged", nd)
g = bench.grid_bench(H, 0); print("grid device_ms", g["device_ms"], "wall", g["wall_ms"])
PY
done
echo done
