#!/bin/bash
# round 2: K5 v2 + NCCL + datagen + batch/grid parity, then the batch bench line
mkdir -p gpurun_out
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_grid.py tests/test_gpu_nccl.py tests/test_gpu_datagen.py tests/test_gpu_baseline_configs.py -x -q --durations=10 > gpurun_out/r2_k5tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_k5tests.log
timeout 300 python - > gpurun_out/r2_k5bench.log 2>&1 <<'PY'
import sys, json; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
ms, nd, st = bench.c5_batch(H, 0, 0, reps=3); print("C5 ms_per_batch", ms, "diverged", nd)
print(json.dumps(bench.grid_bench(H, 0)))
PY
