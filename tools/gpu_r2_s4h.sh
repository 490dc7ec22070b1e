#!/bin/bash
# K5 with the RNG producer warp: parity tests (bounded: a barrier bug would hang) + the C5 bench
mkdir -p gpurun_out/s4h
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_grid.py "tests/test_gpu_baseline_configs.py::test_c5_problems" tests/test_gpu_determinism.py tests/test_gpu_harness.py -x -q --durations=5 > gpurun_out/s4h/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s4h/tests.log
timeout 300 python - > gpurun_out/s4h/k5bench.log 2>&1 <<'PY'
import sys, json; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
ms, nd, st = bench.c5_batch(H, 0, 0, reps=3); print("C5 ms_per_batch", ms, "diverged", nd)
print(json.dumps(bench.grid_bench(H, 0)))
PY
echo "bench rc=$?" >> gpurun_out/s4h/k5bench.log
