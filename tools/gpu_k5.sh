#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_grid.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-fullgrad --no-e2e --no-cpu --steps 2 > gpurun_out/bench_k5.log 2>&1
echo done
