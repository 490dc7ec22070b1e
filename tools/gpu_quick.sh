#!/bin/bash
# quick check: gpu tests, e2e breakdown, default bench (no CPU baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
echo done
