#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_halp.py tests/test_gpu_svrg.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/fg_sweep.py c4 "" HALP_FG_HALF=0 HALP_FG_ROWS=4 > gpurun_out/fg_c4.log 2>&1
echo done
