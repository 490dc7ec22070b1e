#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_halp.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/fg_sweep.py c4 "" FG_WRAND=1 FG_WRAND=1,HALP_FG_F2F=1 > gpurun_out/fg_c4.log 2>&1
timeout 900 python tools/fg_sweep.py c3 FG_WRAND=1 > gpurun_out/fg_c3.log 2>&1
echo done
