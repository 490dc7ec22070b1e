#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/fg_sweep.py c4 "" HALP_FG_WS=0 HALP_FG_STAGES=6 HALP_FG_ROWS=2 > gpurun_out/fg_c4.log 2>&1
echo done
