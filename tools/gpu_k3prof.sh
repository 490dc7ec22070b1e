#!/bin/bash
mkdir -p gpurun_out
HALP_LIB=alt_libs/k3prof.so PROF_T=20000 timeout 300 python tools/prof_run.py c2 > gpurun_out/k3prof_c2.log 2>&1
PROF_T=60000 timeout 300 python tools/prof_run.py c2 > gpurun_out/k3_c2.log 2>&1
timeout 900 python tools/fg_sweep.py c1 "" HALP_FG_WARPROWS=1 > gpurun_out/fg_c1.log 2>&1
echo done
