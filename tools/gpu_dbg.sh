#!/bin/bash
mkdir -p gpurun_out
HALP_DEBUG_LAUNCH=1 PROF_T=8000 timeout 300 python tools/prof_run.py c2 > gpurun_out/dbg.log 2>&1
HALP_DEBUG_LAUNCH=1 PROF_T=8000 CUDA_MODULE_LOADING=EAGER timeout 300 python tools/prof_run.py c2 >> gpurun_out/dbg.log 2>&1
echo done
