#!/bin/bash
mkdir -p gpurun_out
HALP_LIB=alt_libs/k3prof.so PROF_T=20000 timeout 300 python tools/prof_run.py c2 > gpurun_out/k3prof_c2.log 2>&1
HALP_LIB=alt_libs/k3prof.so timeout 300 python tools/prof_run.py c1 > gpurun_out/k3prof_c1.log 2>&1
echo done
