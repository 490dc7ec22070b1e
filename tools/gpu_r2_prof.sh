#!/bin/bash
# round 2: K3 phase split (K3_PROF build) for C2 / C3 / C1 + host facts
mkdir -p gpurun_out
nproc > gpurun_out/r2_host.txt; free -g >> gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt
HALP_LIB=alt_libs/k3prof.so PROF_T=20000 timeout 300 python tools/prof_run.py c2 > gpurun_out/r2_k3prof_c2.log 2>&1
HALP_LIB=alt_libs/k3prof.so timeout 300 python tools/prof_run.py c1 > gpurun_out/r2_k3prof_c1.log 2>&1
HALP_LIB=alt_libs/k3prof.so timeout 300 python tools/sweep_inner.py c3 20000 0:0 > gpurun_out/r2_k3prof_c3.log 2>&1
echo done
