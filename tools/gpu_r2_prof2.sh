#!/bin/bash
# round 2: exchange micro, K5 + K3(C3) ncu captures
mkdir -p gpurun_out
timeout 120 tools/micro/k3x > gpurun_out/r2_k3x.log 2>&1
python tools/prof_run.py c3k3 > gpurun_out/r2_c3k3.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k5_batch -c 1 -o gpurun_out/r2_k5 -f python tools/prof_run.py c5 > gpurun_out/r2_k5_ncu.log 2>&1
PROF_T=20000 timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k3_inner -c 1 -o gpurun_out/r2_k3c3 -f python tools/prof_run.py c3k3 > gpurun_out/r2_k3c3_ncu.log 2>&1
echo done
