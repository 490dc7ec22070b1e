#!/bin/bash
mkdir -p gpurun_out/s4c
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k3x2 tools/micro/k3_exchange2.cu && timeout 300 /tmp/k3x2 > gpurun_out/s4c/k3x2.txt 2>&1
timeout 600 python tools/sweep_inner.py c3 20000 16:4,16:8,8:8,4:8 HALP_IN_LEVELS=1 >> gpurun_out/s4c/sweep.log 2>&1
echo done
