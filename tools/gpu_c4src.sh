#!/bin/bash
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_stream -c 1 -f -o /tmp/c4s python tools/prof_run.py c4 > gpurun_out/ncu_c4s.log 2>&1
ncu -i /tmp/c4s.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof/c4_cuda_src.csv 2>&1
ncu -i /tmp/c4s.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/c4_sass_src.csv 2>&1
echo done
