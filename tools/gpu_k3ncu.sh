#!/bin/bash
mkdir -p gpurun_out/prof
PROF_T=20000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -f -o /tmp/k3 python tools/prof_run.py c2 > gpurun_out/ncu_k3.log 2>&1
python tools/ncu_summary.py /tmp/k3.ncu-rep "K3 k3_inner on C2 (60000x784x10, 16-CTA cluster, M=4, T=20000), round 1 final" > gpurun_out/prof/k3_c2.txt 2>&1
ncu -i /tmp/k3.ncu-rep --page raw --csv > gpurun_out/prof/k3_c2_raw.csv 2>&1
echo done
