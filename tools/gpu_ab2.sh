#!/bin/bash
mkdir -p gpurun_out/prof
for v in cur $1; do
  if [ $v = cur ]; then L=""; else L="HALP_LIB=alt_libs/$v.so"; fi
  env $L PROF_T=8000 timeout 600 ncu --set full --clock-control none -k regex:k3_ -c 1 -f -o /tmp/k3_$v python tools/prof_run.py c2 > gpurun_out/ncu_k3_$v.log 2>&1
  python tools/ncu_summary.py /tmp/k3_$v.ncu-rep "K3 $v" > gpurun_out/prof/k3_$v.txt 2>&1
  ncu -i /tmp/k3_$v.ncu-rep --page raw --csv > gpurun_out/prof/k3_${v}_raw.csv 2>&1
done
echo done
