#!/bin/bash
mkdir -p gpurun_out/prof
for w in c3 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -c 1 -f -o /tmp/k1_$w python tools/prof_run.py $w > gpurun_out/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/k1_$w.ncu-rep "K1 stream $w slice" > gpurun_out/prof/k1s_$w.txt 2>&1
  ncu -i /tmp/k1_$w.ncu-rep --page raw --csv > gpurun_out/prof/k1s_${w}_raw.csv 2>&1
  ncu -i /tmp/k1_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/k1s_${w}_sass.csv 2>&1
done
echo done
