#!/bin/bash
# e2e breakdown + ncu --set full of K1 on C3/C4 slices; reports summarised on the box
mkdir -p gpurun_out/prof
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
for w in c3 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -c 1 -f -o /tmp/k1_$w python tools/prof_run.py $w > gpurun_out/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/k1_$w.ncu-rep "K1 $w slice" > gpurun_out/prof/k1_$w.txt 2>&1
  ncu -i /tmp/k1_$w.ncu-rep --page raw --csv > gpurun_out/prof/k1_${w}_raw.csv 2>&1
  ls -la /tmp/k1_$w.ncu-rep >> gpurun_out/ncu_$w.log
done
echo done
