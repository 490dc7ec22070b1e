#!/bin/bash
mkdir -p gpurun_out/prof

timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -c 1 -f -o /tmp/k1w_c4 python tools/prof_run.py c4 > gpurun_out/ncu_c4r.log 2>&1
python tools/ncu_summary.py /tmp/k1w_c4.ncu-rep "K1 ws c4 slice" > gpurun_out/prof/k1w_c4.txt 2>&1
ncu -i /tmp/k1w_c4.ncu-rep --page raw --csv > gpurun_out/prof/k1w_c4_raw.csv 2>&1
ncu -i /tmp/k1w_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/k1w_c4_sass.csv 2>&1
echo done
