#!/bin/bash
# session 5: K1 C4 conversion-split / split-count retune on the DW+RL kernel, and an ncu capture of it
mkdir -p gpurun_out/s5c
for v in base new of1 ef3; do
  echo "== $v" >> gpurun_out/s5c/sweep.log
  if [ $v = new ]; then unset HALP_LIB; else export HALP_LIB=alt_libs/$v.so; fi
  FG_WRAND=1 timeout 600 python tools/fg_sweep.py c4 >> gpurun_out/s5c/sweep.log 2>&1
done
unset HALP_LIB
echo "== new, split counts" >> gpurun_out/s5c/sweep.log
FG_WRAND=1 timeout 900 python tools/fg_sweep.py c4 HALP_FG_MAX_SPLITS=8192 HALP_FG_MAX_SPLITS=2048 >> gpurun_out/s5c/sweep.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k1_stream -c 1 -o /tmp/k1_c4 -f python tools/prof_run.py c4 > gpurun_out/s5c/k1_c4_ncu.log 2>&1
$NCU -i /tmp/k1_c4.ncu-rep --page details > gpurun_out/s5c/k1_c4_details.txt 2>&1
$NCU -i /tmp/k1_c4.ncu-rep --page raw --csv > gpurun_out/s5c/k1_c4_raw.csv 2>&1
$NCU -i /tmp/k1_c4.ncu-rep --page source --csv > gpurun_out/s5c/k1_c4_source.csv 2>&1
python tools/ncu_summary.py /tmp/k1_c4.ncu-rep "K1 on a c4-shaped slice (tools/prof_run.py c4), DW+RL kernel" > gpurun_out/s5c/k1_c4_summary.txt 2>&1
echo done
