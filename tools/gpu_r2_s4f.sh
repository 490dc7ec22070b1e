#!/bin/bash
mkdir -p gpurun_out/s4f
for v in base pf0 pf1 pf2; do
  for w in c3 c2 c1; do
    echo "== $v $w" >> gpurun_out/s4f/sweep.log
    HALP_LIB=alt_libs/$v.so timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4f/sweep.log 2>&1
  done
done
echo done
