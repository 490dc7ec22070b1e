#!/bin/bash
mkdir -p gpurun_out/s4m
for v in fast d1 d2; do
  for w in c3 r1024 c2; do
    echo "== $v $w" >> gpurun_out/s4m/sweep.log
    HALP_LIB=alt_libs/$v.so timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4m/sweep.log 2>&1
  done
done
echo done
