#!/bin/bash
# A/B of the inner loop: current build vs alt_libs/$1.so on C2
mkdir -p gpurun_out
for T in 8000 30000; do
for i in 1 2; do
  HALP_LIB=alt_libs/$1.so PROF_T=$T timeout 300 python tools/prof_run.py c2 2>&1 | sed "s/^/$1 T=$T /" | cut -c1-300 >> gpurun_out/ab.log
  PROF_T=$T timeout 300 python tools/prof_run.py c2 2>&1 | sed "s/^/cur T=$T /" | cut -c1-300 >> gpurun_out/ab.log
done
done
echo done
