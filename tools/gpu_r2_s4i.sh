#!/bin/bash
mkdir -p gpurun_out/s4i
for v in base k5d1 k5d2; do
echo "== $v" >> gpurun_out/s4i/k5.log
HALP_LIB=alt_libs/$v.so timeout 300 python - >> gpurun_out/s4i/k5.log 2>&1 <<'PY'
import sys, json; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
ms, nd, st = bench.c5_batch(H, 0, 0, reps=3); print("C5 ms_per_batch", ms, "diverged", nd)
PY
done
