#!/bin/bash
mkdir -p gpurun_out/s4j
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py -x -q > gpurun_out/s4j/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4j/tests.log
for v in base fast; do
  for w in c3 c1 r512 r1024; do
    echo "== $v $w" >> gpurun_out/s4j/sweep.log
    HALP_LIB=alt_libs/$v.so timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4j/sweep.log 2>&1
  done
done
echo done
