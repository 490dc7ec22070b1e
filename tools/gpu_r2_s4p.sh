#!/bin/bash
mkdir -p gpurun_out/s4p
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py tests/test_gpu_determinism.py -x -q > gpurun_out/s4p/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4p/tests.log
for v in fast unroll2 wip; do
  L=alt_libs/$v.so; [ $v = wip ] && L=paper_1803_03383_b200/libhalp_b200.so
  for w in c3 r1024 c2; do
    echo "== $v $w" >> gpurun_out/s4p/sweep.log
    HALP_LIB=$L timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4p/sweep.log 2>&1
  done
done
echo done
