#!/bin/bash
mkdir -p gpurun_out/s4k
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py tests/test_gpu_determinism.py -x -q > gpurun_out/s4k/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4k/tests.log
for v in fast fast2; do
  L=alt_libs/$v.so; [ $v = fast2 ] && L=paper_1803_03383_b200/libhalp_b200.so
  for w in c3 r1024 r512; do
    echo "== $v $w" >> gpurun_out/s4k/sweep.log
    HALP_LIB=$L timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4k/sweep.log 2>&1
  done
done
echo "== fast2 plans" >> gpurun_out/s4k/sweep.log
timeout 600 python tools/sweep_inner.py c3 20000 8:4,16:4,8:2 >> gpurun_out/s4k/sweep.log 2>&1
echo done
