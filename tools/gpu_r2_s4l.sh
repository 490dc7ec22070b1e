#!/bin/bash
mkdir -p gpurun_out/s4l
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s4l/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4l/tests.log
for rep in 1 2; do
for v in fast wip; do
  L=alt_libs/$v.so; [ $v = wip ] && L=paper_1803_03383_b200/libhalp_b200.so
  for w in c3 r1024; do
    echo "== $v $w" >> gpurun_out/s4l/sweep.log
    HALP_LIB=$L timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4l/sweep.log 2>&1
  done
done
done
echo done
