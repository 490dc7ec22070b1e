#!/bin/bash
mkdir -p gpurun_out/s4q
HALP_LIB=alt_libs/w1.so timeout 1500 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py tests/test_gpu_svrg.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py -x -q > gpurun_out/s4q/tests_w1.log 2>&1; echo "rc=$?" >> gpurun_out/s4q/tests_w1.log
for v in w0 w1; do
  for pf in -1 0; do
    for w in c3 r1024 c2; do
      echo "== $v pf2=$pf $w" >> gpurun_out/s4q/sweep.log
      HALP_LIB=alt_libs/$v.so HALP_K3_PF2=$pf timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4q/sweep.log 2>&1
    done
  done
done
echo done
