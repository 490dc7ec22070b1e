#!/bin/bash
mkdir -p gpurun_out/s4e
timeout 1500 python -m pytest tests/test_gpu_halp.py tests/test_gpu_svrg.py tests/test_gpu_k3_levels.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py -x -q > gpurun_out/s4e/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4e/tests.log
for w in c3 c2 c1; do
  timeout 600 python tools/sweep_inner.py $w 20000 0:0 >> gpurun_out/s4e/sweep.log 2>&1
done
timeout 600 python tools/sweep_inner.py c3 20000 16:2,8:2 HALP_IN_LEVELS=3 >> gpurun_out/s4e/sweep.log 2>&1
echo done
