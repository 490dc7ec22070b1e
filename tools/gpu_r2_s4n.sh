#!/bin/bash
mkdir -p gpurun_out/s4n
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_halp.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s4n/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4n/tests.log
for pfa in 0 1; do
  for w in c3 r1024 r512 r2048; do
    timeout 600 python tools/sweep_inner.py $w 20000 0:0 HALP_K3_PFA=$pfa >> gpurun_out/s4n/sweep.log 2>&1
  done
  timeout 600 python tools/sweep_inner.py c1 20000 0:0 HALP_K3_PFA=$pfa HALP_K3_FAST_ALL=1 >> gpurun_out/s4n/sweep.log 2>&1
done
timeout 600 python tools/sweep_inner.py c1 20000 0:0 >> gpurun_out/s4n/sweep.log 2>&1
timeout 600 python tools/sweep_inner.py c3 20000 8:4,8:2,16:4 HALP_K3_PFA=1 >> gpurun_out/s4n/sweep.log 2>&1
echo done
