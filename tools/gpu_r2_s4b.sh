#!/bin/bash
# FX exchange with st.async integer records: tests + sweep; latency microbenchmark
mkdir -p gpurun_out/s4b
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/micro/lat.cu && /tmp/lat > gpurun_out/s4b/lat.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_determinism.py -x -q > gpurun_out/s4b/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4b/tests.log
for lv in 1 3; do
  timeout 600 python tools/sweep_inner.py c3 20000 16:2,8:4,8:2,16:1 HALP_IN_LEVELS=$lv >> gpurun_out/s4b/sweep.log 2>&1
  timeout 600 python tools/sweep_inner.py c1 20000 4:2,2:4,1:2,1:1,2:1 HALP_IN_LEVELS=$lv >> gpurun_out/s4b/sweep.log 2>&1
done
echo done
