#!/bin/bash
# session 5: K1 two-class with one rotating warp evaluating the derivative (DW): parity + same-box A/B at C4
mkdir -p gpurun_out/s5b
timeout 1500 python -m pytest tests/test_gpu_halp.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py tests/test_gpu_nccl.py -x -q > gpurun_out/s5b/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s5b/tests.log
for rep in 1 2; do
  for v in base new; do
    echo "== $v" >> gpurun_out/s5b/sweep.log
    if [ $v = base ]; then export HALP_LIB=alt_libs/base.so; else unset HALP_LIB; fi
    FG_WRAND=1 timeout 600 python tools/fg_sweep.py c4 >> gpurun_out/s5b/sweep.log 2>&1
  done
done
unset HALP_LIB
FG_WRAND=1 timeout 600 python tools/fg_sweep.py c3 >> gpurun_out/s5b/sweep.log 2>&1
echo done
