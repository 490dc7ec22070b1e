#!/bin/bash
# session 5: K1 two-class parity + same-box A/B at C4.  Variants are the libraries under alt_libs/
# (tools/build_alt.sh); "new" is the in-tree build.   usage: gpu_r2_s5b.sh [variant ...]
mkdir -p gpurun_out/s5b
timeout 1500 python -m pytest tests/test_gpu_halp.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py tests/test_gpu_nccl.py -x -q > gpurun_out/s5b/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s5b/tests.log
VARS="${@:-base new}"
for rep in 1 2; do
  for v in $VARS; do
    echo "== $v" >> gpurun_out/s5b/sweep.log
    if [ $v = new ]; then unset HALP_LIB; else export HALP_LIB=alt_libs/$v.so; fi
    FG_WRAND=1 timeout 600 python tools/fg_sweep.py c4 >> gpurun_out/s5b/sweep.log 2>&1
  done
done
unset HALP_LIB
FG_WRAND=1 timeout 600 python tools/fg_sweep.py c3 >> gpurun_out/s5b/sweep.log 2>&1
echo done
