#!/bin/bash
mkdir -p gpurun_out/s4g
python -m paper_1803_03383_b200.build > gpurun_out/s4g/build.log 2>&1
for v in base of1 of2 of4 ef3; do
  echo "== $v" >> gpurun_out/s4g/c4.txt
  HALP_LIB=alt_libs/$v.so FG_WRAND=1 timeout 600 python tools/fg_sweep.py c4 "" >> gpurun_out/s4g/c4.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_determinism.py -x -q > gpurun_out/s4g/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4g/tests.log
echo done
