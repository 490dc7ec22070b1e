#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_halp.py -x -q -k "two_level" > gpurun_out/pytest_two.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_two.log
rm -f gpurun_out/ab2.log
for v in 2 1; do
  HALP_IN_LEVELS=$v PROF_T=30000 timeout 300 python tools/prof_run.py c2 2>&1 | sed "s/^/L=$v /" | cut -c1-120 >> gpurun_out/ab2.log
done
timeout 600 python tools/sweep_inner.py c3 8000 0:0 HALP_IN_LEVELS=2 >> gpurun_out/ab2.log 2>&1
timeout 600 python tools/sweep_inner.py c3 8000 0:0 HALP_IN_LEVELS=1 >> gpurun_out/ab2.log 2>&1
echo done
