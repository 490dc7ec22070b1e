#!/bin/bash
mkdir -p gpurun_out
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_harness.py -x -q --durations=10 > gpurun_out/r2_harness.log 2>&1
echo "rc=$?" >> gpurun_out/r2_harness.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k5_batch -s 1 -c 1 -o gpurun_out/r2_k5 -f python tools/prof_run.py c5 > gpurun_out/r2_k5_ncu.log 2>&1
timeout 900 python tools/sweep_inner.py c3 20000 16:1,16:2,16:4,8:2,8:4,8:8,4:8 > gpurun_out/r2_sweep_c3.log 2>&1
timeout 900 python tools/sweep_inner.py c2 20000 16:2,16:4,16:8,8:4,8:8 > gpurun_out/r2_sweep_c2.log 2>&1
echo done
