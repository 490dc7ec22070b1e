#!/bin/bash
mkdir -p gpurun_out/fix
python -m paper_1803_03383_b200.build > gpurun_out/fix/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_k3_levels.py tests/test_gpu_svrg.py -q > gpurun_out/fix/tests.log 2>&1; echo "rc=$?" >> gpurun_out/fix/tests.log
timeout 900 python tools/fg_sweep.py c4 "" HALP_FG_MAX_SPLITS=8192 HALP_FG_MAX_SPLITS=16384 > gpurun_out/fix/fg_c4.log 2>&1
timeout 900 python tools/fg_sweep.py c3 "" HALP_FG_MAX_SPLITS=8192 > gpurun_out/fix/fg_c3.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu > gpurun_out/fix/bench.json 2> gpurun_out/fix/bench.err
echo done
