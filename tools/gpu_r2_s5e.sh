#!/bin/bash
# session 5: K1 with larger tiles per barrier (4-row / 8-row, 64 KB tiles in a 3-deep ring): parity + A/B against the old rows
mkdir -p gpurun_out/s5e
timeout 1500 python -m pytest tests/test_gpu_halp.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py tests/test_gpu_nccl.py tests/test_gpu_svrg.py -x -q > gpurun_out/s5e/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s5e/tests.log
S=gpurun_out/s5e/sweep.log
FG_WRAND=1 timeout 900 python tools/fg_sweep.py c3 "" HALP_FG_ROWS=2,HALP_FG_STAGES=4 "" >> $S 2>&1
FG_WRAND=1 timeout 900 python tools/fg_sweep.py sq:8388608:2048:f32 "" HALP_FG_ROWS=2,HALP_FG_STAGES=4 HALP_FG_ROWS=4,HALP_FG_STAGES=4 >> $S 2>&1
FG_WRAND=1 timeout 900 python tools/fg_sweep.py sq:16777216:1024:f32 "" HALP_FG_ROWS=4,HALP_FG_STAGES=4 >> $S 2>&1
FG_WRAND=1 timeout 900 python tools/fg_sweep.py sq:4194304:2048:f64 "" HALP_FG_ROWS=2,HALP_FG_STAGES=4 >> $S 2>&1
FG_WRAND=1 timeout 900 python tools/fg_sweep.py sq:8388608:4096:bf16 "" HALP_FG_ROWS=2,HALP_FG_STAGES=4 >> $S 2>&1
FG_WRAND=1 timeout 900 python tools/fg_sweep.py c4 >> $S 2>&1
echo done
