#!/bin/bash
mkdir -p gpurun_out/s4d
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/s4d/clocks.csv &
SMI=$!
timeout 900 python tools/fg_sweep.py c4 "" HALP_FG_MAX_SPLITS=8192 HALP_FG_MAX_SPLITS=16384 HALP_FG_MAX_SPLITS=32768 > gpurun_out/s4d/c4.txt 2>&1
timeout 900 python tools/fg_sweep.py c3 "" HALP_FG_MAX_SPLITS=8192 HALP_FG_MAX_SPLITS=16384 > gpurun_out/s4d/c3.txt 2>&1
kill $SMI
echo done
