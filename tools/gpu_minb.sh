#!/bin/bash
mkdir -p gpurun_out
for lib in "" alt_libs/logw0.so; do
echo "== ${lib:-default}"
HALP_LIB=$lib FG_WRAND=1 timeout 900 python tools/fg_sweep.py c4 "" HALP_FG_ROWS=16,HALP_FG_STAGES=3 HALP_FG_ROWS=16,HALP_FG_STAGES=2
done > gpurun_out/minb.log 2>&1
echo done
