#!/bin/bash
# A/B: default build vs alt_libs/minb3.so (__launch_bounds__ min 3 CTAs/SM for K1)
mkdir -p gpurun_out
for lib in "" alt_libs/minb3.so; do
echo "== ${lib:-default}"
HALP_LIB=$lib FG_WRAND=1 timeout 400 python tools/fg_sweep.py c4 ""
HALP_LIB=$lib FG_WRAND=1 timeout 400 python tools/fg_sweep.py c3 ""
done > gpurun_out/minb3.log 2>&1
echo done
