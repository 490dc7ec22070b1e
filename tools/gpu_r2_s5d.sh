#!/bin/bash
# session 5: K1 at C3 with 4-row tiles (x slice in registers: r4reg; x re-read from shared memory: r4rr)
mkdir -p gpurun_out/s5d
for rep in 1 2; do
  echo "== r4reg default plan (2 rows x 4 stages)" >> gpurun_out/s5d/sweep.log
  HALP_LIB=alt_libs/r4reg.so FG_WRAND=1 timeout 600 python tools/fg_sweep.py c3 >> gpurun_out/s5d/sweep.log 2>&1
  for v in r4reg r4rr; do
    echo "== $v" >> gpurun_out/s5d/sweep.log
    HALP_LIB=alt_libs/$v.so FG_WRAND=1 timeout 900 python tools/fg_sweep.py c3 HALP_FG_ROWS=4,HALP_FG_STAGES=3 HALP_FG_ROWS=4,HALP_FG_STAGES=2 >> gpurun_out/s5d/sweep.log 2>&1
  done
done
echo done
