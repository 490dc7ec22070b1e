#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on K1, K3 (cluster plans + blow-up), K5, LM-HALP
mkdir -p gpurun_out/sanitizer
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in k1 k3 k5 lm; do
    timeout 900 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_run.py $case \
      > gpurun_out/sanitizer/${tool}_${case}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_${case}.log
  done
done
timeout 600 $CS --tool initcheck --target-processes all --print-limit 50 python tools/sanitize_run.py k1 k3 \
  > gpurun_out/sanitizer/initcheck_k1k3.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/initcheck_k1k3.log
echo done
