#!/bin/bash
mkdir -p gpurun_out/e2e
python -m paper_1803_03383_b200.build > gpurun_out/e2e/build.log 2>&1
timeout 600 python tools/e2e_overlap_probe.py > gpurun_out/e2e/probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -q > gpurun_out/e2e/batch_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e2e/batch_tests.log
for w in 2 4; do
HALP_K5_WARPS=$w timeout 300 python - >> gpurun_out/e2e/k5.log 2>&1 <<'PY'
import sys, os; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
ms, nd, st = bench.c5_batch(H, 0, 0, reps=3); print("warps", os.environ["HALP_K5_WARPS"], "C5 ms_per_batch", ms, "diverged", nd)
PY
done
echo done
