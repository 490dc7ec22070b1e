#!/bin/bash
mkdir -p gpurun_out/fx
rm -f gpurun_out/parity_counts.jsonl
python -m paper_1803_03383_b200.build > gpurun_out/fx/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_k3_levels.py tests/test_gpu_determinism.py tests/test_gpu_baseline_configs.py::test_c5_problems -x -q > gpurun_out/fx/tests.log 2>&1; echo "rc=$?" >> gpurun_out/fx/tests.log
for lv in 1 3; do
  timeout 600 python tools/sweep_inner.py c3 20000 16:2,8:4,8:2 HALP_IN_LEVELS=$lv >> gpurun_out/fx/sweep.log 2>&1
  timeout 600 python tools/sweep_inner.py c1 20000 4:2,2:4,0:0 HALP_IN_LEVELS=$lv >> gpurun_out/fx/sweep.log 2>&1
done
timeout 600 python tools/e2e_overlap_probe.py > gpurun_out/fx/probe.log 2>&1
echo done
