#!/bin/bash
mkdir -p gpurun_out/k3opt
python -m paper_1803_03383_b200.build > gpurun_out/k3opt/build.log 2>&1
timeout 600 python tools/e2e_overlap_probe.py > gpurun_out/k3opt/probe.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_halp.py tests/test_gpu_k3_levels.py tests/test_gpu_determinism.py tests/test_gpu_svrg.py tests/test_gpu_baseline_configs.py -x -q > gpurun_out/k3opt/tests.log 2>&1; echo "rc=$?" >> gpurun_out/k3opt/tests.log
timeout 600 python tools/sweep_inner.py c3 20000 16:2 > gpurun_out/k3opt/sweep.log 2>&1
timeout 600 python tools/sweep_inner.py c2 20000 16:4 >> gpurun_out/k3opt/sweep.log 2>&1
for w in 1 2 4; do
HALP_K5_WARPS=$w timeout 300 python - >> gpurun_out/k3opt/grid.log 2>&1 <<'PY'
import sys, os; sys.path.insert(0, ".")
import bench, paper_1803_03383_b200 as H
g = bench.grid_bench(H, 0); print("warps", os.environ["HALP_K5_WARPS"], "grid device_ms", g["device_ms"], "wall", g["wall_ms"])
PY
done
echo done
