#!/bin/bash
mkdir -p gpurun_out
python -m paper_1803_03383_b200.build > gpurun_out/r2_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_k3_levels.py -x -q > gpurun_out/r2_lv2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_lv2_tests.log
for lv in 1 2; do
  timeout 600 python tools/sweep_inner.py c3 20000 16:2,16:4,8:4,8:2 HALP_IN_LEVELS=$lv >> gpurun_out/r2_lv2_sweep.log 2>&1
done
timeout 300 python - > gpurun_out/r2_h2d.log 2>&1 <<'PY'
import torch, time
x = torch.empty(8 * 2**30, dtype=torch.uint8, pin_memory=True); d = torch.empty_like(x, device="cuda")
for _ in range(2): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); d.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("pinned H2D GB/s", x.numel() / e0.elapsed_time(e1) / 1e6)
PY
echo done
