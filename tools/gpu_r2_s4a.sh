#!/bin/bash
# session-4 re-verification: GPU suite, smoke, bench, FX (in_levels=3) sweep
mkdir -p gpurun_out/s4a
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/s4a/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/s4a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/s4a/smoke.log
for lv in 1 3; do
  timeout 600 python tools/sweep_inner.py c3 20000 16:2,8:4,8:2 HALP_IN_LEVELS=$lv >> gpurun_out/s4a/sweep.log 2>&1
  timeout 600 python tools/sweep_inner.py c1 20000 4:2,2:4,0:0 HALP_IN_LEVELS=$lv >> gpurun_out/s4a/sweep.log 2>&1
done
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4a/bench.json 2> gpurun_out/s4a/bench.err
echo "rc=$?" >> gpurun_out/s4a/bench.err
echo done
