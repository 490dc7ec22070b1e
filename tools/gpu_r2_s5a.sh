#!/bin/bash
# session 5 re-entry check: GPU suite, smoke, bench at the driver's flags
mkdir -p gpurun_out/s5a
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s5a/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/s5a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5a/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/s5a/smoke.log
timeout 1500 python bench.py > gpurun_out/s5a/bench.json 2> gpurun_out/s5a/bench.err
echo "rc=$?" >> gpurun_out/s5a/bench.err
echo done
