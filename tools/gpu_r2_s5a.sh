#!/bin/bash
# session 5 check of HEAD on a fresh box: build check, GPU suite, smoke, bench and reference arm at the driver's default flags
mkdir -p gpurun_out/s5a
rm -f gpurun_out/s5a/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5a/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s5a/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/s5a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5a/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/s5a/smoke.log
timeout 1500 python bench.py --impl reference > gpurun_out/s5a/ref.json 2> gpurun_out/s5a/ref.err
echo "rc=$?" >> gpurun_out/s5a/ref.err
timeout 1500 python bench.py > gpurun_out/s5a/bench.json 2> gpurun_out/s5a/bench.err
echo "rc=$?" >> gpurun_out/s5a/bench.err
echo done
