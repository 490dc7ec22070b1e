#!/bin/bash
# round 2 end-to-end check: GPU suite, smoke, bench (driver flags), reference arm, ncu launch list + K1 captures
mkdir -p gpurun_out/final
rm -f gpurun_out/final/*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/final/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
echo "rc=$?" >> gpurun_out/final/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 1 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
echo "rc=$?" >> gpurun_out/final/ref.err
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-e2e --no-cpu \
  > gpurun_out/final/ncu_launch.log 2>&1
# full captures are read on the box (the .ncu-rep files exceed the 64 MiB return limit)
for w in c3 c4; do
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k1_stream -c 1 -o /tmp/k1_$w -f python tools/prof_run.py $w > gpurun_out/final/k1_${w}_ncu.log 2>&1
  $NCU -i /tmp/k1_$w.ncu-rep --page details > gpurun_out/final/k1_${w}_details.txt 2>&1
  $NCU -i /tmp/k1_$w.ncu-rep --page raw --csv > gpurun_out/final/k1_${w}_raw.csv 2>&1
  $NCU -i /tmp/k1_$w.ncu-rep --page source --csv > gpurun_out/final/k1_${w}_source.csv 2>&1
done
echo done
