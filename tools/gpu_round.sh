#!/bin/bash
# round evidence: bench line, ncu launch list of the bench, ncu --set full of the top kernels
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --fg-reps 2 > gpurun_out/ncu_bench.log 2>&1
for w in c3 c4 c2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_|k3_' -c 2 -f -o /tmp/full_$w python tools/prof_run.py $w > gpurun_out/ncu_full_$w.log 2>&1
  python tools/ncu_summary.py /tmp/full_$w.ncu-rep "$w" > gpurun_out/prof/full_$w.txt 2>&1
  ncu -i /tmp/full_$w.ncu-rep --page raw --csv > gpurun_out/prof/full_${w}_raw.csv 2>&1
done
echo done
