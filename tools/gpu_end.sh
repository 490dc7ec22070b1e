#!/bin/bash
# round-end evidence: GPU parity suite, smoke, reference arm, torchrun, default bench, launch list, C4/C3 K1 full capture
mkdir -p gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_final.sh
for w in c4 c3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_' -c 1 -f -o /tmp/full_$w python tools/prof_run.py $w > gpurun_out/ncu_full_$w.log 2>&1
  python tools/ncu_summary.py /tmp/full_$w.ncu-rep "$w" > gpurun_out/prof/full_$w.txt 2>&1
done
echo alldone
