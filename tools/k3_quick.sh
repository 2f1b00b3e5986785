#!/bin/bash
# Quick K3 check on the GPU box: the placement parity subset, one bench line
# (device-resident steps) and the ncu duration / instruction count of the K3
# launches.  Usage: gpurun -- 'bash tools/k3_quick.sh <tag> [pytest -k expr]'
T=$1
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "${2:-placement or config4_full or randomized or tau}" > gpurun_out/${T}_tests.log 2>&1
echo rc=$? >> gpurun_out/${T}_tests.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/${T}_bench.jsonl 2>&1
timeout 300 ncu --clock-control none -k regex:place \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --csv python bench.py --images 8 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${T}_ncu.csv 2>/dev/null
