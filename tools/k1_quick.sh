#!/bin/bash
# Quick K1 check on the GPU box: the K1 + K2 parity subset with the mma.sync
# projection (default) , one bench line each for DPM_K1MMA=1 / 0 (device-
# resident steps) and the ncu counters of both K1 kernels.
# Usage: gpurun -- 'bash tools/k1_quick.sh <tag> [pytest -k expr]'
T=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_accuracy_table.py -x -q -m gpu \
  -k "${2:-correlate or cp_engine or dense or config1 or config2 or tensor_core or randomized or accuracy or known or prefix}" \
  > gpurun_out/${T}_tests.log 2>&1
echo rc=$? >> gpurun_out/${T}_tests.log
for m in 1 0 1 0; do
  DPM_K1MMA=$m timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | grep '^{' \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'DPM_K1MMA': $m, 'ms_per_step': d['ms_per_step'], 'value': d['value'], 'kernel_ms': d['kernel_ms'], 'k1': d['rooflines']['k1_project']}))" \
    >> gpurun_out/${T}_ab.jsonl
done
for m in 1 0; do
  DPM_K1MMA=$m timeout 300 ncu --clock-control none -k regex:project -c 1 \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum \
    --csv python bench.py --images 8 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${T}_ncu_mma$m.csv 2>/dev/null
done
tail -3 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_ab.jsonl
