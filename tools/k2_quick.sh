#!/bin/bash
# Quick K2 check on the GPU box: the correlation parity subset and the
# per-config bench lines (device-resident steps).  Usage:
#   gpurun -- 'bash tools/k2_quick.sh <tag> [pytest -k expr]'
T=$1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "${2:-correlat or cp_engines or dense or config2 or config3 or config5 or detect or tensor_core or prefix}" \
  > gpurun_out/${T}_tests.log 2>&1
echo rc=$? >> gpurun_out/${T}_tests.log
: > gpurun_out/${T}_configs.jsonl
for args in "--config 4" "--config 2 --rank 16" "--config 3 --steps 5" "--config 5 --steps 5" \
            "--config 5 --rank 32 --steps 5"; do
  timeout 300 python bench.py $args --no-cpu --no-e2e 2>> gpurun_out/${T}_configs.err | grep '^{' >> gpurun_out/${T}_configs.jsonl
done
