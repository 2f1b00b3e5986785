#!/bin/bash
# K2 FFMA A/B on the GPU box: parity subset, then per-config bench lines with
# an environment switch off (=0) and on (default).  Usage:
#   gpurun -- 'bash tools/k2_ab.sh <tag> <ENVVAR> [pytest -k expr]'
T=$1; V=$2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "${3:-correlat or cp_engines or dense or config2 or config3 or config5 or prefix or randomized}" \
  > gpurun_out/${T}_tests.log 2>&1
echo rc=$? >> gpurun_out/${T}_tests.log
: > gpurun_out/${T}_ab.jsonl
for args in "--config 5 --rank 32 --steps 5" "--config 5 --basis dense --steps 5" \
            "--config 2 --rank 32" "--config 2 --rank 16" "--config 3 --steps 5"; do
  for v in 0 1; do
    env $V=$v timeout 300 python bench.py $args --no-cpu --no-e2e 2>> gpurun_out/${T}_ab.err \
      | grep '^{' | sed "s/^{/{\"ab\": \"$V=$v\", /" >> gpurun_out/${T}_ab.jsonl
  done
done
