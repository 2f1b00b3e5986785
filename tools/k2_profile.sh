#!/bin/bash
# ncu --set full of the FFMA K2 kernels at one config (default: config 5, R = 32).
#   gpurun -- 'bash tools/k2_profile.sh <tag> ["--config 5 --rank 32"]'
set -u
T=${1:-k2p}; A=${2:---config 5 --rank 32}
O=gpurun_out; mkdir -p $O
python bench.py $A --steps 3 --warmup 2 --no-cpu --no-e2e > $O/${T}_bench.jsonl 2> $O/${T}_bench.err
ncu --set full --clock-control none --import-source on -k regex:"corr_kernel|corr_few" -c 4 \
  -o $O/${T}_full python bench.py $A --images 1 --steps 1 --warmup 0 --no-cpu --no-e2e > $O/${T}_ncu.log 2>&1
echo done
