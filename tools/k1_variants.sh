#!/bin/bash
# K1 time of several builds of the library (DPM_LIB), device-resident steps.
#   gpurun -- 'bash tools/k1_variants.sh <tag> <lib.so> [<lib.so> ...]'
T=$1; shift
mkdir -p gpurun_out; : > gpurun_out/${T}_variants.jsonl
for rep in 1 2; do
  for lib in default "$@"; do
    if [ $lib = default ]; then unset DPM_LIB; else export DPM_LIB=$PWD/$lib; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep '^{' \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'ms_per_step': round(d['ms_per_step'],4), 'k1_ms': round(d['kernel_ms']['k1_project'],4), 'k1_frac': round(d['rooflines']['k1_project']['frac'],4)}))" \
      | tee -a gpurun_out/${T}_variants.jsonl
  done
done
unset DPM_LIB
