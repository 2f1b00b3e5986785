#!/bin/bash
# A/B of two builds of the library (DPM_LIB) on per-config bench lines.
#   gpurun -- 'bash tools/lib_ab.sh <tag> <variant.so> "<bench args>" ["<bench args>" ...]'
T=$1; V=$2; shift 2
mkdir -p gpurun_out; : > gpurun_out/${T}_ab.jsonl
for args in "$@"; do
  for lib in default $V; do
    if [ $lib = default ]; then unset DPM_LIB; else export DPM_LIB=$PWD/$lib; fi
    timeout 300 python bench.py $args --no-cpu --no-e2e 2>> gpurun_out/${T}_ab.err \
      | grep '^{' | sed "s|^{|{\"lib\": \"$lib\", |" >> gpurun_out/${T}_ab.jsonl
  done
done
unset DPM_LIB
