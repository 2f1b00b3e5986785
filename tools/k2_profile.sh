set -u
O=gpurun_out
python bench.py --config 5 --rank 32 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/k2p_c5r32.jsonl 2> $O/k2p_c5r32.err
ncu --set full --clock-control none --import-source on -k regex:"corr_kernel|corr_few" -c 4 \
  -o $O/k2p_c5r32_full python bench.py --config 5 --rank 32 --images 1 --steps 1 --warmup 0 --no-cpu --no-e2e > $O/k2p_ncu.log 2>&1
echo done
