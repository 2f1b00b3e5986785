#!/bin/bash
# One measurement campaign on the GPU box: the bench line, the reference arm,
# the other configs through the full path, the launch list and one --set full
# capture of every path kernel.  Outputs go to gpurun_out/<tag>_*; copy the
# ones to keep into profiles/ and summarise with tools/ncu_summary.py.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/run_campaign.sh r2c'
set -u
TAG=${1:?tag}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
python bench.py --impl reference > $OUT/${TAG}_bench_reference.jsonl 2> $OUT/${TAG}_ref.err
: > $OUT/${TAG}_configs.jsonl
for args in "--config 1" "--config 2 --rank 4" "--config 2 --rank 8" "--config 2 --rank 16" \
            "--config 2 --rank 32" "--config 3 --steps 5" "--config 5 --steps 5" \
            "--config 5 --rank 32 --steps 5" "--config 5 --basis dense --steps 5"; do
  python bench.py $args --no-e2e 2>> $OUT/${TAG}_configs.err | grep '^{' >> $OUT/${TAG}_configs.jsonl
done
python tools/bench_images.py > $OUT/${TAG}_images_e2e.jsonl 2> $OUT/${TAG}_images.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv \
    python bench.py --images 8 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"project_|corr_|prefix_kernel|place|ranges_init" -c 9 \
    -o $OUT/${TAG}_full python bench.py --images 8 --steps 1 --warmup 0 --no-cpu --no-e2e \
    > $OUT/${TAG}_full.log 2>&1
echo done
