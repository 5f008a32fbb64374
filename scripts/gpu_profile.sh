#!/bin/bash
# Runs on the GPU box (via gpurun): launch lists + one full ncu capture of each hot
# kernel.  Output under gpurun_out/prof_<tag>/ ; summaries are copied to profiles/.
set -u
TAG=${1:-r1}
WL=${2:-c2}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
# 1) per-launch device times of one bench run (cold-cache, serialised)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${WL}.csv \
  python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu_${WL}.log 2>&1
# 2) full sets of the hot kernels (skip the warm-up launches)
for K in stream_kernel dense_kernel merge_kernel; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $OUT/full_${WL}_${K} python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_${WL}_${K}.log 2>&1
done
ls -la $OUT
