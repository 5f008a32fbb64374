#!/bin/bash
# Profiling pass on the GPU box: launch lists (per-launch device times) of the bench on
# c2 (the default workload) and c4, and one --set full capture of each hot kernel.
TAG=${1:-r1c}
OUT=gpurun_out/prof_${TAG}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
for W in c2 c4; do
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${W}.csv \
  python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu_${W}.log 2>&1
done
for W in c4 c5; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 -o $OUT/full_${W}_dense_kernel python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${W}_dense.log 2>&1
done
for W in c2 c3; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:streamw_kernel -s 1 -c 1 -o $OUT/full_${W}_streamw_kernel python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${W}_streamw.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:merge_kernel -s 1 -c 1 -o $OUT/full_c2_merge_kernel python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c2_merge.log 2>&1
ls -la $OUT
