#!/bin/bash
# ncu --set full captures for the C2 (default bench) kernels and the C4 dense kernel
TAG=${1:-c2x}
OUT=gpurun_out/prof_${TAG}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
for K in dense_kernel streamw_kernel merge_kernel; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/full_c2_$K python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c2_$K.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 -o $OUT/full_c4_dense_kernel python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c4_dense.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu_c2.log 2>&1
ls -la $OUT
