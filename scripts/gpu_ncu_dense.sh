#!/bin/bash
TAG=${1:-r1c}
OUT=gpurun_out/prof_${TAG:-r1c}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for W in c4 c5; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 -o $OUT/full_${W}_dense_kernel python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${W}_dense.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:streamw_kernel -s 1 -c 1 -o $OUT/full_c2_streamw_kernel python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c2_streamw.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:streamw_kernel -s 1 -c 1 -o $OUT/full_c3_streamw_kernel python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3_streamw.log 2>&1
ls -la $OUT
