#!/bin/bash
# round-2 pass b: new GPU tests, default bench (C4), reference arm, ncu launch list + full captures
TAG=${1:-r2b}
OUT=gpurun_out/$TAG; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sharded or tp_slices or abi or fill" 2>&1 | tail -3
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 1500 $OUT/bench_default.json; tail -3 $OUT/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>&1; tail -c 300 $OUT/bench_reference.json
for W in c2 c5 c4_t0.8 c4_t1.4; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > $OUT/bench_$W.json; done
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_under_ncu_c4.log 2>&1
for K in dense_kernel streamw_kernel; do
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/full_c4_$K python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c4_$K.log 2>&1
done
ls $OUT
