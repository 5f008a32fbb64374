#!/bin/bash
# Round measurement pass: parity, smoke, default bench (with the CPU-oracle baseline),
# the reference arm, benches of the other configs, ncu launch lists and full captures.
TAG=${1:-r1d}
OUT=gpurun_out/prof_${TAG}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -4
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 400 $OUT/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>&1; tail -c 300 $OUT/bench_reference.json
for W in c3 c4 c5; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $OUT/bench_$W.json; done
for W in c2 c4; do
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${W}.csv \
  python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu_${W}.log 2>&1
done
for W in c2 c4 c5; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 -o $OUT/full_${W}_dense_kernel python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${W}_dense.log 2>&1
done
for W in c2 c3 c4 c5; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:streamw_kernel -s 1 -c 1 -o $OUT/full_${W}_streamw_kernel python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${W}_streamw.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:merge_kernel -s 1 -c 1 -o $OUT/full_c2_merge_kernel python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c2_merge.log 2>&1
ls $OUT
