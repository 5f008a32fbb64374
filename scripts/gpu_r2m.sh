#!/bin/bash
# round-2 closing pass m: the final planner (dense cap from the two-tile share); kernels as in r2l
# (whose ncu full captures stand): GPU suite, bench lines, C4 launch list.
OUT=gpurun_out/r2m; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 400 $OUT/bench_default.json; echo
for W in c2 c3 c5 c4_t0.8 c4_t1.2 c4_t1.4; do timeout 400 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/bench_$W.json; python -c "
import json; d=json.loads(open('$OUT/bench_$W.json').read()); print('$W', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['passes_ms'].items() if isinstance(v,float)}, d['clocks']['sm_mhz'])"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>&1; tail -c 300 $OUT/bench_reference.json; echo
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_under_ncu_c4.log 2>&1
ls $OUT
