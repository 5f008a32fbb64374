#!/bin/bash
# round-2 pass d: dense per-unit descriptor prefetch -- parity, C4/C5 bench, per-unit trace
OUT=gpurun_out/r2d; mkdir -p $OUT
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for W in c4 c5 c2; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/bench_$W.json; python -c "
import json,sys; d=json.loads(open('$OUT/bench_$W.json').read()); print('$W', d['ms_per_step'], d['passes_ms'], d['clocks']['sm_mhz'])"; done
BLEND_LIB=paper_2411_16102_b200/libblend_tu.so timeout 300 python scripts/trace_dense.py c4 > $OUT/trace_units_c4.txt 2>&1; cat $OUT/trace_units_c4.txt | head -40
