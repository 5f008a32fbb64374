#!/bin/bash
# round-2 pass f: 128-key-block dense mainloop -- quick parity, numerics, bench, trace
OUT=gpurun_out/r2f; mkdir -p $OUT
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_bf16 or random_trees_bf16 or group_sizes" 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py -q -x 2>&1 | tail -4
for W in c4 c5 c2; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/bench_$W.json; python -c "
import json,sys; d=json.loads(open('$OUT/bench_$W.json').read()); print('$W', d['ms_per_step'], d['passes_ms'], d['clocks']['sm_mhz'])"; done
BLEND_LIB=paper_2411_16102_b200/libblend_tu.so timeout 300 python scripts/trace_dense.py c4 > $OUT/trace_units_c4.txt 2>&1; head -16 $OUT/trace_units_c4.txt
