#!/bin/bash
# round-2 measurement pass l (final, after the L2 evict-first streaming loads): full GPU suite, bench lines (default C4 with cpu_baseline + e2e,
# C2/C3/C5, the C4 density sweep, whole-workload run, reference arm), ncu launch lists and
# full captures of the dominant kernels.
OUT=gpurun_out/r2l; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 400 $OUT/bench_default.json; echo
for W in c2 c3 c5 c4_t0.8 c4_t1.2 c4_t1.4; do timeout 400 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/bench_$W.json; python -c "
import json; d=json.loads(open('$OUT/bench_$W.json').read()); print('$W', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['passes_ms'].items() if isinstance(v,float)}, d['clocks']['sm_mhz'])"; done
timeout 900 python bench.py --whole --whole-samples 16 > $OUT/bench_whole.json 2> $OUT/bench_whole.err; tail -c 300 $OUT/bench_whole.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>&1; tail -c 300 $OUT/bench_reference.json; echo
for W in c4 c2; do
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$W.csv \
  python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_under_ncu_$W.log 2>&1
done
for KV in "dense_kernel:12dense_kernelI" "dense_ks_kernel:15dense_ks_kernelI" "streamw_kernel:14streamw_kernelI"; do
K=${KV%%:*}; RX=${KV#*:}
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$RX -s 3 -c 1 -o $OUT/full_c4_$K python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c4_$K.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:14streamw_kernelI -s 3 -c 1 -o $OUT/full_c2_streamw_kernel python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c2_streamw.log 2>&1
ls $OUT
