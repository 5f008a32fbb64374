#!/bin/bash
# quick iteration on the GPU box: parity, c2/c3 benches, ncu of the streaming kernel on c2
TAG=${1:-iter}
OUT=gpurun_out/prof_${TAG}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for W in c2 c3 c5; do timeout 240 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$W.json; done
for f in gpurun_out/bench_c2.json gpurun_out/bench_c3.json gpurun_out/bench_c5.json; do
  python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {k: round(v,4) for k, v in d['passes_ms'].items() if k != 'note'})"
done
if [ -n "${NCU_C2:-}" ]; then
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:streamw_kernel -s 3 -c 1 -o $OUT/full_c2_streamw python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_c2_streamw.log 2>&1
fi
