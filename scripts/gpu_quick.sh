#!/bin/bash
# quick iteration on the GPU box: build, parity (-m gpu), benches of the listed workloads
WLS=${1:-"c2 c4 c5"}
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for W in $WLS; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$W.json; done
for W in $WLS; do
  python -c "import json; d=json.load(open('gpurun_out/bench_$W.json')); print('$W', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), {k: round(v,4) for k, v in d['passes_ms'].items() if k != 'note'})" 2>&1 | tail -1
done
