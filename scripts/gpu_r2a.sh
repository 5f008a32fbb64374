#!/bin/bash
# round-2 first pass: build, full GPU parity, quick benches
python -m paper_2411_16102_b200.compile > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -rs 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; tail -6 gpurun_out/pytest_gpu.txt
timeout 300 python -m pytest tests/test_gpu_numerics.py -q -s -k peaked 2>&1 | grep "path counters" > gpurun_out/counters.txt
for W in c2 c4 c5; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$W.json; done
for W in c2 c4 c5; do
  python -c "import json; d=json.load(open('gpurun_out/bench_$W.json')); print('$W', round(d['value']), round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), {k: round(v,4) for k, v in d['passes_ms'].items() if k != 'note'}, d['clocks'])" 2>&1 | tail -1
done
