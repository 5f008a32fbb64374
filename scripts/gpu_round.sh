#!/bin/bash
# one GPU round: smoke, parity, benches, ncu captures -> gpurun_out/
TAG=${1:-r1b}
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -4 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for W in c2 c3 c5 c4; do timeout 240 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$W.json; done
timeout 240 python bench.py --workload c2 --steps 20 --warmup 3 --dense-split 2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c2_ds2.json
