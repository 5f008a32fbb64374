#!/bin/bash
# round-2 pass c: NEXT-2/NEXT-3 GPU tests, whole-workload bench, full GPU suite
OUT=gpurun_out/r2c; mkdir -p $OUT
python -m paper_2411_16102_b200.compile > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "alg2 or scheduled" 2>&1 | tail -3
timeout 900 python bench.py --whole --whole-samples 16 > $OUT/bench_whole.json 2> $OUT/bench_whole.err; tail -c 1500 $OUT/bench_whole.json; tail -3 $OUT/bench_whole.err
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
