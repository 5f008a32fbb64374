#!/bin/bash
# ncu --set full capture (with source) of one kernel of one workload's step; exports the SASS
# source page (per-instruction stall samples) as CSV for reading here.
# usage: bash scripts/gpu_ncu_kernel.sh <out-tag> <workload> <mangled-name regex>
OUT=gpurun_out/$1; W=$2; RX=$3; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$RX -s 3 -c 1 -o $OUT/full python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
$NCU -i $OUT/full.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2> $OUT/source.err
$NCU -i $OUT/full.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ls -la $OUT
