#!/bin/bash
# ncu --set full capture (with source) of the C4 two-tile dense kernel, serialised step; the
# source page (SASS, per-instruction stall samples) is exported as CSV for reading here.
OUT=gpurun_out/${1:-ncu_dense}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:12dense_kernelI -s 3 -c 1 -o $OUT/full_c4_dense python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
$NCU -i $OUT/full_c4_dense.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2> $OUT/source.err
$NCU -i $OUT/full_c4_dense.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ls -la $OUT
