#!/bin/bash
# diagnostics: dense / streaming pass times of variant builds (BLEND_LIB) on the given workloads
# usage: bash scripts/gpu_variants.sh "c5 c4" base p2 x32 ...   (base = libblend.so)
WLS=$1; shift
python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
for W in $WLS; do for V in "$@"; do
  if [ "$V" = base ]; then LIBP=paper_2411_16102_b200/libblend.so; else LIBP=paper_2411_16102_b200/libblend_$V.so; fi
  BLEND_LIB=$LIBP timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); p=d['passes_ms']; print(f\"$W %-6s step %8.3f ms  dense %8.3f  stream %8.3f  merge %6.3f  clk %s\" % ('$V', d['ms_per_step'], p['dense'], p['stream'], p['merge'], d['clocks']['sm_mhz']))
except Exception as e: print('$W $V failed', e)"
done; done
