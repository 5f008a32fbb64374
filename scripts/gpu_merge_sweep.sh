python -m paper_2411_16102_b200.compile >/dev/null 2>&1
for cfg in "256 1 0" "64 1 0" "128 1 60" "256 0 0" "64 0 0"; do
  set -- $cfg
  echo "threads=$1 pdl=$2 smem=$3"
  BLEND_MT=$1 BLEND_MPDL=$2 BLEND_MSMEM=$3 python scripts/trace_stream.py c2 0 2>/dev/null | grep merge
  BLEND_MT=$1 BLEND_MPDL=$2 BLEND_MSMEM=$3 timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us', {k: round(v*1000,2) for k, v in d['passes_ms'].items() if k != 'note'})"
done
