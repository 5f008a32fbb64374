python -m paper_2411_16102_b200.compile >/dev/null 2>&1
for W in c4 c5 c3; do for CAP in 0 128 112 96; do
  BLEND_DENSE_CTAS=$CAP timeout 300 python bench.py --workload $W --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W cap=$CAP', round(d['ms_per_step'],4), {k: round(v,4) for k, v in d['passes_ms'].items() if k != 'note'})"
done; done
