python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed; exit 1; }
python scripts/trace_dense.py c2 > gpurun_out/trace_c2.txt 2>&1
for P in 0 10 12; do
  for W in c5 c4; do BLEND_POLY=$P timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/poly_${P}_$W.json
  python -c "import json; d=json.load(open('gpurun_out/poly_${P}_$W.json')); print('$P $W', round(d['ms_per_step'],4), {k: round(v,4) for k, v in d['passes_ms'].items() if k != 'note'})"; done
done
cat gpurun_out/trace_c2.txt
