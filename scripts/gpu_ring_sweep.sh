for cfg in "4 3" "3 4" "5 2"; do
  set -- $cfg
  sed -i "s/#define SW_WARPS_CFG [0-9]*/#define SW_WARPS_CFG $1/; s/#define SW_STAGES_CFG [0-9]*/#define SW_STAGES_CFG $2/" paper_2411_16102_b200/csrc/streamw.cu
  touch paper_2411_16102_b200/csrc/streamw.cu
  python -m paper_2411_16102_b200.compile > /dev/null 2>&1 || { echo build failed $cfg; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_full or large_configs" 2>&1 | tail -1
  for W in c2 c3; do
    timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warps=$1 stages=$2 $W', round(d['ms_per_step']*1000,2), 'us', {k: round(v*1000,2) for k, v in d['passes_ms'].items() if k != 'note'})"
  done
done
