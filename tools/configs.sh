#!/bin/bash
for wl in "$@"; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --mode ${MODE:-tf32} --omega ${OMEGA:-fast} --e2e-steps 2 > gpurun_out/cfg_$wl.log 2>&1
  echo "workload=$wl rc=$?"
  tail -1 gpurun_out/cfg_$wl.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), 'tflops', round(d['tflops'],1), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), 'parity', d.get('parity'), 'cpu', d.get('cpu_baseline',{}).get('value'), 'e2e', d.get('e2e',{}).get('value'))
except Exception as e: print('no json', e)"
done
