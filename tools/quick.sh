#!/bin/bash
# quick GPU check: parity tests + c2 bench (accurate / fast transforms, tf32x3), no e2e / oracle timing
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for cfg in "tf32 accurate" "tf32 fast" "tf32x3 accurate" "bf16 accurate" "bf16 fast"; do
  set -- $cfg
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --mode $1 --omega $2 > gpurun_out/b_$1_$2.log 2>&1; echo "bench $1 $2 rc=$?"
  tail -1 gpurun_out/b_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['roofline']['bound'], d.get('parity'))"
done
