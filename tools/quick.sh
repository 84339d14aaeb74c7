#!/bin/bash
# quick GPU check: parity tests + c2 bench (accurate / fast transforms), no e2e / oracle timing
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for om in accurate fast; do
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --omega $om "$@" > gpurun_out/b_$om.log 2>&1; echo "bench $om rc=$?"
  tail -1 gpurun_out/b_$om.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phases_ms_per_step'], d['roofline']['frac'], d['roofline']['bound'], d.get('parity'))"
done
