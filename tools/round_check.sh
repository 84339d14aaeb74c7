# full GPU suite + default bench + bf16/fast bench line
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_all.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?"
python bench.py --steps 20 --warmup 3 --omega fast --no-e2e --no-cpu-baseline > gpurun_out/bench_fast.log 2>&1; echo "bench fast rc=$?"
for f in bench_default bench_fast; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), round(d['value'],1), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, round(d['roofline']['frac'],3), d['clocks'], d.get('parity'), {k: round(v['ms_per_step'],3) for k,v in d.get('other_modes',{}).items() if 'ms_per_step' in v})"; done
