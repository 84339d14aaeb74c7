# round-end check: GPU suite, smoke, default bench line, reference arm
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/final_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), d['config']['omega_transform'], round(d['roofline']['frac'],3), d['roofline']['traffic'], d['clocks'], d['gpu_launches'], d['e2e']['value'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_ref.log | cut -c1-300
