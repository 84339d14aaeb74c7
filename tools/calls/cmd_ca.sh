# full-size parity after the core-plan changes, then the x3 / default bench lines
timeout 1200 python -m pytest tests/test_full_size_gpu.py -q -x > gpurun_out/r2ca_full.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2ca_bench.json 2> gpurun_out/r2ca_bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --mode tf32x3 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2ca_bench_x3.json 2> gpurun_out/r2ca_bench_x3.err
