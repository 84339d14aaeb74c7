timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ay_tests.log 2>&1
tail -3 gpurun_out/r2ay_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ay_bench.json 2> gpurun_out/r2ay_bench.err
