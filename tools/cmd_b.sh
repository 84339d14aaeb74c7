set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2b_tests.log 2>&1
tail -3 gpurun_out/r2b_tests.log
CFGS='[["tf32x3","accurate",0],["bf16","fast",0]]' ROUNDS=3 timeout 600 python tools/abmulti.py ab_old/pre_x3 new > gpurun_out/r2b_ab.txt 2>&1
SK_DEBUG_PLAN=1 timeout 300 python bench.py --mode tf32x3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2b_bench_x3.json 2> gpurun_out/r2b_bench_x3.err
