# round-2 GPU check: full -m gpu suite, x3 A/B against the pre-promotion build, c4 single vs two passes
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1
tail -3 gpurun_out/r2c_tests.log
CFGS='[["tf32x3","accurate",0]]' ROUNDS=3 timeout 600 python tools/abmulti.py ab_old/pre_x3 new > gpurun_out/r2c_ab.txt 2>&1
for ncol in 2 1; do
SK_NCOL=$ncol SK_DEBUG_PLAN=1 timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2c_c4_ncol$ncol.json 2> gpurun_out/r2c_c4_ncol$ncol.err
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2c_c2.json 2> gpurun_out/r2c_c2.err
