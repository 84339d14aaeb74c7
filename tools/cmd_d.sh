# GPU check: full -m gpu suite; x3 A/B (REDG drain vs pre-promotion build); c4 with 8-CTA clusters
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1
tail -3 gpurun_out/r2d_tests.log
CFGS='[["tf32x3","accurate",0]]' ROUNDS=3 timeout 600 python tools/abmulti.py ab_old/pre_x3 new > gpurun_out/r2d_ab.txt 2>&1
SK_NCOL_CL=4 SK_DEBUG_PLAN=1 timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2d_c4_cl4.json 2> gpurun_out/r2d_c4_cl4.err
timeout 300 python bench.py --mode tf32x3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2d_c2_x3.json 2> gpurun_out/r2d_c2_x3.err
