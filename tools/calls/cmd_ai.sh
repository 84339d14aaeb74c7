# after the producer-warp change: GPU suite, default bench; tf32 producer warps 8 / 12 / 16 A/B
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ai_tests.log 2>&1
tail -3 gpurun_out/r2ai_tests.log
timeout 600 python bench.py > gpurun_out/r2ai_bench.json 2> gpurun_out/r2ai_bench.err
CFGS='[["tf32","accurate",0],["tf32","fast",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/rwt8 ab_old/rwt12 new > gpurun_out/r2ai_tf32.txt 2>&1
CFGS='[["tf32","accurate",0]]' ROUNDS=3 N1=4000000 N=2048 R=128 timeout 900 python tools/abmulti.py ab_old/rwt8 ab_old/rwt12 new > gpurun_out/r2ai_tf32_c3.txt 2>&1
