timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ap_tests.log 2>&1
tail -3 gpurun_out/r2ap_tests.log
CFGS='[["tf32","fast",0],["tf32","accurate",0],["bf16","fast",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/rwt8 new > gpurun_out/r2ap_ab.txt 2>&1
