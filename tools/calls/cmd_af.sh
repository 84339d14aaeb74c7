# producer warp count A/B (compile-time SK_RNG_WARPS_BF16 = 12 / 16 (in-tree) / 20): c2, 8-GPU share, c4 shape
CFGS='[["bf16","fast",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/rw12 new ab_old/rw20 > gpurun_out/r2af_c2.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=6250 timeout 900 python tools/abmulti.py ab_old/rw12 new ab_old/rw20 > gpurun_out/r2af_share.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=1000000 R=512 timeout 900 python tools/abmulti.py ab_old/rw12 new ab_old/rw20 > gpurun_out/r2af_c4.txt 2>&1
