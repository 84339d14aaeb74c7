# producer warp count A/B (compile-time SK_RNG_WARPS_BF16 = 8 / 10 / 12 / 14 / 16 in-tree)
CFGS='[["bf16","fast",0],["bf16","accurate",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/rw8 ab_old/rw10 ab_old/rw12 ab_old/rw14 new > gpurun_out/r2ag_c2.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=6250 timeout 900 python tools/abmulti.py ab_old/rw8 ab_old/rw10 ab_old/rw12 ab_old/rw14 new > gpurun_out/r2ag_share.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=1000000 R=512 timeout 900 python tools/abmulti.py ab_old/rw8 ab_old/rw10 ab_old/rw12 ab_old/rw14 new > gpurun_out/r2ag_c4.txt 2>&1
