# c2 bf16 producer warps 6 / 7 vs 8 (in-tree)
CFGS='[["bf16","fast",0],["bf16","accurate",0]]' ROUNDS=4 timeout 900 python tools/abmulti.py ab_old/rw6 ab_old/rw7 new > gpurun_out/r2cj_c2.txt 2>&1
