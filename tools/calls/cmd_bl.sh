# c4 (two column blocks) producer warps 10 / 12 (in-tree) / 14 / 16 with the current ring plan
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=2000000 R=512 timeout 900 python tools/abmulti.py ab_old/c4w10 new ab_old/c4w14 ab_old/c4w16 > gpurun_out/r2bl.txt 2>&1
