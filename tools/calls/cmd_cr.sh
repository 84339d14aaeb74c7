# c4 full size: HEAD vs the build of the c4 ncu summary (38cf9d3), same box
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=4000000 R=512 timeout 1200 python tools/abmulti.py ab_old/c4old new > gpurun_out/r2cr_c4.txt 2>&1
