# producer warp count, second box, more rounds: c2 (the headline) and the c4 shape
CFGS='[["bf16","fast",0]]' ROUNDS=6 timeout 900 python tools/abmulti.py ab_old/rw8 ab_old/rw12 new > gpurun_out/r2ah_c2.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=4 N1=2048 N=1000000 R=512 timeout 900 python tools/abmulti.py ab_old/rw8 ab_old/rw12 ab_old/rw14 new > gpurun_out/r2ah_c4.txt 2>&1
