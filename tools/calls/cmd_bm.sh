# c4 / c2 ablations: Omega generation off (1), share copies 1/8 (128), both (129), A loads off (2)
CFGS='[["bf16","fast",0],["bf16","fast",1],["bf16","fast",128],["bf16","fast",129],["bf16","fast",2]]' ROUNDS=3 N1=2048 N=2000000 R=512 timeout 900 python tools/abmulti.py new > gpurun_out/r2bm_c4.txt 2>&1
CFGS='[["bf16","fast",0],["bf16","fast",1],["bf16","fast",128],["bf16","fast",129],["bf16","fast",2]]' ROUNDS=3 timeout 900 python tools/abmulti.py new > gpurun_out/r2bm_c2.txt 2>&1
