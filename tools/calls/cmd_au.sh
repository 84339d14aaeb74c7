# bf16 tile writer with two independent items per iteration (ILP2) vs in-tree
CFGS='[["bf16","fast",0],["bf16","accurate",0]]' ROUNDS=4 timeout 900 python tools/abmulti.py ab_old/ilp2 new > gpurun_out/r2au_c2.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=1000000 R=512 timeout 900 python tools/abmulti.py ab_old/ilp2 new > gpurun_out/r2au_c4.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=6250 timeout 900 python tools/abmulti.py ab_old/ilp2 new > gpurun_out/r2au_share.txt 2>&1
