# same-box A/B: round-1 build, current with the round-1 fast transform, current (c2)
CFGS='[["bf16","fast",0],["bf16","accurate",0],["tf32","accurate",0]]' ROUNDS=4 timeout 900 python tools/abmulti.py ab_old/r1 ab_old/oldfast new > gpurun_out/r2s_ab.txt 2>&1
