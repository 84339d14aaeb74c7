# same-box A/B: round-1 build vs current, c2 bf16 fast / accurate and tf32 (interleaved, idle-clock starts)
CFGS='[["bf16","fast",0],["bf16","accurate",0],["tf32","accurate",0]]' ROUNDS=4 timeout 900 python tools/abmulti.py ab_old/r1 new > gpurun_out/r2r_ab.txt 2>&1
