# c2 knobs with the new producer count: spin-waiting producers (ablation bit 5), A prefetch into L2
CFGS='[["bf16","fast",0],["bf16","fast",32],["bf16","fast",0,{"SK_PREFETCH":2}],["bf16","fast",0,{"SK_PREFETCH":6}]]' ROUNDS=3 timeout 900 python tools/abmulti.py new > gpurun_out/r2al.txt 2>&1
