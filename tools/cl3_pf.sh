CFGS='[["bf16","fast",0],["bf16","fast",0,{"SK_PREFETCH":2}],["bf16","fast",0,{"SK_PREFETCH":4}],["bf16","fast",0,{"SK_PREFETCH":8}]]' ROUNDS=5 timeout 900 python tools/abmulti.py new 2>&1 | tail -4
