CFGS='[["bf16","fast",0],["bf16","accurate",0],["bf16","fast",0,{"CG":8}]]' ROUNDS=5 timeout 900 python tools/abmulti.py ab_old/cur new 2>&1 | tail -3
N=25000 CFGS='[["bf16","fast",0]]' ROUNDS=5 timeout 900 python tools/abmulti.py ab_old/cur new 2>&1 | tail -1
