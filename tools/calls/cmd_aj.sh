# converter warps 2 / 4 / 8 (bf16 and tf32x3 A transform); cluster size with the new producer count
CFGS='[["bf16","fast",0],["bf16","accurate",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/cvt2 ab_old/cvt8 new > gpurun_out/r2aj_cvt.txt 2>&1
CFGS='[["bf16","fast",0],["bf16","fast",0,{"CG":8}],["bf16","fast",0,{"CG":4}],["bf16","accurate",0],["bf16","accurate",0,{"CG":6}]]' ROUNDS=3 timeout 900 python tools/abmulti.py new > gpurun_out/r2aj_cl.txt 2>&1
