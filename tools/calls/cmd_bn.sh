# c4 ablations, part 2: converters off (64), MMAs off (4), no A + no converters (66), + no Omega gen (67), + small copies (195)
CFGS='[["bf16","fast",0],["bf16","fast",64],["bf16","fast",4],["bf16","fast",66],["bf16","fast",67],["bf16","fast",195]]' ROUNDS=3 N1=2048 N=2000000 R=512 timeout 900 python tools/abmulti.py new > gpurun_out/r2bn_c4.txt 2>&1
