# bf16 converter loop: unroll 8 (un8), 2 warps x unroll 8 (cv2) vs in-tree (4 warps x unroll 4)
CFGS='[["bf16","fast",0],["bf16","accurate",0]]' ROUNDS=3 timeout 900 python tools/abmulti.py ab_old/un8 ab_old/cv2 new > gpurun_out/r2bq_c2.txt 2>&1
CFGS='[["bf16","fast",0]]' ROUNDS=3 N1=2048 N=2000000 R=512 timeout 900 python tools/abmulti.py ab_old/un8 ab_old/cv2 new > gpurun_out/r2bq_c4.txt 2>&1
