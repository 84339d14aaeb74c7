# L2-multicast Omega shares, producers writing the global mirror (bf16 Gaussian): bit-identity, c4 / c2 timing
timeout 300 python tools/oshare_check.py > gpurun_out/r2bo_check.txt 2>&1 || exit 1
CFGS='[["bf16","fast",0],["bf16","fast",0,{"SK_OSHARE_L2":"1"}]]' ROUNDS=3 N1=2048 N=2000000 R=512 timeout 600 python tools/abmulti.py new > gpurun_out/r2bo_c4.txt 2>&1
CFGS='[["bf16","fast",0],["bf16","fast",0,{"SK_OSHARE_L2":"1"}],["tf32","fast",0],["tf32","fast",0,{"SK_OSHARE_L2":"1"}]]' ROUNDS=3 timeout 600 python tools/abmulti.py new > gpurun_out/r2bo_c2.txt 2>&1
