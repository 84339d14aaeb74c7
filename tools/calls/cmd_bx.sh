# ncu of the core GEMM at the 8-GPU share (6250 rows, r = 256, bf16 / fast)
timeout 300 python tools/core_one.py || exit 1
timeout 600 ncu --set full --clock-control none -k regex:core_gemm_tc -s 3 -c 1 -o gpurun_out/r2bx_core python tools/core_one.py > gpurun_out/r2bx_ncu.log 2>&1
