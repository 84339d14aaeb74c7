# core GEMM plan sweep: blocks of C (nacc 2 / 1) x rows per chunk, bf16 r = 256
timeout 900 python tools/core_sweep.py > gpurun_out/r2cc_core_sweep.txt 2>&1
