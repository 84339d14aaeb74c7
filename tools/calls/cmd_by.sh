# core GEMM: 128-row C blocks (nacc = 1) for short B (new) vs 256-row blocks (core_old)
ROWS=3000,6250,9000,12500,50000 timeout 600 python tools/core_ab.py ab_old/core_old new > gpurun_out/r2by_core.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_virtual_gpu.py tests/test_virtual_fuzz_gpu.py -q -x > gpurun_out/r2by_tests.txt 2>&1
