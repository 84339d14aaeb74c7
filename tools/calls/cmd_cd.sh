# core plan wave model (nacc x rows per chunk) with a 128-offset workspace loop: defaults over row counts, suites
ROWS=3000,6250,9000,12500,18750,25000,37500,50000 timeout 900 python tools/core_sweep.py > gpurun_out/r2cd_core_sweep.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_virtual_gpu.py tests/test_virtual_fuzz_gpu.py tests/test_full_size_gpu.py -q -x > gpurun_out/r2cd_tests.txt 2>&1
