# core chunk reduce: 8-group float4 kernel (new) vs scalar loop (cr_old); then the parity / determinism tests touching C
timeout 600 python tools/core_ab.py ab_old/cr_old new > gpurun_out/r2bw_core.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_virtual_gpu.py -q -x > gpurun_out/r2bw_tests.txt 2>&1
