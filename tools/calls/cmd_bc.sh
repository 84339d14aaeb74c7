SK_DEBUG_PLAN=1 python tools/prof_shape.py 2048 4000000 512 bf16 fast gaussian 4 > gpurun_out/r2bc.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size_gpu.py -q -p no:cacheprovider -k "wide_r or c4 or identity or c5_shape" > gpurun_out/r2bc_tests.log 2>&1
tail -2 gpurun_out/r2bc_tests.log
