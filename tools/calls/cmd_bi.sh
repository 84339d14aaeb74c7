timeout 600 python -m pytest tests/test_curand_pin_gpu.py -q -p no:cacheprovider > gpurun_out/r2bi_tests.log 2>&1
tail -3 gpurun_out/r2bi_tests.log
