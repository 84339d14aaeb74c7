timeout 1200 python -m pytest tests/test_virtual_gpu.py -q -p no:cacheprovider > gpurun_out/r2ar_tests.log 2>&1
tail -3 gpurun_out/r2ar_tests.log
