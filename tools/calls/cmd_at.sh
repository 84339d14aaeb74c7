timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k concurrent_inplace > gpurun_out/r2at_tests.log 2>&1
tail -3 gpurun_out/r2at_tests.log
