free -g > gpurun_out/r2ak_mem.txt; nproc >> gpurun_out/r2ak_mem.txt
timeout 1200 python -m pytest tests/test_full_size_gpu.py -q -p no:cacheprovider > gpurun_out/r2ak_tests.log 2>&1
tail -3 gpurun_out/r2ak_tests.log
