# virtual + dist tests x3 (flakiness check after removing the overlapped core)
for i in 1 2 3; do timeout 900 python -m pytest tests/test_virtual_gpu.py tests/test_dist_gpu.py -q -p no:cacheprovider 2>&1 | tail -1; done > gpurun_out/r2aw_tests.log 2>&1
