# Redist with ragged column blocks of C (virtual ranks)
timeout 600 python -m pytest tests/test_virtual_fuzz_gpu.py -q -x -k ragged > gpurun_out/r2bv_ragged.txt 2>&1
