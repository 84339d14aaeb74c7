# seeded random sweep of the multi-GPU layouts through virtual ranks (one GPU), 96 cases
timeout 1200 python -m pytest tests/test_virtual_fuzz_gpu.py -q -x > gpurun_out/r2bu_vfuzz.txt 2>&1
