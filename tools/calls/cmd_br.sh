# seeded random-configuration parity sweep (64 cases)
timeout 900 python -m pytest tests/test_fuzz_gpu.py -q -x > gpurun_out/r2br_fuzz.txt 2>&1
