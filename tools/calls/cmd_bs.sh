# seeded random-configuration parity sweep, 160 cases
timeout 900 python -m pytest tests/test_fuzz_gpu.py -q -x > gpurun_out/r2bs_fuzz.txt 2>&1
