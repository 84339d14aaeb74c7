# core block offsets against the queried workspace (new internal bound check)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "core" > gpurun_out/r2ck_core_tests.txt 2>&1
