timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "box_muller_fast_sweeps" > gpurun_out/r2bk.log 2>&1
grep -E "fast Box-Muller|passed|failed" gpurun_out/r2bk.log
