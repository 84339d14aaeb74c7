# 4-GPU box: c5 (n = 200,000, r = 1024: 40 GB of A per rank), the new virtual epilogue-RS x3 test
timeout 900 python bench.py --gpus 4 --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2v_c5_n4.json 2> gpurun_out/r2v_c5_n4.err
timeout 600 python -m pytest tests/test_virtual_gpu.py -q -p no:cacheprovider -k "epilogue_rs_tf32x3 or overlapped" > gpurun_out/r2v_tests.log 2>&1
