# 2-GPU box: NCCL / symmetric-memory tests, bench --gpus 2 (self-launching torchrun) per workload / variant
nvidia-smi topo -m > gpurun_out/r2g_topo.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2g_dist_tests.log 2>&1
tail -2 gpurun_out/r2g_dist_tests.log
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_c2_n2.json 2> gpurun_out/r2g_c2_n2.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --layout 1x2 > gpurun_out/r2g_c2_n2_col.json 2> gpurun_out/r2g_c2_n2_col.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --variant redist > gpurun_out/r2g_c2_n2_redist.json 2> gpurun_out/r2g_c2_n2_redist.err
timeout 600 python bench.py --gpus 2 --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2g_c4_n2.json 2> gpurun_out/r2g_c4_n2.err
timeout 600 python bench.py --gpus 2 --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2g_c3_n2.json 2> gpurun_out/r2g_c3_n2.err
