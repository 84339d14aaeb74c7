# 4-GPU box: c2 at 1/2/4 GPUs back to back (graphs on), layouts 2x2 (auto) and 4x1; dist tests (4 ranks)
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n1.json 2> gpurun_out/r2p_c2_n1.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n2.json 2> gpurun_out/r2p_c2_n2.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n4.json 2> gpurun_out/r2p_c2_n4.err
timeout 600 python bench.py --gpus 4 --layout row --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n4_row.json 2> gpurun_out/r2p_c2_n4_row.err
timeout 600 python bench.py --gpus 4 --graph off --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n4_eager.json 2> gpurun_out/r2p_c2_n4_eager.err
SK_NVLS=0 timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2p_c2_n4_peer.json 2> gpurun_out/r2p_c2_n4_peer.err
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2p_dist_tests.log 2>&1
