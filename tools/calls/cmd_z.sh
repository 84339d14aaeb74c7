# 4-GPU box: full 1-GPU suite, dist tests (4 ranks), c2 at 1 / 2 / 4 GPUs back to back, c2 4-GPU 2x2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2z_tests.log 2>&1
tail -3 gpurun_out/r2z_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2z_c2_n1.json 2> gpurun_out/r2z_c2_n1.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2z_c2_n2.json 2> gpurun_out/r2z_c2_n2.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2z_c2_n4.json 2> gpurun_out/r2z_c2_n4.err
timeout 600 python bench.py --gpus 4 --layout 2x2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2z_c2_n4_2x2.json 2> gpurun_out/r2z_c2_n4_2x2.err
