# core GEMM / reduce change: GPU suite; c2 at 1 and 4 GPUs (phase times)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2aq_tests.log 2>&1
tail -3 gpurun_out/r2aq_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2aq_c2_n1.json 2> gpurun_out/r2aq_c2_n1.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2aq_c2_n4.json 2> gpurun_out/r2aq_c2_n4.err
timeout 600 python bench.py --gpus 4 --layout row --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2aq_c2_n4_row.json 2> gpurun_out/r2aq_c2_n4_row.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2aq_c2_n2.json 2> gpurun_out/r2aq_c2_n2.err
