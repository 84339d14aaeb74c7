# f4 Omega ablation with the final kernel: fused vs materialise + cuBLAS vs all-gather (1 and 2 GPUs), c2 and c4
timeout 900 python bench.py --omega-ablation --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity > gpurun_out/r2ao_c2_n1.json 2> gpurun_out/r2ao_c2_n1.err
timeout 900 python bench.py --gpus 2 --omega-ablation --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity > gpurun_out/r2ao_c2_n2.json 2> gpurun_out/r2ao_c2_n2.err
timeout 900 python bench.py --workload c4 --omega-ablation --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity > gpurun_out/r2ao_c4_n1.json 2> gpurun_out/r2ao_c4_n1.err
