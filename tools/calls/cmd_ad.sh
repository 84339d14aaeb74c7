# 4-GPU box: balanced row-block -- virtual + dist tests, c2 at 1 / 2 / 4 GPUs (balanced vs plain row split)
timeout 900 python -m pytest tests/test_virtual_gpu.py tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2ad_tests.log 2>&1
tail -3 gpurun_out/r2ad_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2ad_c2_n1.json 2> gpurun_out/r2ad_c2_n1.err
for n in 2 4; do
  timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2ad_c2_n$n.json 2> gpurun_out/r2ad_c2_n$n.err
  timeout 600 python bench.py --gpus $n --no-balance --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2ad_c2_n${n}_plain.json 2> gpurun_out/r2ad_c2_n${n}_plain.err
done
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --no-other-modes > gpurun_out/r2ad_c2_n4_e2e.json 2> gpurun_out/r2ad_c2_n4_e2e.err
