# sum_peers kernel A/B at 2 and 4 ranks, then bench 2x2 A/B (4 GPUs)
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29621 tools/sumpeers_bench.py >> gpurun_out/r2cn_sumpeers.txt 2>&1; done
for rep in 1 2; do
  timeout 900 python bench.py --gpus 4 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2cn_bench_n4_new$rep.json 2> /dev/null
  SK_SUM_PEERS_V1=1 timeout 900 python bench.py --gpus 4 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2cn_bench_n4_v1$rep.json 2> /dev/null
done
timeout 600 python -m pytest tests/test_dist_gpu.py -q -x > gpurun_out/r2cn_dist_tests.txt 2>&1
