# 4-GPU box: multicast probe, dist tests (2 and 4 ranks), c2 at 4 GPUs (2x2 auto, row, redist), c3 / c4
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/symm_mc_probe.py > gpurun_out/r2i_mc.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2i_dist_tests.log 2>&1
for cfg in "c2 auto noredist" "c2 row noredist" "c2 row redist" "c3 auto noredist" "c4 auto noredist"; do
  set -- $cfg
  timeout 600 python bench.py --gpus 4 --workload $1 --layout $2 --variant $3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2i_$1_$2_$3.json 2> gpurun_out/r2i_$1_$2_$3.err
done
