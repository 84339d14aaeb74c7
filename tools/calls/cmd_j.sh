# 2-GPU box: multicast probe, dist tests, c2 layouts with NVLS vs NVLink peer reads
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/symm_mc_probe.py > gpurun_out/r2j_mc.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2j_dist_tests.log 2>&1
for lay in 2x1 1x2; do
  for nv in 1 0; do
    SK_NVLS=$nv timeout 600 python bench.py --gpus 2 --layout $lay --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --no-parity > gpurun_out/r2j_c2_${lay}_nvls$nv.json 2> gpurun_out/r2j_c2_${lay}_nvls$nv.err
  done
done
