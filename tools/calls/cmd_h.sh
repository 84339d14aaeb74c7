# 2-GPU box: dist tests (NVLS default), c2 row / col layouts with NVLS vs NVLink peer reads vs NCCL
python - > gpurun_out/r2h_mc.txt 2>&1 <<'PY'
import torch
print(torch.cuda.device_count())
PY
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2h_dist_tests.log 2>&1
tail -2 gpurun_out/r2h_dist_tests.log
for lay in 2x1 1x2; do
  for nv in 1 0; do
    SK_NVLS=$nv timeout 600 python bench.py --gpus 2 --layout $lay --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --no-parity > gpurun_out/r2h_c2_${lay}_nvls$nv.json 2> gpurun_out/r2h_c2_${lay}_nvls$nv.err
  done
  timeout 600 python bench.py --gpus 2 --layout $lay --nccl-ar --rs nccl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --no-parity > gpurun_out/r2h_c2_${lay}_nccl.json 2> gpurun_out/r2h_c2_${lay}_nccl.err
done
