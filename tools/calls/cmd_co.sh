# 4 GPUs (2x2 and 4x1): AllReduce of C by NCCL vs fused symmetric-memory sum; reduce-scatter NCCL vs peer
B="timeout 900 python bench.py --gpus 4 --no-e2e --no-cpu-baseline --no-other-modes"
for rep in 1 2; do
  $B > gpurun_out/r2co_2x2_default$rep.json 2>/dev/null
  $B --nccl-ar > gpurun_out/r2co_2x2_ncclar$rep.json 2>/dev/null
  $B --rs nccl > gpurun_out/r2co_2x2_ncclrs$rep.json 2>/dev/null
  $B --rs nccl --nccl-ar > gpurun_out/r2co_2x2_ncclboth$rep.json 2>/dev/null
  $B --layout row > gpurun_out/r2co_4x1_default$rep.json 2>/dev/null
  $B --layout row --nccl-ar > gpurun_out/r2co_4x1_ncclar$rep.json 2>/dev/null
done
