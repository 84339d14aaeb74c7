#!/bin/bash
# multi-GPU c2 (row-block = zero B communication; 2x2 grid = Alg. 1 reduce-scatter) at N = 2, 4
for N in 2 4; do
  for lay in row 2x2; do
    [ "$N" = "2" ] && [ "$lay" = "2x2" ] && continue
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $N --layout $lay --no-other-modes > gpurun_out/res_c2_n${N}_${lay}.log 2>&1; echo "c2 n$N $lay rc=$?"
  done
done
