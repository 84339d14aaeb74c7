#!/bin/bash
# multi-GPU with the BASELINE layouts (bench --layout auto): c2 2D grid at N = 2, 4; c4 column-block
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $N --no-other-modes > gpurun_out/res2_c2_n${N}.log 2>&1; echo "c2 n$N rc=$?"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $N --workload c4 --no-other-modes --no-e2e > gpurun_out/res2_c4_n${N}.log 2>&1; echo "c4 n$N rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --workload c3 --mode tf32 --no-other-modes --no-e2e > gpurun_out/res2_c3_n4.log 2>&1; echo "c3 n4 rc=$?"
