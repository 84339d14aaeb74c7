#!/bin/bash
# full results sweep for BASELINE.md: default bench at N=1 (all modes in one line), c3, and multi-GPU
python bench.py > gpurun_out/res_c2_n1.log 2>&1; echo "c2 n1 rc=$?"
python bench.py --workload c3 --mode tf32 --no-other-modes > gpurun_out/res_c3_n1.log 2>&1; echo "c3 n1 rc=$?"
for N in 2 4; do
  for lay in row 2x1 2x2; do
    [ "$N" = "2" ] && [ "$lay" = "2x2" ] && continue
    [ "$N" = "4" ] && [ "$lay" = "2x1" ] && continue
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $N --layout $lay --no-other-modes > gpurun_out/res_c2_n${N}_${lay}.log 2>&1; echo "c2 n$N $lay rc=$?"
  done
done
