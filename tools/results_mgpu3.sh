#!/bin/bash
# c2 default (bf16, transform auto = fast) at N = 2, 4: BASELINE's 2D grid (auto) and row-block
for N in 2 4; do
  for lay in auto row; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $N --layout $lay --no-other-modes > gpurun_out/res3_c2_n${N}_${lay}.log 2>&1; echo "c2 n$N $lay rc=$?"
    tail -1 gpurun_out/res3_c2_n${N}_${lay}.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), d['config']['layout'], round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks'], d.get('e2e',{}).get('value'))"
  done
done
