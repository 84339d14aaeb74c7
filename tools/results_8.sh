#!/bin/bash
# c2 default at N = 8: BASELINE's 2D grid (auto: 4x2) and row-block
for lay in auto row; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 8 --layout $lay --no-other-modes --no-e2e > gpurun_out/res8_c2_${lay}.log 2>&1; echo "c2 n8 $lay rc=$?"
  tail -1 gpurun_out/res8_c2_${lay}.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), d['config']['layout'], round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks'], d['comm'])"
done
