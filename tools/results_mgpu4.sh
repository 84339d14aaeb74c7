#!/bin/bash
# c2 default at N = 4 row-block (12500-row shares now on clusters of 3 pairs) and 2x2; c4 default at N = 1, 4
for lay in row auto; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --layout $lay --no-other-modes > gpurun_out/res4_c2_n4_${lay}.log 2>&1; echo "c2 n4 $lay rc=$?"
  tail -1 gpurun_out/res4_c2_n4_${lay}.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['value'],1), d['config']['layout'], round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks'], d.get('e2e',{}).get('value'))"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload c4 --no-other-modes > gpurun_out/res4_c4_n1.log 2>&1; echo "c4 n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --workload c4 --no-other-modes --no-e2e > gpurun_out/res4_c4_n4.log 2>&1; echo "c4 n4 rc=$?"
for f in res4_c4_n1 res4_c4_n4; do tail -1 gpurun_out/$f.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), round(d['value'],1), d['config']['layout'], d['config']['omega_transform'], round(d['roofline']['frac'],3), d['roofline']['bound'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks'], d.get('e2e',{}).get('value'))"; done
