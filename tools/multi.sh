#!/bin/bash
# multi-GPU bench runs: tools/multi.sh N [layouts...]
N=$1; shift
for lay in "$@"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $N --steps 20 --warmup 3 --layout $lay --mode ${MODE:-tf32} --omega ${OMEGA:-fast} > gpurun_out/multi_${N}_${lay}.log 2>&1
  echo "N=$N layout=$lay rc=$?"
  tail -1 gpurun_out/multi_${N}_${lay}.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'host', round(d['host_submit_ms_per_step'],3), round(d['value'],1), d['comm'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d.get('e2e',{}).get('value'))
except Exception as e: print('no json', e)"
done
