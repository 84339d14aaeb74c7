run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --workload c4 --omega accurate --no-other-modes --no-e2e --no-cpu-baseline --no-parity "$@" 2>&1 | tail -1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['comm'].get('reduce_scatter'))"; }
R=$PWD
echo pre; (cd ab_old/pre_r1d && run)
echo new; run
echo new-nccl; run --rs nccl
echo pre; (cd ab_old/pre_r1d && run)
