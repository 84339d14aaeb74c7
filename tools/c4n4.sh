for om in fast accurate fast; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --workload c4 --omega $om --no-other-modes --no-e2e --no-cpu-baseline --no-parity > gpurun_out/c4n4_$om.log 2>&1; echo "c4 n4 $om rc=$?"
tail -1 gpurun_out/c4n4_$om.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['config']['omega_transform'], {k: round(v,3) for k,v in d['phases_ms_per_step'].items()}, d['clocks'], d.get('per_rank_ms'))"
done
