# per-phase device timeline of the distributed step at 4 GPUs (2x2 and 4x1) and 2 GPUs (2x1, 1x2)
for spec in 2x2 4x1; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/dist_phases.py $spec >> gpurun_out/r2cg_phases.txt 2>&1; done
