# sketch_sum_peers over NVLink peer mappings: the templated kernel (default) vs the scalar loop
# (SK_SUM_PEERS_V1); usage: torchrun --nproc-per-node N tools/sumpeers_bench.py
import os, sys; sys.path.insert(0, '.')
import torch, torch.distributed as tdist
import torch.distributed._symmetric_memory as symm_mem
import paper_2603_20966_b200 as sk
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
lr = int(os.environ.get("LOCAL_RANK", 0)); torch.cuda.set_device(lr); dev = torch.device("cuda", lr)
tdist.init_process_group("nccl", device_id=dev)
for mb in (0.25, 3.2, 12.8, 25.6):
    elems = int(mb * 1e6 / 4) // 4 * 4
    buf = symm_mem.empty((elems,), dtype=torch.float32, device=dev)
    hdl = symm_mem.rendezvous(buf, tdist.group.WORLD.group_name)
    buf.fill_(rank + 1.0); hdl.barrier(channel=0)
    out = torch.empty(elems, device=dev)
    ptrs = [int(p) for p in hdl.buffer_ptrs]
    res = {}
    for rnd in range(3):
        for v1 in (False, True):
            if v1: os.environ["SK_SUM_PEERS_V1"] = "1"
            else: os.environ.pop("SK_SUM_PEERS_V1", None)
            sk.sum_peers(ptrs, elems, out); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): sk.sum_peers(ptrs, elems, out)
            e1.record(); torch.cuda.synchronize()
            res.setdefault(v1, []).append(e0.elapsed_time(e1) / 20 * 1000)
    assert torch.all(out == world * (world + 1) / 2)
    hdl.barrier(channel=0)
    if rank == 0:
        t2, t1 = sorted(res[False])[1], sorted(res[True])[1]
        print(f"P={world} {mb:5.2f} MB per rank: templated {t2:.1f} us ({elems * 4 * (world - 1) / t2 / 1e3:.0f} GB/s remote), scalar {t1:.1f} us", flush=True)
    del hdl, buf
tdist.destroy_process_group()
