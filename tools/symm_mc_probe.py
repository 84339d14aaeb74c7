"""Does torch symmetric memory give this box's GPUs a multicast (NVLS) mapping?  torchrun --nproc-per-node 2"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
buf = symm_mem.empty((1024,), dtype=torch.float32, device="cuda")
hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
print(f"rank {rank}: multicast_ptr={mc:#x}", flush=True)
if mc:
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2603_20966_b200 as sk
    buf.fill_(rank + 1.0)
    hdl.barrier(channel=0)
    out = torch.empty(1024, device="cuda")
    sk.multimem_sum(mc, 1024, out)
    torch.cuda.synchronize()
    print(f"rank {rank}: NVLS sum = {out[:4].tolist()} (expect {sum(range(1, dist.get_world_size() + 1))})", flush=True)
dist.destroy_process_group()
