# probe torch symmetric memory on this box: rendezvous, peer pointers, a P2P write, barrier
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
group = dist.group.WORLD
try:
    symm_mem.enable_symm_mem_for_group(group.group_name)
except Exception as e:
    print("enable:", repr(e))
t = symm_mem.empty((world, 1024), dtype=torch.float32, device="cuda")
t.zero_()
h = symm_mem.rendezvous(t, group.group_name)
print(rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "mc", hex(h.multicast_ptr) if h.multicast_ptr else None, flush=True)
peer = (rank + 1) % world
remote = h.get_buffer(peer, (world, 1024), torch.float32)
h.barrier()
remote[rank].fill_(rank + 1.0)
h.barrier()
torch.cuda.synchronize()
print(rank, "slot sums", [float(t[j].sum()) for j in range(world)], flush=True)
dist.destroy_process_group()
