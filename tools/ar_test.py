import os, torch, torch.distributed as dist, time
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); lr = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(lr); dev = torch.device("cuda", lr)
dist.init_process_group("nccl", device_id=dev)
for nbytes in (256 * 1024, 4 << 20, 26 << 20):
    x = torch.ones(nbytes // 4, device=dev)
    for _ in range(10): dist.all_reduce(x)
    torch.cuda.synchronize(); dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): dist.all_reduce(x)
    e1.record(); torch.cuda.synchronize()
    ar = e0.elapsed_time(e1) / 50
    y = torch.empty(nbytes // 4 // world, device=dev)
    for _ in range(10): dist.reduce_scatter_tensor(y, x)
    torch.cuda.synchronize(); dist.barrier()
    e0.record()
    for _ in range(50): dist.reduce_scatter_tensor(y, x)
    e1.record(); torch.cuda.synchronize()
    rs = e0.elapsed_time(e1) / 50
    if rank == 0: print(f"world={world} bytes={nbytes}: allreduce {ar*1e3:.1f} us, reduce_scatter {rs*1e3:.1f} us", flush=True)
dist.destroy_process_group()
