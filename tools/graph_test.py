import os, sys, torch, torch.distributed as dist
sys.path.insert(0, '.')
import paper_2603_20966_b200 as sk
from paper_2603_20966_b200.dist import DistSketch, Layout
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); lr = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(lr); dev = torch.device("cuda", lr)
dist.init_process_group("nccl", device_id=dev)
n, r = 50000, 256
for lay in ("row", "2x2"):
    layout = Layout.parse(lay, world)
    local = sk.Sketch(42, "gaussian", n, r, mode="tf32", omega="fast")
    ds = DistSketch(42, "gaussian", n, n, r, layout, local=local)
    r0, r1, c0, c1 = ds.a_block_range()
    A = torch.empty((r1 - r0, c1 - c0), device=dev).uniform_(-0.5, 0.5)
    for _ in range(3): ds.nystrom_core(A)
    torch.cuda.synchronize(); dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ds.nystrom_core(A)
    e1.record(); torch.cuda.synchronize()
    t_eager = e0.elapsed_time(e1) / 20
    # graph capture of one step
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2): out = ds.nystrom_core(A)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = ds.nystrom_core(A)
    for _ in range(3): g.replay()
    torch.cuda.synchronize(); dist.barrier()
    e0.record()
    for _ in range(20): g.replay()
    e1.record(); torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 20
    if rank == 0: print(f"world={world} layout={lay}: eager {t_eager:.3f} ms, graph {t_graph:.3f} ms", flush=True)
dist.destroy_process_group()
