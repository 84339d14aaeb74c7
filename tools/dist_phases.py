# Per-phase device timeline of one distributed Nystrom step (eager), for the comm / sync overhead.
# usage: torchrun --nproc-per-node N tools/dist_phases.py [LAYOUT]   (c2: n = 50,000, r = 256, bf16 / fast)
import os, sys; sys.path.insert(0, '.')
import torch, torch.distributed as tdist
import paper_2603_20966_b200 as sk
from paper_2603_20966_b200.dist import DistSketch, Layout, SymmBuf
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
lr = int(os.environ.get("LOCAL_RANK", 0)); torch.cuda.set_device(lr); dev = torch.device("cuda", lr)
tdist.init_process_group("nccl", device_id=dev)
spec = sys.argv[1] if len(sys.argv) > 1 else "2x2"
n, r = 50000, 256
local = sk.Sketch(12345, "gaussian", n, r, mode="bf16", omega="fast")
ds = DistSketch(12345, "gaussian", n, n, r, Layout.parse(spec, world), local=local, fused_rs="peer", fused_ar=True)
r0, r1, c0, c1 = ds.a_block_range()
A = torch.empty((r1 - r0, c1 - c0), device=dev).uniform_(-0.5, 0.5)
ev = []
def wrap(obj, name, label):
    f = getattr(obj, name)
    def g(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True); e0.record()
        out = f(*a, **k)
        e1 = torch.cuda.Event(enable_timing=True); e1.record()
        ev.append((label, e0, e1)); return out
    setattr(obj, name, g)
wrap(ds.local, "apply_block", "sketch"); wrap(ds.local, "core_block", "core"); wrap(ds, "_reduce", "reduce")
orig_barrier = SymmBuf.barrier
def bar(self):
    e0 = torch.cuda.Event(enable_timing=True); e0.record(); orig_barrier(self)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(); ev.append(("barrier", e0, e1))
SymmBuf.barrier = bar
for _ in range(5): ds.nystrom_core(A)
torch.cuda.synchronize(); tdist.barrier()
acc = {}
for it in range(20):
    ev.clear()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record(); ds.nystrom_core(A); s1.record(); torch.cuda.synchronize()
    prev = s0
    for i, (lab, e0, e1) in enumerate(ev):
        key = f"{i}:{lab}"
        acc.setdefault(key, []).append((prev.elapsed_time(e0) * 1000, e0.elapsed_time(e1) * 1000))
        prev = e1
    acc.setdefault("total", []).append((0, s0.elapsed_time(s1) * 1000))
    tdist.barrier()
med = lambda v: sorted(v)[len(v) // 2]
line = " | ".join(f"{k}: gap {med([g for g, _ in v]):.1f} dur {med([d for _, d in v]):.1f}" for k, v in acc.items())
print(f"[rank {rank} {spec}] us: {line}", flush=True)
tdist.destroy_process_group()
