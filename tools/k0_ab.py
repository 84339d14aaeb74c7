# sketch of one 25000 x 25000 block at Omega row offsets k0 = 0 / 25000 / 24960 (same A): does k0 change the time?
import os, sys; sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as sk
n = 25000
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
s = sk.Sketch(12345, "gaussian", 50000, 256, mode="bf16", omega="fast")
B = torch.empty((n, 256), device='cuda')
res = {}
for rnd in range(3):
    for k0 in (0, 25000, 24960, 24576, 1):
        s.apply_block(A, k0, out=B); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): s.apply_block(A, k0, out=B)
        e1.record(); torch.cuda.synchronize()
        res.setdefault(k0, []).append(e0.elapsed_time(e1) / 10)
for k0, v in res.items(): print(f"k0={k0:6d} {sorted(v)[1]*1000:.1f} us", s.plan_info(n, n) if k0 == 0 else "")
