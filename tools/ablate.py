"""Ablation timing of the sketch GEMM on c2-shaped A (device only)."""
import sys, time, json
sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
res = {}
for cg in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else '12')]:
    for omega in ('accurate', 'fast'):
        for abl in (0, 1, 2, 3, 4, 5, 6):
            s = sk.Sketch(42, 'gaussian', n, r, omega=omega, cta_group=cg)
            s.set_ablation(abl)
            for _ in range(2): s.apply(A, out=B)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): s.apply(A, out=B)
            e1.record(); torch.cuda.synchronize()
            res[f"cg{cg}_{omega}_abl{abl}"] = round(e0.elapsed_time(e1) / 5, 3)
            print(f"cg{cg} {omega} ablate={abl}: {res[f'cg{cg}_{omega}_abl{abl}']} ms", flush=True)
