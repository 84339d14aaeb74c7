import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
cases = [(m, o, cg, abl) for (m, o) in [("tf32", "fast"), ("bf16", "fast"), ("tf32x3", "accurate")]
         for cg in (2, 4) for abl in (0, 1, 2, 3, 5, 7)]
for mode, omega, cg, abl in cases:
    s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
    s.set_ablation(abl)
    for _ in range(2): s.apply(A, out=B)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): s.apply(A, out=B)
    e1.record(); torch.cuda.synchronize()
    print(f"{mode:6s} {omega:8s} cg{cg} ablate={abl}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
