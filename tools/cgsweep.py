import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
for mode, omega in [("bf16", "accurate"), ("bf16", "fast"), ("tf32", "accurate"), ("tf32", "fast"), ("tf32x3", "accurate")]:
    for cg, abl in ((2, 0), (2, 32), (4, 0), (4, 32), (8, 0)):
        s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
        s.set_ablation(abl)
        for _ in range(2): s.apply(A, out=B)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(6): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize()
        print(f"{mode:6s} {omega:8s} cg{cg} {'spin' if abl else 'sleep'}: {e0.elapsed_time(e1)/6:.3f} ms", flush=True)
