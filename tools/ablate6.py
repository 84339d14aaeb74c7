import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
cfgs = [("bf16", "accurate", 4), ("bf16", "fast", 4), ("bf16", "accurate", 2), ("tf32", "fast", 4), ("tf32", "accurate", 4), ("tf32", "fast", 2)]
names = {0: "full", 1: "no-RNG", 2: "no-A", 3: "MMA+sync only", 5: "A-only", 6: "RNG-only", 7: "sync only", 64: "no-convert", 71: "sync no-conv"}
for mode, omega, cg in cfgs:
    for abl in ((0, 1, 6, 7, 64, 71) if cg == 4 else (0,)):
        s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
        s.set_ablation(abl)
        for _ in range(2): s.apply(A, out=B)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(6): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize()
        print(f"{mode} {omega} cg{cg} {names[abl]:14s}: {e0.elapsed_time(e1)/6:.3f} ms", flush=True)
