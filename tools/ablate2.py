import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
for cg, abl in [(1, 5), (1, 7), (1, 0), (2, 5), (2, 21), (2, 7), (2, 0), (2, 16), (2, 1), (2, 2), (2, 3)]:
    s = sk.Sketch(42, 'gaussian', n, r, omega='fast', cta_group=cg)
    s.set_ablation(abl)
    for _ in range(2): s.apply(A, out=B)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): s.apply(A, out=B)
    e1.record(); torch.cuda.synchronize()
    print(f"cg{cg} ablate={abl}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
