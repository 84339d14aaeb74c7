import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tf32"]
for mode in modes:
    for cg in (2, 4):
        for abl in (0, 1, 2, 3, 5, 6, 7):
            s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega="fast" if mode != "tf32x3" else "accurate", cta_group=cg)
            s.set_ablation(abl)
            for _ in range(2): s.apply(A, out=B)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): s.apply(A, out=B)
            e1.record(); torch.cuda.synchronize()
            print(f"{mode} cg{cg} ablate={abl}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
