# idle-start interleaved timing of ablation masks on one shape: python tools/shapeab.py n1 n2 r mode omega abl1,abl2,...
import os, sys, time; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n1, n2, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mode, omega = sys.argv[4], sys.argv[5]
abls = [int(x) for x in sys.argv[6].split(",")]
cgs = [int(x) for x in sys.argv[7].split(",")] if len(sys.argv) > 7 else [0]
A = torch.empty((n1, n2), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n1, r), device='cuda')
res = {(a, c): [] for a in abls for c in cgs}
for rnd in range(3):
    for a, cg in res:
        s = sk.Sketch(42, 'gaussian', n2, r, mode=mode, omega=omega, cta_group=cg)
        s.set_ablation(a)
        s.apply(A, out=B); torch.cuda.synchronize(); time.sleep(0.4)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize(); res[(a, cg)].append(e0.elapsed_time(e1) / 3)
for (a, cg), v in res.items():
    v = sorted(v); print(f"{n1}x{n2} r={r} {mode}/{omega} abl={a} cg={cg}: median {v[1]:.3f} ms (min {v[0]:.3f})", flush=True)
