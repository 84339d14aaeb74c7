# CTA-grouping A/B at one shape (idle-start, interleaved): python tools/clab.py n1 n2 r mode omega cg1,cg2,...
import sys, time; sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as sk
n1, n2, r, mode, omega = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
cgs = [int(c) for c in sys.argv[6].split(",")]
A = torch.empty((n1, n2), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n1, r), device='cuda')
res = {c: [] for c in cgs}
for rnd in range(5):
    for c in cgs:
        s = sk.Sketch(42, 'gaussian', n2, r, mode=mode, omega=omega, cta_group=c)
        s.apply(A, out=B); torch.cuda.synchronize(); time.sleep(0.4)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize(); res[c].append(e0.elapsed_time(e1) / 3)
print(f"{n1}x{n2} r={r} {mode}/{omega}: " + "  ".join(f"cg{c}={sorted(v)[2]:.3f}" for c, v in res.items()), flush=True)
