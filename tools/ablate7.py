# sync-skeleton study of the cluster path (c2 shape): ring depths x wait flavour
import os, sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
def run(mode, omega, cg, abl, a=None, o=None):
    for k, v in (("SK_A_STAGES", a), ("SK_O_STAGES", o)):
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = str(v)
    s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
    s.set_ablation(abl)
    for _ in range(2): s.apply(A, out=B)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(6): s.apply(A, out=B)
    e1.record(); torch.cuda.synchronize()
    print(f"{mode} {omega} cg{cg} abl={abl:3d} A{a} O{o}: {e0.elapsed_time(e1)/6:.3f} ms", flush=True)
for abl in (7, 39, 0, 32):
    run("bf16", "accurate", 4, abl)
for a, o in ((2, 4), (1, 8), (2, 2), (3, 2)):
    run("bf16", "accurate", 4, 7, a, o)
    run("bf16", "accurate", 4, 0, a, o)
for a, o in ((2, 4), (1, 8), (3, 2)):
    run("bf16", "accurate", 2, 7, a, o)
    run("bf16", "accurate", 2, 0, a, o)
