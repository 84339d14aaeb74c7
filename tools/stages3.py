# bf16 ring-depth sweep at c2 (A ring / Y ring / Omega ring), cluster and pair paths
import os, sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
def run(omega, cg, a=None, y=None, o=None, abl=0):
    for k, v in (("SK_A_STAGES", a), ("SK_Y_STAGES", y), ("SK_O_STAGES", o)):
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = str(v)
    s = sk.Sketch(42, 'gaussian', n, r, mode="bf16", omega=omega, cta_group=cg)
    s.set_ablation(abl)
    for _ in range(2): s.apply(A, out=B)
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 5)
    print(f"bf16 {omega} cg{cg} A{a} Y{y} O{o} abl{abl}: {min(ts):.3f} ms", flush=True)
for omega in ("accurate",):
    run(omega, 4)
    for a, y, o in ((3, 2, 4), (3, 3, 2), (2, 3, 4), (2, 4, 2), (4, 3, 0), (2, 2, 6)):
        run(omega, 4, a, y, o)
run("accurate", 2)
run("accurate", 2, 2, 2, 6)
run("accurate", 8)
run("accurate", 4, abl=1)
run("accurate", 4, abl=65)
