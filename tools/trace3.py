import os, sys, json; sys.path.insert(0, '.')
import numpy as np, torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
S = 1200
os.makedirs('gpurun_out', exist_ok=True)
for mode, omega, cg, abl in json.loads(sys.argv[1]):
    s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
    s.set_ablation(abl)
    buf = torch.zeros(1280 * S, dtype=torch.int64, device='cuda')
    s.apply(A, out=B); torch.cuda.synchronize()
    s.set_trace(buf, S)
    s.apply(A, out=B); torch.cuda.synchronize()
    s.set_trace(None, 0)
    tr = buf.view(160, 8, S)[:8].cpu().numpy()
    np.savez(f'gpurun_out/trace3_{mode}_{omega}_cg{cg}_a{abl}.npz', tr=tr)
    print(mode, omega, cg, abl, "span us", (tr.max() - tr[tr > 0].min()) / 1e3, flush=True)
