import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2603_20966_b200 as sk, oracle
r, m = 32, 64
for name, Bm in [("ones", np.ones((m, r), np.float32)), ("e0", np.eye(m, r, dtype=np.float32))]:
    for core in ("simt", "auto"):
        s = sk.Sketch(42, "rademacher", 1000, r, core=core)
        C = s.core_block(torch.from_numpy(Bm).cuda(), 0).cpu().numpy()
        ref = oracle.core(42, "rademacher", Bm.astype(np.float64))
        print(name, core, "max|C|", np.abs(C).max(), "err", np.abs(C - ref).max(), "C[0,:4]", C[0, :4], "ref", ref[0, :4])
