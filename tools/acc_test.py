"""relF of B vs the fp64 oracle as a function of the K accumulated per TMEM accumulator (split-K)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2603_20966_b200 as sk, oracle
from inputs import synth
K = 50000
A = synth.uniform(13, 296, K)
Ad = torch.from_numpy(A).cuda()
ref = oracle.sketch(42, "gaussian", A, 64)
Ai = synth.int_matrix(5, 296, K, -4, 4)
for mode in ("tf32x3", "tf32"):
    for split in (1, 2, 4, 8, 16, 32, 64):
        s = sk.Sketch(42, "gaussian", K, 64, mode=mode, split_k=split)
        B = s.apply(Ad).double().cpu().numpy()
        err = np.linalg.norm(B - ref) / np.linalg.norm(ref)
        bias = np.mean((B - ref) * np.sign(ref)) / np.mean(np.abs(ref))
        print(f"{mode:7s} split={split:3d} K/acc={K // split:6d} relF={err:.3e} signed-bias={bias:+.3e}", flush=True)
