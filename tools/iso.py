import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_20966_b200 as sk, oracle
from inputs import synth
case = sys.argv[1]
if case.startswith('blk'):
    k0 = int(case[3:])
    A = synth.uniform(9, 300, 700)
    s = sk.Sketch(42, "gaussian", 2000, 40)
    B = s.apply_block(torch.from_numpy(A).cuda(), k0).cpu().numpy()
    ref = oracle.sketch(42, "gaussian", A, 40, k0=k0)
    print(case, np.linalg.norm(B-ref)/np.linalg.norm(ref))
elif case == 'core':
    Bm = synth.uniform(8, 500, 48)
    s = sk.Sketch(42, "gaussian", 1000, 48)
    C = s.core_block(torch.from_numpy(Bm).cuda(), 0).cpu().numpy()
    ref = oracle.core(42, "gaussian", Bm.astype(np.float64))
    print(case, np.linalg.norm(C-ref)/np.linalg.norm(ref))
elif case == 'nys':
    A = synth.symmetric_uniform(6, 512)
    s = sk.Sketch(42, "gaussian", 512, 16)
    B, C = s.nystrom_core(torch.from_numpy(A).cuda())
    print(case, float(C.abs().sum()))
