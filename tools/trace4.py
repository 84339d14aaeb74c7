# pipeline trace with a trace-enabled build (ab_old/trace): python tools/trace4.py '[[mode, omega, cg, abl, n1, n2, r], ...]'
import importlib.util, os, sys, json; sys.path.insert(0, '.')
import numpy as np, torch
spec = importlib.util.spec_from_file_location("pkg_trace", "ab_old/trace/__init__.py", submodule_search_locations=["ab_old/trace"])
sk = importlib.util.module_from_spec(spec); sys.modules["pkg_trace"] = sk; spec.loader.exec_module(sk)
S = 1500
os.makedirs('gpurun_out', exist_ok=True)
for mode, omega, cg, abl, n1, n2, r in json.loads(sys.argv[1]):
    A = torch.empty((n1, n2), device='cuda').uniform_(-0.5, 0.5)
    B = torch.empty((n1, r), device='cuda')
    s = sk.Sketch(42, 'gaussian', n2, r, mode=mode, omega=omega, cta_group=cg)
    s.set_ablation(abl)
    buf = torch.zeros(1280 * S, dtype=torch.int64, device='cuda')
    s.apply(A, out=B); torch.cuda.synchronize()
    s.set_trace(buf, S)
    s.apply(A, out=B); torch.cuda.synchronize()
    s.set_trace(None, 0)
    tr = buf.view(160, 8, S)[:16].cpu().numpy()
    tag = f"{mode}_{omega}_cg{cg}_a{abl}_{n1}x{n2}_r{r}"
    np.savez(f'gpurun_out/trace4_{tag}.npz', tr=tr)
    print(tag, "span us", (tr.max() - tr[tr > 0].min()) / 1e3, flush=True)
    del A, B
