# Old-vs-new library A/B in one process (interleaved, min over rounds): ab_old/pkg_old = a previous build
import importlib.util, os, sys, json; sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as new
spec = importlib.util.spec_from_file_location("pkg_old", "ab_old/pkg_old/__init__.py", submodule_search_locations=["ab_old/pkg_old"])
old = importlib.util.module_from_spec(spec); sys.modules["pkg_old"] = old; spec.loader.exec_module(old)
try:
    import pynvml; pynvml.nvmlInit(); H = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM)
except Exception:
    clk = lambda: -1
n, r = int(os.environ.get("N", 50000)), 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
cfgs = json.loads(os.environ.get("CFGS", '[["bf16","accurate",0],["bf16","fast",0],["tf32","accurate",0],["tf32","fast",0],["tf32x3","accurate",0]]'))
res = {}
for rnd in range(3):
    for m, o, abl in cfgs:
        for name, mod in (("old", old), ("new", new)):
            s = mod.Sketch(42, 'gaussian', n, r, mode=m, omega=o)
            s.set_ablation(abl)
            s.apply(A, out=B); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(6): s.apply(A, out=B)
            e1.record(); c = clk(); torch.cuda.synchronize()
            res.setdefault((m, o, abl, name), []).append((e0.elapsed_time(e1) / 6, c))
for m, o, abl in cfgs:
    a = min(res[(m, o, abl, "old")]); b = min(res[(m, o, abl, "new")])
    print(f"{m:7s} {o:8s} abl{abl} old {a[0]:.3f} new {b[0]:.3f} ms  ratio {a[0]/b[0]:.3f}  clk old {[c for _, c in res[(m,o,abl,'old')]]} new {[c for _, c in res[(m,o,abl,'new')]]}", flush=True)
