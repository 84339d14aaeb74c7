# A/B of several library builds in one process (interleaved, min over rounds).
# usage: CFGS='[["tf32","fast",0]]' python tools/abmulti.py ab_old/pkgA ab_old/pkgB ...   ("new" = in-tree package)
import importlib.util, os, sys, json; sys.path.insert(0, '.')
import torch
mods = []
for path in sys.argv[1:]:
    if path == "new":
        import paper_2603_20966_b200 as m
    else:
        name = "pkg_" + os.path.basename(path)
        spec = importlib.util.spec_from_file_location(name, path + "/__init__.py", submodule_search_locations=[path])
        m = importlib.util.module_from_spec(spec); sys.modules[name] = m; spec.loader.exec_module(m)
    mods.append((path, m))
import threading, time
try:
    import pynvml; pynvml.nvmlInit(); H = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM)
except Exception:
    clk = lambda: 1965
class Sampler:
    def __enter__(self):
        self.v, self.run = [], True
        def f():
            while self.run:
                self.v.append(clk()); time.sleep(0.002)
        self.t = threading.Thread(target=f, daemon=True); self.t.start(); return self
    def __exit__(self, *a):
        self.run = False; self.t.join()
n, r = int(os.environ.get("N", 50000)), int(os.environ.get("R", 256))
n1 = int(os.environ.get("N1", n))  # A is n1 x n (N1 / N / R env: any shape)
A = torch.empty((n1, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n1, r), device='cuda')
cfgs = json.loads(os.environ.get("CFGS", '[["tf32","fast",0],["tf32","fast",7],["bf16","accurate",0]]'))
res = {}
for rnd in range(int(os.environ.get("ROUNDS", 3))):
    for cfg in cfgs:
        m_, o, abl = cfg[:3]
        env = cfg[3] if len(cfg) > 3 else {}
        for k in {"SK_A_STAGES", "SK_Y_STAGES", "SK_O_STAGES", "SK_PREFETCH"} | {k for c in cfgs if len(c) > 3 for k in c[3]}:
            os.environ.pop(k, None)
        for k, v in env.items(): os.environ[k] = str(v)
        cg = int(env.get("CG", 0))
        for name, mod in mods:
            s = mod.Sketch(42, 'gaussian', n, r, mode=m_, omega=o, cta_group=cg)
            s.set_ablation(abl)
            s.apply(A, out=B); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            time.sleep(float(os.environ.get("IDLE", 0.4)))  # start every measurement from idle clocks
            s.apply(A, out=B)
            with Sampler() as sm:
                e0.record()
                for _ in range(int(os.environ.get("REPS", 5))): s.apply(A, out=B)
                e1.record(); torch.cuda.synchronize()
            c = sum(sm.v) / max(1, len(sm.v))
            res.setdefault((m_, o, abl, json.dumps(env), name), []).append((e0.elapsed_time(e1) / int(os.environ.get('REPS', 5)), c))
for cfg in cfgs:
    m_, o, abl = cfg[:3]
    env = cfg[3] if len(cfg) > 3 else {}
    def med(v): v = sorted(v); return v[len(v) // 2]
    print(f"{m_:7s} {o:8s} abl{abl:<3d} {json.dumps(env)} " + "  ".join(
        f"{os.path.basename(nm)}={med([t for t, _ in res[(m_, o, abl, json.dumps(env), nm)]]):.3f}/{med([t * c / 1965 for t, c in res[(m_, o, abl, json.dumps(env), nm)]]):.3f}"
        for nm, _ in mods) + "   (median ms / clock-normalised to 1965 MHz)", flush=True)
