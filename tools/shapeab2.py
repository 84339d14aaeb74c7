# shape x library-build A/B (idle-start, interleaved): python tools/shapeab2.py n1 n2 r mode omega pkgA,pkgB,...
import importlib.util, os, sys, time; sys.path.insert(0, '.')
import torch
n1, n2, r, mode, omega = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
mods = []
for path in sys.argv[6].split(","):
    if path == "new":
        import paper_2603_20966_b200 as m
    else:
        name = "pkg_" + os.path.basename(path)
        spec = importlib.util.spec_from_file_location(name, path + "/__init__.py", submodule_search_locations=[path])
        m = importlib.util.module_from_spec(spec); sys.modules[name] = m; spec.loader.exec_module(m)
    mods.append((path, m))
A = torch.empty((n1, n2), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n1, r), device='cuda')
res = {p: [] for p, _ in mods}
for rnd in range(3):
    for p, m in mods:
        s = m.Sketch(42, 'gaussian', n2, r, mode=mode, omega=omega)
        s.apply(A, out=B); torch.cuda.synchronize(); time.sleep(0.4)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): s.apply(A, out=B)
        e1.record(); torch.cuda.synchronize(); res[p].append(e0.elapsed_time(e1) / 3)
print(f"{n1}x{n2} r={r} {mode}/{omega}: " + "  ".join(f"{os.path.basename(p)}={sorted(v)[1]:.3f}" for p, v in res.items()), flush=True)
