# per-phase device times (sketch_set_profiling) for several library builds, interleaved
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
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
for m_, o in json.loads(os.environ.get("CFGS", '[["tf32","fast"],["tf32","accurate"]]')):
    for rnd in range(3):
        for name, mod in mods:
            s = mod.Sketch(42, 'gaussian', n, r, mode=m_, omega=o)
            s.apply(A, out=B); torch.cuda.synchronize()
            s.set_profiling(True)
            for _ in range(5): s.apply(A, out=B)
            torch.cuda.synchronize()
            ph = s.profile_read()
            s.set_profiling(False)
            print(m_, o, os.path.basename(name), {k: (round(v[0] / max(1, v[1]), 3), v[1]) for k, v in ph.items() if v[1]}, "ws", s.workspace_size(n), flush=True)
