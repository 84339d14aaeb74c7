# A/B of the core C = Omega^T B (core GEMM + fixed-order chunk reduce) across library builds.
# usage: python tools/core_ab.py ab_old/pkgA new ...   ("new" = in-tree package)
import importlib.util, os, sys, time; sys.path.insert(0, '.')
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
reps = 50
for mode in ("bf16", "tf32x3"):
    for mrows in (int(x) for x in os.environ.get("ROWS", "6250,12500,50000").split(",")):
        B = torch.empty((mrows, 256), device='cuda').uniform_(-1, 1)
        res, outs = {}, {}
        for rnd in range(3):
            for name, mod in mods:
                s = mod.Sketch(42, 'gaussian', 50000, 256, mode=mode)
                C = s.core_block(B, 0); torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps): s.core_block(B, 0, out=C)
                e1.record(); torch.cuda.synchronize()
                res.setdefault(name, []).append(e0.elapsed_time(e1) / reps * 1000)
                outs[name] = C.double()
        ref = outs[mods[0][0]]
        print(f"{mode:6s} m={mrows:6d} " + "  ".join(
            f"{os.path.basename(n)}={sorted(v)[1]:.1f}us(relF vs first {float((outs[n] - ref).norm() / ref.norm()):.1e})"
            for n, v in res.items()), flush=True)
