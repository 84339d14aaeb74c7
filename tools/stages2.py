import sys, os, subprocess
code = r'''
import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
for mode, omega, cg in [("bf16", "accurate", 4), ("bf16", "fast", 4), ("bf16", "accurate", 2), ("bf16", "accurate", 8)]:
    s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
    for _ in range(2): s.apply(A, out=B)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(6): s.apply(A, out=B)
    e1.record(); torch.cuda.synchronize()
    print(f"{sys.argv[1]} {mode:6s} {omega:8s} cg{cg}: {e0.elapsed_time(e1)/6:.3f} ms", flush=True)
'''
for cfg in sys.argv[1:]:
    a, o = cfg.split(",")
    env = dict(os.environ)
    if a != "-": env["SK_A_STAGES"] = a
    if o != "-": env["SK_O_STAGES"] = o
    subprocess.run([sys.executable, "-c", code, f"A{a}/O{o}"], env=env, timeout=300)
