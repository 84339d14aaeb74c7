import sys, os, subprocess
# sweep SK_O_STAGES for cluster (cg4) vs pairs (cg2) on tf32 fast / bf16 fast / tf32x3
code = r'''
import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
for mode, omega in [("tf32", "fast"), ("tf32", "accurate"), ("bf16", "fast"), ("tf32x3", "accurate")]:
    for cg in (2, 4):
        try:
            s = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=cg)
            for _ in range(2): s.apply(A, out=B)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): s.apply(A, out=B)
            e1.record(); torch.cuda.synchronize()
            print(f"ost={sys.argv[1]} {mode:6s} {omega:8s} cg{cg}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
        except Exception as ex:
            print(f"ost={sys.argv[1]} {mode} {omega} cg{cg}: {ex}", flush=True)
'''
for ost in sys.argv[1:]:
    env = dict(os.environ, SK_O_STAGES=ost)
    subprocess.run([sys.executable, "-c", code, ost], env=env, timeout=300)
