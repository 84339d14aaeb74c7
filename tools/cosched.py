# Experiment: clusters-of-4-pairs kernel on rows [0, n1a) + pairs kernel on rows [n1a, n1) concurrently
# (two streams), to use the SMs the 8-CTA clusters cannot occupy.
import os, sys, time; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for mode, omega in (("bf16", "accurate"), ("tf32", "fast")):
    main = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=8)
    aux = sk.Sketch(42, 'gaussian', n, r, mode=mode, omega=omega, cta_group=2)
    for n1b in (0, 2048, 4096, 5120, 6144, 7168, 8192):
        n1a = n - n1b
        def run():
            ev = torch.cuda.Event(); ev.record()
            s1.wait_event(ev); s2.wait_event(ev)
            main.apply(A[:n1a], out=B[:n1a], stream=s1)
            if n1b: aux.apply(A[n1a:], out=B[n1a:], stream=s2)
            torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        run(); torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            time.sleep(0.3)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): run()
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 5)
        print(f"{mode} {omega} n1b={n1b}: {min(ts):.3f} ms", flush=True)
