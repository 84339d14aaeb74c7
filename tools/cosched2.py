# Co-scheduling experiment: clusters-of-4-pairs kernel on rows [0, n1a) first, then a pairs kernel capped
# at the SMs the 8-CTA clusters leave idle (SK_MAX_WORKERS pairs) on rows [n1a, n1), on two streams.
import os, sys, time; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
main = sk.Sketch(42, 'gaussian', n, r, mode="bf16", cta_group=8)
for aux_workers in (14, 12):
    for n1a in (50000, 45056, 43008, 40960):
        n1b = n - n1a
        os.environ["SK_MAX_WORKERS"] = str(aux_workers)
        aux = sk.Sketch(42, 'gaussian', n, r, mode="bf16", cta_group=2)
        def run():
            ev = torch.cuda.Event(); ev.record()
            s1.wait_event(ev); s2.wait_event(ev)
            os.environ.pop("SK_MAX_WORKERS", None)
            main.apply(A[:n1a], out=B[:n1a], stream=s1)
            os.environ["SK_MAX_WORKERS"] = str(aux_workers)
            if n1b: aux.apply(A[n1a:], out=B[n1a:], stream=s2)
            torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        run(); torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            time.sleep(0.4)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): run()
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 3)
        print(f"aux pairs {aux_workers} main rows {n1a} aux rows {n1b}: {sorted(ts)[1]:.3f} ms", flush=True)
        if n1b == 0: pass
