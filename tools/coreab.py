import sys, time; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
for m, r in ((50000, 1024), (50000, 256), (25000, 512)):
    B = torch.empty((m, r), device='cuda').uniform_(-1, 1)
    for core in ("auto", "simt"):
        s = sk.Sketch(42, 'gaussian', 200000, r, mode="bf16", core=core)
        s.core_block(B, 0); torch.cuda.synchronize(); time.sleep(0.2)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): s.core_block(B, 0)
        e1.record(); torch.cuda.synchronize()
        print(f"core m={m} r={r} {core}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
