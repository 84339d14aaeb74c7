# Potential of the 16 SMs the 6-CTA clusters leave idle at c2: the last s rows of A sketched by a
# second, unshared-pair handle on a second stream, concurrently with the main launch on the rest.
import os, sys; sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as sk
n, r = 50000, 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
main = sk.Sketch(42, "gaussian", n, r, mode="bf16", omega="fast")
side = sk.Sketch(42, "gaussian", n, r, mode="bf16", omega="fast", cta_group=int(os.environ.get("SIDE_CG", "2")))
s0 = torch.cuda.current_stream(); s1 = torch.cuda.Stream()
def run(s):
    fork = torch.cuda.Event(); fork.record(s0)
    main.apply(A[: n - s], out=B[: n - s])
    if s:
        s1.wait_event(fork)
        os.environ["SK_INPLACE"] = "0"
        with torch.cuda.stream(s1):
            side.apply(A[n - s:], out=B[n - s:], stream=s1)
        os.environ.pop("SK_INPLACE", None)
        join = torch.cuda.Event(); join.record(s1); s0.wait_event(join)
ref = None
for s in [0] + [int(x) for x in os.environ.get("SIDES", "256,512,768,1024,1536,2048").split(",")]:
    for _ in range(2): run(s)
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for _ in range(5): run(s)
        e1.record(s0); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 5)
    Bc = B.clone()
    if ref is None: ref = Bc
    print(f"side rows {s:5d}: {sorted(ts)[2]:.3f} ms  (max |B - B_s0| = {(Bc - ref).abs().max().item():.2e})", flush=True)
