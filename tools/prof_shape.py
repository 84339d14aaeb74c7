"""B = A Omega on one shape, for ncu / sanitizer runs and quick timings.
usage: [CG=0|1|2|4|6|8] python tools/prof_shape.py N1 N2 R MODE OMEGA DIST [REPS]
(A ~ U[-1/2, 1/2) generated on the GPU; CG = sketch_set_cta_group override)"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_20966_b200 as sk  # noqa: E402

n1, n2, r = (int(x) for x in sys.argv[1:4])
mode, omega, dist = sys.argv[4:7]
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
A = torch.empty((n1, n2), device="cuda").uniform_(-0.5, 0.5)
s = sk.Sketch(42, dist, n2, r, mode=mode, omega=omega, cta_group=int(os.environ.get("CG", "0")))
B = torch.empty((n1, r), device="cuda")
s.apply(A, out=B)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    s.apply(A, out=B)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{n1}x{n2} r={r} {mode}/{omega}/{dist}: {ms:.3f} ms/apply, {4.0 * n1 * n2 / ms / 1e6:.1f} GB/s of A")
