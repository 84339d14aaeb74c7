"""Small cases of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
sketch GEMM in each mode and CTA grouping (single CTAs, pairs, clusters of 2 / 3 / 4 pairs, the
two-column-block variant with clusters of 4 and 8 pairs), split-K and stream-K reduces, the tcgen05
core GEMM (tf32 and 3xTF32), the SIMT core, Omega materialisation, peer sum and column pack.
Each case is checked against the fp64 oracle so a silent corruption also fails the run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2603_20966_b200 as sk  # noqa: E402
from inputs import synth  # noqa: E402

SEED = 42
TOL = {"tf32": 5e-3, "bf16": 5e-3, "tf32x3": 1e-5}
fails = 0


def rel(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / np.linalg.norm(ref))


def case(name, n1, n2, r, mode, dist="gaussian", cg=0, omega="accurate", nystrom=False):
    global fails
    A = synth.symmetric_uniform(3, n1) if nystrom else synth.uniform(3, n1, n2)
    s = sk.Sketch(SEED, dist, n2, r, mode=mode, cta_group=cg, omega=omega)
    Ad = torch.from_numpy(A).cuda()
    if nystrom:
        B, C = s.nystrom_core(Ad)
        Bref, Cref = oracle.nystrom_core(SEED, dist, A, r)
        e = max(rel(B.cpu().numpy(), Bref), rel(C.cpu().numpy(), Cref))
    else:
        B = s.apply(Ad)
        e = rel(B.cpu().numpy(), oracle.sketch(SEED, dist, A, r))
    torch.cuda.synchronize()
    ok = e <= TOL[mode]
    fails += 0 if ok else 1
    print(f"{'ok ' if ok else 'BAD'} {name}: relF {e:.2e}", flush=True)


for mode in ("tf32", "bf16", "tf32x3"):
    case(f"single CTA {mode}", 200, 700, 40, mode, cg=1)
    case(f"pairs {mode}", 600, 900, 64, mode, cg=2)
    case(f"nystrom {mode}", 700, 700, 48, mode, nystrom=True)
for cg in (4, 6, 8):
    case(f"cluster cg={cg} bf16", 2100, 600, 128, "bf16", cg=cg)
case("cluster cg=6 bf16 fast (auto)", 6200, 300, 64, "bf16", omega="fast")
case("two column blocks, clusters of 4 pairs", 900, 500, 400, "bf16")
case("two column blocks, clusters of 8 pairs", 2048, 500, 512, "tf32")
case("rademacher pairs", 600, 900, 64, "tf32", dist="rademacher")
case("uniform clusters", 2100, 600, 128, "tf32", dist="uniform")
s = sk.Sketch(SEED, "gaussian", 1000, 32)
Om = s.generate(0, 100).cpu().numpy()
assert np.abs(Om.astype(np.float64) - oracle.omega(SEED, "gaussian", 0, 100, 0, 32)).max() < 1e-5
print("generate ok", flush=True)
x = torch.arange(1024, dtype=torch.float32, device="cuda")
out = torch.empty(1024, device="cuda")
sk.sum_peers([x.data_ptr(), x.data_ptr()], 1024, out)
torch.cuda.synchronize()
assert torch.equal(out, 2 * x)
Bm = torch.arange(40 * 12, dtype=torch.float32, device="cuda").view(40, 12)
pk = s.pack_cols(Bm, [0, 5, 12])
assert torch.equal(pk[:200], Bm[:, :5].reshape(-1)) and torch.equal(pk[200:], Bm[:, 5:].reshape(-1))
print("sum_peers / pack_cols ok", flush=True)
print("FAILURES", fails)
sys.exit(1 if fails else 0)
