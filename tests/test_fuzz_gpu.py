"""Seeded random-configuration parity sweep: the CUDA path against the fp64 oracle on shapes, offsets,
strides, distributions, modes, transforms, split-K factors and CTA groupings drawn at random.

Every case is reproducible from its index (numpy PCG64 seeded with 1000 + index).  Each case checks:
- the integer regime (A in {-4..4}, Rademacher Omega: every partial sum is an exact fp32 integer, so
  B, and C for square A, are bit-exact in every mode and plan);
- a float A with the case's distribution: relF(B) (and relF(C)) within the north-star tolerance of the
  mode (5e-3 tf32 / bf16, 1e-5 tf32x3).
Alg. 1 local product, Alg. 2 core C = Omega^T B, block offsets
(global Omega rows).
"""
import numpy as np
import pytest

import oracle
from inputs import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"tf32": 5e-3, "bf16": 5e-3, "tf32x3": 1e-5}
NCASES = 160


def _relF(x, ref):
    x = np.asarray(x, np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


def _case(i):
    g = np.random.default_rng(1000 + i)
    square = g.random() < 0.3
    while True:  # at most 3e9 multiply-adds per oracle call: the fp64 oracle stays within seconds
        # square problems stay at n <= 2600, so the integer-regime B fits tf32's 11 bits in the core
        n1 = int(g.choice([1, 7, 129, 300, 777, 1500, 2600] if square else [1, 7, 128, 129, 300, 777, 1500, 2048, 4100, 6200]))
        n2 = n1 if square else int(g.choice([1, 3, 64, 100, 513, 1024, 2047, 5000, 9000]))
        r = int(g.choice([1, 5, 16, 40, 100, 256, 300, 520]))
        if n1 * n2 * r + (n1 * r * r if square else 0) <= 3e9:
            break
    mode = str(g.choice(["tf32x3", "tf32", "bf16"]))
    dist = str(g.choice(["gaussian", "rademacher", "uniform"]))
    omega = "accurate" if mode == "tf32x3" or dist != "gaussian" else str(g.choice(["accurate", "fast"]))
    split = int(g.choice([0, 0, 1, 2, 5]))
    cg = int(g.choice([0, 0, 0, 1, 2, 4, 6, 8]))
    k0 = 0 if square else int(g.choice([0, 0, 1, 3, 64, 1001, 2**33 + 5]))
    pad = int(g.choice([0, 0, 4, 12]))   # lda = n2 + pad (multiple of 4 keeps TMA's 16-B rows)
    lda = -(-n2 // 4) * 4 + pad
    return dict(n1=n1, n2=n2, r=r, mode=mode, dist=dist, omega=omega, split=split, cg=cg, k0=k0, lda=lda,
                seed=int(g.integers(0, 2**63)))


def _run(sk, c, A):
    """B (and C for square problems at k0 = 0) through the library, A stored with leading dimension lda."""
    n1, n2, lda = c["n1"], c["n2"], c["lda"]
    buf = torch.zeros((n1, lda), device="cuda")
    buf[:, :n2] = torch.from_numpy(np.ascontiguousarray(A))
    Ad = buf[:, :n2]
    if c["n1"] == c["n2"] and c["k0"] == 0:
        s = sk.Sketch(c["seed"], c["dist"], n2, c["r"], mode=c["mode"], omega=c["omega"], split_k=c["split"],
                      cta_group=c["cg"])
        B, C = s.nystrom_core(Ad)
        return B.cpu().numpy(), C.cpu().numpy()
    s = sk.Sketch(c["seed"], c["dist"], c["k0"] + n2, c["r"], mode=c["mode"], omega=c["omega"],
                  split_k=c["split"], cta_group=c["cg"])
    B = s.apply_block(Ad, c["k0"]) if c["k0"] else s.apply(Ad)
    return B.cpu().numpy(), None


@pytest.mark.parametrize("i", range(NCASES))
def test_fuzz_case(i):
    import paper_2603_20966_b200 as sk
    c = _case(i)
    square = c["n1"] == c["n2"] and c["k0"] == 0
    # integer regime: bit-exact whatever the plan
    ci = dict(c, dist="rademacher", omega="accurate")
    Ai = synth.int_matrix(i, c["n1"], c["n2"], -4, 4, symmetric=square)
    B, C = _run(sk, ci, Ai)
    if square:
        Bref, Cref = oracle.nystrom_core(ci["seed"], "rademacher", Ai, c["r"])
        assert np.array_equal(C.astype(np.float64), Cref), c
    else:
        Bref = oracle.sketch(ci["seed"], "rademacher", Ai, c["r"], k0=c["k0"])
    assert np.array_equal(B.astype(np.float64), Bref), c
    # float A with the case's distribution: north-star tolerance
    A = synth.symmetric_uniform(i, c["n1"]) if square else synth.uniform(i, c["n1"], c["n2"])
    B, C = _run(sk, c, A)
    if square:
        Bref, Cref = oracle.nystrom_core(c["seed"], c["dist"], A, c["r"])
        assert _relF(C, Cref) <= TOL[c["mode"]], c
    else:
        Bref = oracle.sketch(c["seed"], c["dist"], A, c["r"], k0=c["k0"])
    assert _relF(B, Bref) <= TOL[c["mode"]], c
