"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

c2 (n = 50,000 RBF kernel, r = 256, bf16 with the bench's transform = fast, clusters of 3 CTA
pairs) and c3 (4,000,000 x 2,048, r = 128 Rademacher, tf32): sampled outputs against the fp64
oracle computed row by row, plus properties that hold at any size (C symmetric within twice the
tolerance -- C and its transpose each sit within TOL of the exact symmetric Omega^T A Omega --,
bit-identical reruns, bit-exact B in c3's integer regime).
"""
import numpy as np
import pytest

import oracle
from inputs import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 42
TOL = 5e-3  # tf32 / bf16 modes (north star)


def _relF(x, ref):
    x = np.asarray(x, np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


def test_c2_full_size_default(capfd, monkeypatch):
    import paper_2603_20966_b200 as sk
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    n, r = 50000, 256
    A = torch.empty((n, n), dtype=torch.float32, device="cuda")
    synth.rbf_kernel_device(2, n, 3072, out=A)
    s = sk.Sketch(SEED, "gaussian", n, r, mode="bf16", omega="fast")
    B, C = s.nystrom_core(A)
    B2, C2 = s.nystrom_core(A)
    torch.cuda.synchronize()
    plans = [l for l in capfd.readouterr().err.splitlines() if l.startswith("[sketch plan]") and f"n1={n}" in l]
    assert plans and all(" cl=3 " in l for l in plans), plans[:2]
    assert torch.equal(B, B2) and torch.equal(C, C2)
    rows = sorted(set(np.linspace(0, n - 1, 24).astype(int).tolist()) | {1, n - 2})
    Bref = oracle.sketch(SEED, "gaussian", A[rows].cpu().numpy(), r)
    assert _relF(B[rows].cpu().numpy(), Bref) <= TOL
    Bh = B.double().cpu().numpy()
    Cown = oracle.core(SEED, "gaussian", Bh, 0)
    Cg = C.double().cpu().numpy()
    assert _relF(Cg, Cown) <= TOL
    assert _relF(Cg, Cg.T) <= 2 * TOL


def test_c3_full_size_integer_exact():
    import paper_2603_20966_b200 as sk
    n1, n2, r = 4_000_000, 2048, 128
    A = synth.int_matrix_device(3, n1, n2, -4, 4)
    s = sk.Sketch(SEED, "rademacher", n2, r, mode="tf32")
    B = s.apply(A)
    torch.cuda.synchronize()
    rows = sorted(set(np.linspace(0, n1 - 1, 32).astype(int).tolist()) | {n1 - 1, n1 - 129})
    Bref = oracle.sketch(SEED, "rademacher", A[rows].double().cpu().numpy(), r)
    assert np.array_equal(B[rows].double().cpu().numpy(), Bref)
    # every B entry is an integer of magnitude <= 4 n2 (a property of the whole output)
    assert torch.equal(B, B.round()) and float(B.abs().max()) <= 4 * n2
    del A, B
    torch.cuda.empty_cache()


def test_c2_full_size_tf32x3():
    """The API's default, fp32-accurate mode at c2's full size (K = 50,000 per B row: 49 promoted TMEM
    chunks): sampled rows of B and all of C within the north star's 1e-5."""
    import paper_2603_20966_b200 as sk
    n, r = 50000, 256
    A = torch.empty((n, n), dtype=torch.float32, device="cuda")
    synth.rbf_kernel_device(2, n, 3072, out=A)
    s = sk.Sketch(SEED, "gaussian", n, r, mode="tf32x3")
    B, C = s.nystrom_core(A)
    torch.cuda.synchronize()
    rows = sorted(set(np.linspace(0, n - 1, 16).astype(int).tolist()) | {1, n - 2})
    Bref = oracle.sketch(SEED, "gaussian", A[rows].cpu().numpy(), r)
    assert _relF(B[rows].cpu().numpy(), Bref) <= 1e-5
    Cown = oracle.core(SEED, "gaussian", B.double().cpu().numpy(), 0)
    assert _relF(C.double().cpu().numpy(), Cown) <= 1e-5
    del A
    torch.cuda.empty_cache()


def test_c4_full_size_sampled_rows():
    """c4 at full size (2,048 x 4,000,000, r = 512 Gaussian, bf16 / fast): ONE pass over A with two N = 256
    column blocks per CTA, in the bench's launch configuration; sampled rows against the oracle (which
    materialises Omega for all 4M rows in fp64 -- 16 GB of host memory -- so only a few rows)."""
    import paper_2603_20966_b200 as sk
    n1, n2, r = 2048, 4_000_000, 512
    A = synth.uniform_device(4, n1, n2)
    s = sk.Sketch(SEED, "gaussian", n2, r, mode="bf16", omega="fast")
    B = s.apply(A)
    torch.cuda.synchronize()
    rows = [0, 777, 2047]
    Bref = oracle.sketch(SEED, "gaussian", A[rows].cpu().numpy(), r)
    assert _relF(B[rows].cpu().numpy(), Bref) <= TOL
    del A
    torch.cuda.empty_cache()
