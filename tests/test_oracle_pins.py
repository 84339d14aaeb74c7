"""Pins for oracle/ (CPU only, -m "not gpu").

The oracle is checked against things other than itself: published known-answer
vectors, independently computed worked values, closed forms, library routines
(numpy matmul / pinv, scipy's normal CDF), invariants and brute force.  Each test
names the plausible mistake it is there to catch.
"""
import math
import os
import struct

import numpy as np
import pytest
import scipy.stats

import oracle
from inputs import synth
from tests.conftest import golden_path

GAUSS, RADE, UNIF = oracle.GAUSSIAN, oracle.RADEMACHER, oracle.UNIFORM


def _f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def _relF(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / max(np.linalg.norm(ref), 1e-300))


# --------------------------------------------------------------------------- Philox
def _read_kat():
    rows = []
    for line in open(golden_path("philox_kat.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(t, 16) for t in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answer_vectors():
    # catches: wrong multiplier / Weyl constant, swapped hi/lo, wrong round count, key bump order
    kats = _read_kat()
    assert len(kats) == 3
    for ctr, key, out in kats:
        assert list(oracle.philox4x32_10(ctr, key)) == out


# --------------------------------------------------------------------------- Omega mapping
def _read_worked():
    rows = []
    for line in open(golden_path("omega_worked.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, words, gauss, rade = [s.split() for s in line.split("|")]
        rows.append((int(head[0]), int(head[1]), [int(w, 16) for w in words],
                     [int(g, 16) for g in gauss], [(-1.0 if s == "-" else 1.0) for s in rade]))
    return rows


def test_zero_kat_by_construction():
    # seed 0, col 0, rows 0..3: counter (0,0,0,0), key (0,0) -> the zero KAT vector
    words = oracle.omega_words(0, GAUSS, 0, 4, 0, 1).ravel().tolist()
    assert words == _read_kat()[0][2]


def test_worked_values_survey_appendix_a():
    # catches: counter layout (q vs j, column slot, tag slot), pair selection p = j & 2,
    # cos/sin branch per row parity, Rademacher bit indexing
    for seed, col, words, gauss_bits, rade in _read_worked():
        assert oracle.omega_words(seed, GAUSS, 0, 4, col, 1).ravel().tolist() == words
        g = oracle.omega(seed, GAUSS, 0, 4, col, 1).ravel()
        assert [_f32_bits(float(v)) for v in g] == gauss_bits
        assert oracle.omega(seed, RADE, 0, 8, col, 1).ravel().tolist() == rade
    u = oracle.omega(0, UNIF, 0, 4, 0, 1).ravel()
    np.testing.assert_allclose(u, [0.399046421, 0.880520165, 0.735712767, 0.605481803], rtol=0, atol=5e-9)


def test_rademacher_words_match_tag1_counter():
    # Rademacher row j uses Philox((j>>7, 0, k, 1)) word (j>>5)&3, bit j&31 (reading O1)
    seed = 7
    for j in (0, 31, 32, 127, 128, 1000, 2**33 + 5):
        for k in (0, 3):
            g = j >> 7
            x = oracle.philox4x32_10([g & 0xffffffff, g >> 32, k, 1], [seed, 0])
            assert oracle.omega_words(seed, RADE, j, 1, k, 1)[0, 0] == x[(j >> 5) & 3]
            bit = (x[(j >> 5) & 3] >> (j & 31)) & 1
            assert oracle.omega(seed, RADE, j, 1, k, 1)[0, 0] == (-1.0 if bit else 1.0)


def test_64bit_seed_and_row_split():
    # key = (seed lo, seed hi); counter word0/word1 = q lo / q hi
    seed = (0x12345678 << 32) | 0x9ABCDEF0
    j = (5 << 34) + 6  # q = j >> 2 has a nonzero high word
    q = j >> 2
    x = oracle.philox4x32_10([q & 0xffffffff, q >> 32, 11, 0], [0x9ABCDEF0, 0x12345678])
    assert oracle.omega_words(seed, GAUSS, j, 1, 11, 1)[0, 0] == x[j & 3]


# --------------------------------------------------------------------------- Box-Muller closed forms
def _w(v24: int) -> int:
    return (v24 << 8) | 0xAB  # low 8 bits are discarded by the mapping


@pytest.mark.parametrize("u1_24", [0, 1, 12345, (1 << 23), (1 << 24) - 2, (1 << 24) - 1])
def test_box_muller_angles_closed_form(u1_24):
    # catches: sin/cos swapped per parity, wrong quadrant signs, a dropped 2 in 2*pi*u2
    u1 = (u1_24 + 1) / 2**24
    R = math.sqrt(-2.0 * math.log(u1))
    s2 = math.sqrt(0.5)
    cases = {  # u2 -> (cos 2 pi u2, sin 2 pi u2)
        0: (1.0, 0.0), 1 << 21: (s2, s2), 1 << 22: (0.0, 1.0), 3 << 21: (-s2, s2),
        1 << 23: (-1.0, 0.0), 5 << 21: (-s2, -s2), 3 << 22: (0.0, -1.0), 7 << 21: (s2, -s2),
    }
    for u2_24, (c, s) in cases.items():
        ze, zo = oracle.box_muller(_w(u1_24), _w(u2_24))
        assert ze == pytest.approx(R * c, rel=1e-15, abs=1e-300)
        assert zo == pytest.approx(R * s, rel=1e-15, abs=1e-300)


def test_box_muller_radius_extremes():
    # u1 = 1 (word >> 8 = 2^24 - 1) -> R = 0 ; u1 = 2^-24 -> R = sqrt(48 ln 2) = max |z|
    ze, zo = oracle.box_muller(_w((1 << 24) - 1), _w(12345))
    assert ze == 0.0 and zo == 0.0
    ze, zo = oracle.box_muller(_w(0), _w(0))
    assert ze == pytest.approx(math.sqrt(48.0 * math.log(2.0)), rel=1e-15)
    assert ze == pytest.approx(5.768107, abs=1e-6)
    assert zo == 0.0


def test_box_muller_quarter_turn_symmetry():
    # cos(2 pi (u2 + 1/4)) = -sin(2 pi u2), sin(2 pi (u2 + 1/4)) = cos(2 pi u2): exact in the
    # quarter-turn reduction; catches a reduction that is only approximately periodic
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = int(rng.integers(0, 1 << 24))
        b = int(rng.integers(0, 3 << 22))
        ze, zo = oracle.box_muller(_w(a), _w(b))
        ze2, zo2 = oracle.box_muller(_w(a), _w(b + (1 << 22)))
        assert ze2 == -zo and zo2 == ze


# --------------------------------------------------------------------------- statistics
def test_gaussian_moments_and_ks():
    # catches: missing sqrt / -2 factor (variance), biased angle (mean), heavy tails (kurtosis)
    z = oracle.omega(42, GAUSS, 0, 1 << 14, 0, 64).astype(np.float64).ravel()  # 2^20 samples
    n = z.size
    assert abs(z.mean()) < 5.0 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 5.0 * math.sqrt(2.0 / n)
    kurt = ((z - z.mean()) ** 4).mean() / z.var() ** 2
    assert abs(kurt - 3.0) < 5.0 * math.sqrt(24.0 / n)
    assert scipy.stats.kstest(z, "norm").pvalue > 1e-4
    assert np.abs(z).max() <= math.sqrt(48.0 * math.log(2.0)) + 1e-6
    # even rows (cos branch) and odd rows (sin branch) are each N(0,1) and uncorrelated
    Z = oracle.omega(42, GAUSS, 0, 1 << 14, 0, 64).astype(np.float64)
    ev, od = Z[0::2].ravel(), Z[1::2].ravel()
    assert scipy.stats.kstest(ev, "norm").pvalue > 1e-4
    assert scipy.stats.kstest(od, "norm").pvalue > 1e-4
    assert abs(np.corrcoef(ev, od)[0, 1]) < 5.0 / math.sqrt(ev.size)


def test_omega_gram_is_identity_in_expectation():
    # E[Omega Omega^T]/r = I  <=>  Omega^T Omega / n2 -> I_r  (north star statistic)
    n2, r = 1 << 16, 64
    for dist in (GAUSS, RADE):
        Om = oracle.omega(5, dist, 0, n2, 0, r).astype(np.float64)
        G = Om.T @ Om / n2
        assert np.abs(G - np.eye(r)).max() <= 6.0 / math.sqrt(n2)
    Om = oracle.omega(5, RADE, 0, 1000, 0, 16).astype(np.float64)
    assert np.array_equal(np.diag(Om.T @ Om), np.full(16, 1000.0))  # exact for +-1


def test_rademacher_balance():
    Om = oracle.omega(9, RADE, 0, 1 << 15, 0, 32)
    assert set(np.unique(Om).tolist()) == {-1.0, 1.0}
    frac = (Om < 0).mean()
    assert abs(frac - 0.5) < 5.0 * 0.5 / math.sqrt(Om.size)


def test_uniform_grid_and_moments():
    u = oracle.omega(11, UNIF, 0, 1 << 14, 0, 64).astype(np.float64).ravel()
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.all(u * 2**24 == np.floor(u * 2**24))  # exact 24-bit grid
    assert abs(u.mean() - 0.5) < 5.0 * math.sqrt(1.0 / 12.0 / u.size)
    assert abs(u.var() - 1.0 / 12.0) < 0.002


# --------------------------------------------------------------------------- purity / block consistency
@pytest.mark.parametrize("dist", [GAUSS, RADE, UNIF])
def test_block_consistency(dist):
    big = oracle.omega(3, dist, 0, 300, 0, 20)
    assert np.array_equal(oracle.omega(3, dist, 97, 150, 5, 11), big[97:247, 5:16])
    bw = oracle.omega_words(3, dist, 0, 300, 0, 20)
    assert np.array_equal(oracle.omega_words(3, dist, 131, 33, 2, 3), bw[131:164, 2:5])
    # prefix consistency in r and independence of the block origin
    assert np.array_equal(oracle.omega(3, dist, 0, 300, 0, 8), big[:, :8])


# --------------------------------------------------------------------------- B = A Omega
def test_sketch_matches_numpy_matmul():
    # library routine on the materialised Omega (catches transposed operand / wrong index)
    A = synth.uniform(1, 37, 203)
    for dist in (GAUSS, RADE, UNIF):
        Om = oracle.omega(42, dist, 0, 203, 0, 24).astype(np.float64)
        B = oracle.sketch(42, dist, A, 24)
        assert _relF(B, A.astype(np.float64) @ Om) < 1e-13


def test_sketch_block_offset():
    # block form: A_blk's column 0 pairs with Omega row k0 (PAPER.md:411 GenRandom per block)
    A = synth.uniform(2, 16, 100)
    full = oracle.sketch(4, GAUSS, A, 8)
    part = oracle.sketch(4, GAUSS, A[:, :60], 8) + oracle.sketch(4, GAUSS, A[:, 60:], 8, k0=60)
    assert _relF(part, full) < 1e-14


def test_sketch_special_matrices():
    n = 64
    Om = oracle.omega(42, GAUSS, 0, n, 0, 16).astype(np.float64)
    assert np.array_equal(oracle.sketch(42, GAUSS, np.eye(n, dtype=np.float32), 16), Om)
    E = np.zeros((5, n), dtype=np.float32)
    E[3, 17] = 1.0
    B = oracle.sketch(42, GAUSS, E, 16)
    assert np.array_equal(B[3], Om[17]) and not B[[0, 1, 2, 4]].any()
    assert not oracle.sketch(42, GAUSS, np.zeros((3, n), np.float32), 16).any()


def test_sketch_brute_force_tiny():
    A = synth.uniform(8, 3, 9)
    for dist in (GAUSS, RADE):
        B = oracle.sketch(1, dist, A, 5)
        for i in range(3):
            for k in range(5):
                ref = math.fsum(float(A[i, j]) * float(oracle.omega(1, dist, j, 1, k, 1)[0, 0]) for j in range(9))
                assert B[i, k] == pytest.approx(ref, rel=1e-15, abs=1e-15)


def test_sketch_integer_exact_regime():
    A = synth.int_matrix(3, 50, 300, -4, 4)
    Om = oracle.omega(42, RADE, 0, 300, 0, 16)
    B = oracle.sketch(42, RADE, A, 16)
    assert np.array_equal(B, (A.astype(np.int64) @ Om.astype(np.int64)).astype(np.float64))


# --------------------------------------------------------------------------- C = Omega^T B
def test_core_associativity_nonsymmetric():
    # (Omega^T A) Omega == Omega^T (A Omega): catches a transposed C
    A = synth.uniform(5, 120, 120)
    B, C = oracle.nystrom_core(42, GAUSS, A, 12)
    Om = oracle.omega(42, GAUSS, 0, 120, 0, 12).astype(np.float64)
    assert _relF(C, (Om.T @ A.astype(np.float64)) @ Om) < 1e-12
    assert _relF(B, A.astype(np.float64) @ Om) < 1e-13


def test_core_symmetry_and_identity():
    A = synth.symmetric_uniform(6, 150)
    B, C = oracle.nystrom_core(42, GAUSS, A, 16)
    assert _relF(C, C.T) < 1e-13
    Om = oracle.omega(42, GAUSS, 0, 150, 0, 16).astype(np.float64)
    _, CI = oracle.nystrom_core(42, GAUSS, np.eye(150, dtype=np.float32), 16)
    assert _relF(CI, Om.T @ Om) < 1e-14


def test_core_lowrank_closed_form():
    # A = X X^T: B = X (X^T Omega), C = (X^T Omega)^T (X^T Omega), exactly symmetric PSD
    A, X = synth.lowrank_psd(7, 200, 6)
    for dist in (GAUSS, RADE):
        B, C = oracle.nystrom_core(42, dist, A, 10)
        Om = oracle.omega(42, dist, 0, 200, 0, 10).astype(np.float64)
        Y = X.T @ Om
        assert _relF(B, X @ Y) < 1e-13
        assert _relF(C, Y.T @ Y) < 1e-12
        if dist == RADE:
            assert np.array_equal(C, Y.T @ Y)  # integer-exact


def test_core_block_offset():
    A = synth.symmetric_uniform(8, 90)
    B, C = oracle.nystrom_core(42, GAUSS, A, 8)
    Cp = oracle.core(42, GAUSS, B[:40]) + oracle.core(42, GAUSS, B[40:], i0=40)
    assert _relF(Cp, C) < 1e-14


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_nystrom_exact_recovery(seed):
    # rank-20 SPSD, n=400, r=40: B C^+ B^T = A (pinv tol 1e-12)
    A, _ = synth.lowrank_psd(seed, 400, 20)  # integer X: A is exact in fp32, rank 20
    B, C = oracle.nystrom_core(seed, GAUSS, A, 40)
    At = B @ np.linalg.pinv(C, rcond=1e-12, hermitian=True) @ B.T
    assert np.linalg.norm(At - A.astype(np.float64)) / np.linalg.norm(A.astype(np.float64)) < 1e-8


def test_nystrom_error_decreases_with_rank():
    A = synth.rbf_kernel(4, 600, 8)
    errs = []
    for r in (10, 40, 120):
        B, C = oracle.nystrom_core(42, GAUSS, A, r)
        At = B @ np.linalg.pinv(C, rcond=1e-12, hermitian=True) @ B.T
        errs.append(np.linalg.norm(At - A) / np.linalg.norm(A))
    assert errs[0] > errs[1] > errs[2]


def test_worked_values_regenerate_from_independent_generator():
    """tests/golden/omega_worked.txt is reproduced by its committed generator (an independent pure-Python
    Philox4x32-10 + O1 mapping that imports neither oracle/ nor the package)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    gen = os.path.join(here, "golden", "gen_omega_worked.py")
    src = open(gen).read()
    assert "import oracle" not in src and "paper_2603_20966_b200" not in src
    out = subprocess.run([sys.executable, gen], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(here, "golden", "omega_worked.txt")) as f:
        assert out == f.read()
