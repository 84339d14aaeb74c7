"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerances (north star):
  Omega words / Rademacher signs / uniforms: bit-exact;  Gaussians: <= 2 ulp (accurate transform);
  B, C: relF <= 5e-3 in tf32 / bf16 modes, <= 1e-5 in tf32x3; bit-exact in the integer regime
  (A in {-4..4}, Rademacher Omega: every partial sum is an exact fp32 integer, any order).
"""
import numpy as np
import pytest

import oracle
from inputs import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 42


def _sk():
    import paper_2603_20966_b200 as sk
    return sk


def _relF(x, ref):
    x = np.asarray(x, np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


def _ulp(a, b):
    """ulp distance between fp32 arrays, +0 == -0."""
    def ordered(x):
        i = np.asarray(x, np.float32).view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    return np.abs(ordered(a) - ordered(b))


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


TOL = {"tf32": 5e-3, "bf16": 5e-3, "tf32x3": 1e-5}


# ----------------------------------------------------------------------------- Omega
@pytest.mark.parametrize("dist", ["gaussian", "rademacher", "uniform"])
@pytest.mark.parametrize("block", [(0, 64, 0, 16), (3, 130, 5, 9), (1000, 257, 0, 33), (2**33 + 1, 40, 2, 7)])
def test_generate_bits_exact(dist, block):
    sk = _sk()
    row0, nrows, col0, ncols = block
    s = sk.Sketch(SEED, dist, 2**40, 48)
    got = s.generate_bits(row0, nrows, col0, ncols).cpu().numpy().view(np.uint32)
    ref = oracle.omega_words(SEED, dist, row0, nrows, col0, ncols)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("dist", ["rademacher", "uniform"])
def test_generate_values_exact(dist):
    sk = _sk()
    s = sk.Sketch(7, dist, 10**6, 40)
    got = s.generate(77, 1000, 0, 40).cpu().numpy()
    assert np.array_equal(got, oracle.omega(7, dist, 77, 1000, 0, 40))


def test_generate_gaussian_ulp():
    sk = _sk()
    s = sk.Sketch(SEED, "gaussian", 10**7, 64)
    got = s.generate(5, 4096, 0, 64).cpu().numpy()
    ref = oracle.omega(SEED, "gaussian", 5, 4096, 0, 64)
    assert _ulp(got, ref).max() <= 2


@pytest.mark.parametrize("transform", ["accurate"])
def test_box_muller_ulp_sweeps(transform):
    """Every u1 (radius sweep, u2 = 0 so z_even = R exactly) and every u2 at fixed u1s."""
    sk = _sk()
    n = 1 << 24
    w1 = (np.arange(n, dtype=np.uint64) << 8).astype(np.uint32)
    w2 = np.zeros(n, dtype=np.uint32)
    ge, go = sk.debug_box_muller(_dev(w1.view(np.int32)), _dev(w2.view(np.int32)), transform)
    re_, ro = oracle.box_muller_many(w1, w2)
    assert _ulp(ge.cpu().numpy(), re_).max() <= 2
    assert np.all(go.cpu().numpy() == 0.0)
    for u1 in (0, 12345, 1 << 23, (1 << 24) - 2):
        w1c = np.full(n, u1 << 8, dtype=np.uint32)
        ge, go = sk.debug_box_muller(_dev(w1c.view(np.int32)), _dev(w1.view(np.int32)), transform)
        re_, ro = oracle.box_muller_many(w1c, w1)
        assert _ulp(ge.cpu().numpy(), re_).max() <= 2
        assert _ulp(go.cpu().numpy(), ro).max() <= 2


def _fast_err(g, r):
    return np.abs(np.asarray(g, np.float64) - r) / np.maximum(np.abs(r), 1.0)


FAST_BOUND = 2.0 ** -18  # reading R5: |fast - exact| <= 2^-18 max(|z|, 1)


def test_box_muller_fast_sweeps():
    """Fast (MUFU) transform, exhaustively like the accurate one: every u1 (u2 = 0, so z_even = R and
    z_odd must be exactly 0) and every u2 at four u1 values, against the correctly rounded oracle:
    error <= 2^-18 max(|z|, 1) (reading R5), exact zeros at u2 in {0, 1/4, 1/2, 3/4} (reading R14)."""
    sk = _sk()
    n = 1 << 24
    w1 = (np.arange(n, dtype=np.uint64) << 8).astype(np.uint32)
    w2 = np.zeros(n, dtype=np.uint32)
    ge, go = sk.debug_box_muller(_dev(w1.view(np.int32)), _dev(w2.view(np.int32)), "fast")
    re_, ro = oracle.box_muller_many(w1, w2)
    worst = _fast_err(ge.cpu().numpy(), re_).max()
    assert np.all(go.cpu().numpy() == 0.0)
    for u1 in (0, 12345, 1 << 23, (1 << 24) - 2):
        w1c = np.full(n, u1 << 8, dtype=np.uint32)
        ge, go = sk.debug_box_muller(_dev(w1c.view(np.int32)), _dev(w1.view(np.int32)), "fast")
        re_, ro = oracle.box_muller_many(w1c, w1)
        ge, go = ge.cpu().numpy(), go.cpu().numpy()
        worst = max(worst, _fast_err(ge, re_).max(), _fast_err(go, ro).max())
        # quarter turns: u2 = k/4 -> exactly one of cos / sin is zero
        for k, (zc, zs) in enumerate(((False, True), (True, False), (False, True), (True, False))):
            i = k << 22
            assert (ge[i] == 0.0) == zc and (go[i] == 0.0) == zs, (u1, k, ge[i], go[i])
    print(f"fast Box-Muller: max |fast - exact| / max(|z|,1) = 2^{np.log2(worst):.2f}")
    assert worst <= FAST_BOUND


def test_box_muller_fast_random_pairs():
    """... and on 4M random (u1, u2) pairs."""
    sk = _sk()
    rng = np.random.default_rng(0)
    n = 1 << 22
    w1 = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    w2 = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    ge, go = sk.debug_box_muller(_dev(w1.view(np.int32)), _dev(w2.view(np.int32)), "fast")
    re_, ro = oracle.box_muller_many(w1, w2)
    for g, r in ((ge.cpu().numpy(), re_), (go.cpu().numpy(), ro)):
        assert _fast_err(g, r).max() <= FAST_BOUND


# ----------------------------------------------------------------------------- B = A Omega
SHAPES = [
    (512, 512, 16),     # c1
    (300, 1000, 48),    # ragged M / K / N
    (129, 33, 17),      # one row past a tile, tiny K
    (1000, 4099, 256),  # several tiles, ragged K, N = 256
    (64, 2000, 300),    # two column passes (256 + 44)
    (2000, 777, 128),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dist", ["gaussian", "rademacher"])
@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
def test_sketch_parity(shape, dist, mode):
    sk = _sk()
    n1, n2, r = shape
    A = synth.uniform(1, n1, n2)
    s = sk.Sketch(SEED, dist, n2, r, mode=mode)
    B = s.apply(_dev(A)).cpu().numpy()
    ref = oracle.sketch(SEED, dist, A, r)
    assert _relF(B, ref) <= TOL[mode]


@pytest.mark.parametrize("split", [1, 3, 7])
def test_sketch_split_k_and_determinism(split):
    sk = _sk()
    A = synth.uniform(3, 700, 3000)
    s = sk.Sketch(SEED, "gaussian", 3000, 64, split_k=split, mode="tf32")
    Ad = _dev(A)
    B1 = s.apply(Ad)
    B2 = s.apply(Ad)
    assert torch.equal(B1, B2)  # fixed-order reductions: bit-identical reruns
    assert _relF(B1.cpu().numpy(), oracle.sketch(SEED, "gaussian", A, 64)) <= 5e-3


@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
@pytest.mark.parametrize("split", [1, 4])
def test_sketch_integer_exact(mode, split):
    sk = _sk()
    A = synth.int_matrix(5, 777, 1500, -4, 4)
    s = sk.Sketch(SEED, "rademacher", 1500, 80, mode=mode, split_k=split)
    B = s.apply(_dev(A)).cpu().numpy()
    assert np.array_equal(B.astype(np.float64), oracle.sketch(SEED, "rademacher", A, 80))


def test_sketch_identity_reproduces_omega():
    sk = _sk()
    n = 256
    s = sk.Sketch(SEED, "rademacher", n, 32)
    B = s.apply(_dev(np.eye(n, dtype=np.float32))).cpu().numpy()
    assert np.array_equal(B, oracle.omega(SEED, "rademacher", 0, n, 0, 32))


@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
@pytest.mark.parametrize("k0", [0, 1, 100, 128, 333])
def test_apply_block_offsets(k0, mode):
    sk = _sk()
    n2 = 2000
    A = synth.uniform(9, 300, 700)
    s = sk.Sketch(SEED, "gaussian", n2, 40, mode=mode)
    Bp = s.apply_block(_dev(A), k0).cpu().numpy()
    ref = oracle.sketch(SEED, "gaussian", A, 40, k0=k0)
    assert _relF(Bp, ref) <= TOL[mode]
    si = sk.Sketch(SEED, "rademacher", n2, 40, mode=mode)
    Ai = synth.int_matrix(9, 300, 700)
    assert np.array_equal(si.apply_block(_dev(Ai), k0).cpu().numpy().astype(np.float64),
                          oracle.sketch(SEED, "rademacher", Ai, 40, k0=k0))


def test_lda_padding_and_strided_out():
    sk = _sk()
    A = synth.uniform(4, 200, 516)
    Ad = _dev(A)[:, :500]  # lda = 516 > n2 = 500
    s = sk.Sketch(SEED, "gaussian", 500, 24)
    out = torch.zeros((200, 40), device="cuda")[:, 3:27]  # ldb = 40, offset output
    s.apply(Ad, out=out)
    assert _relF(out.cpu().numpy(), oracle.sketch(SEED, "gaussian", A[:, :500], 24)) <= 5e-3


# ----------------------------------------------------------------------------- C = Omega^T B
@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
@pytest.mark.parametrize("n,r", [(512, 16), (1000, 64), (777, 100), (2048, 256)])
def test_nystrom_core_parity(n, r, mode):
    sk = _sk()
    A = synth.symmetric_uniform(6, n)
    s = sk.Sketch(SEED, "gaussian", n, r, mode=mode)
    B, C = s.nystrom_core(_dev(A))
    Bref, Cref = oracle.nystrom_core(SEED, "gaussian", A, r)
    assert _relF(B.cpu().numpy(), Bref) <= TOL[mode]
    assert _relF(C.cpu().numpy(), Cref) <= TOL[mode]
    # C against the oracle core applied to the GPU's own B isolates the core GEMM
    Cown = oracle.core(SEED, "gaussian", B.cpu().numpy().astype(np.float64))
    assert _relF(C.cpu().numpy(), Cown) <= TOL[mode]


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_c5_shape_four_column_passes_clusters(mode):
    """c5's r = 1024 at a shape that takes clusters of 4 CTA pairs: four 256-column passes of the
    sketch and the tcgen05 core in 16 blocks of 256 x 256, against the oracle on sampled rows and on C."""
    sk = _sk()
    n, r = 4100, 1024
    A = synth.symmetric_uniform(8, n)
    s = sk.Sketch(SEED, "gaussian", n, r, mode=mode)
    B, C = s.nystrom_core(_dev(A))
    rows = np.linspace(0, n - 1, 40).astype(int)
    Bref_rows = oracle.sketch(SEED, "gaussian", A[rows], r)
    assert _relF(B.cpu().numpy()[rows], Bref_rows) <= TOL[mode]
    Cown = oracle.core(SEED, "gaussian", B.cpu().numpy().astype(np.float64))
    assert _relF(C.cpu().numpy(), Cown) <= TOL[mode]


def test_nystrom_core_integer_exact():
    sk = _sk()
    A, X = synth.lowrank_psd(3, 1024, 8, -2, 2)
    s = sk.Sketch(SEED, "rademacher", 1024, 64)
    B, C = s.nystrom_core(_dev(A))
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, 64)
    assert np.array_equal(B.cpu().numpy().astype(np.float64), Bref)
    assert np.array_equal(C.cpu().numpy().astype(np.float64), Cref)
    assert torch.equal(C, C.T)


@pytest.mark.parametrize("core", ["auto", "simt"])
@pytest.mark.parametrize("i0", [0, 5, 130, 4000])
@pytest.mark.parametrize("r", [48, 256, 16, 300, 640])
def test_core_block(i0, r, core):
    sk = _sk()
    Bm = synth.uniform(8, 5000, r).astype(np.float32)
    s = sk.Sketch(SEED, "gaussian", 10000, r, core=core, mode="tf32")
    Cp = s.core_block(_dev(Bm), i0).cpu().numpy()
    tol = 1e-5 if core == "simt" else 5e-3  # fp32 FMA vs tf32 operands
    assert _relF(Cp, oracle.core(SEED, "gaussian", Bm.astype(np.float64), i0=i0)) <= tol


@pytest.mark.parametrize("core", ["auto", "simt"])
@pytest.mark.parametrize("i0", [0, 77, 1000])
def test_core_block_integer_exact(i0, core):
    sk = _sk()
    Bm = synth.int_matrix(9, 3000, 64, -16, 16)
    s = sk.Sketch(SEED, "rademacher", 5000, 64, core=core, mode="tf32")
    Cp = s.core_block(_dev(Bm), i0).cpu().numpy()
    assert np.array_equal(Cp.astype(np.float64), oracle.core(SEED, "rademacher", Bm.astype(np.float64), i0=i0))


# ----------------------------------------------------------------------------- errors
def test_error_codes():
    sk = _sk()
    s = sk.Sketch(SEED, "gaussian", 100, 8)
    A = torch.zeros((10, 100), device="cuda")
    with pytest.raises(sk.SketchError) as e:
        s.apply(torch.zeros((10, 99), device="cuda"))
    assert e.value.name == "SK_ERR_SHAPE_MISMATCH"
    lib = sk.load_library()
    Am = torch.zeros((10, 103), device="cuda")[:, 1:101]
    ws = s.workspace(10)
    Bm = torch.empty((10, 8), device="cuda")
    st = lib.sketch_apply(s._h, Am.data_ptr(), 10, 100, 103, Bm.data_ptr(), 8, ws.data_ptr(), ws.numel() * 4, None)
    assert lib.sketch_status_string(st) == b"SK_ERR_ALIGNMENT"
    # the binding realigns such inputs (one copy) instead of failing
    assert s.apply(Am).abs().max().item() == 0.0
    with pytest.raises(sk.SketchError) as e:
        s.generate(0, 4, 5, 8)
    assert e.value.name == "SK_ERR_INVALID_VALUE"
    assert s.apply(A).abs().max().item() == 0.0
    assert s.apply(torch.zeros((0, 100), device="cuda")).shape == (0, 8)


@pytest.mark.parametrize("cg", [1, 2, 4, 6])
@pytest.mark.parametrize("shape", [(1000, 3000, 256), (600, 1000, 48), (2049, 700, 128), (5000, 2000, 256)])
def test_cta_group_variants(cg, shape):
    """Single-CTA tiles, CTA pairs (tcgen05 cta_group::2) and clusters of two / three pairs sharing
    the generated Omega slices (cg=4, n1 >= 1024; cg=6, n1 >= 1536, uneven 8-row-atom shares) agree
    with the oracle in every mode."""
    sk = _sk()
    n1, n2, r = shape
    Ai = synth.int_matrix(11, n1, n2, -4, 4)
    A = synth.uniform(12, n1, n2)
    ref = oracle.sketch(SEED, "gaussian", A, r)
    for mode in ("tf32", "tf32x3", "bf16"):
        si = sk.Sketch(SEED, "rademacher", n2, r, cta_group=cg, mode=mode)
        assert np.array_equal(si.apply(_dev(Ai)).cpu().numpy().astype(np.float64),
                              oracle.sketch(SEED, "rademacher", Ai, r))
        for omega in (("accurate", "fast") if mode != "tf32x3" else ("accurate",)):
            s = sk.Sketch(SEED, "gaussian", n2, r, cta_group=cg, omega=omega, mode=mode)
            assert _relF(s.apply(_dev(A)).cpu().numpy(), ref) <= TOL[mode]


@pytest.mark.parametrize("cg", [0, 1])
def test_tf32x3_long_k_accuracy(cg):
    """fp32-accurate mode at long K (50k): the planner caps K per TMEM accumulator (the tensor core's
    fp32 accumulation truncates, bias ~ 7e-9 x K, tools/acc_test.py) and sums partials in fp32 RN."""
    sk = _sk()
    A = synth.uniform(13, 300, 50000)
    ref = oracle.sketch(SEED, "gaussian", A, 64)
    s = sk.Sketch(SEED, "gaussian", 50000, 64, mode="tf32x3", cta_group=cg)
    assert _relF(s.apply(_dev(A)).cpu().numpy(), ref) <= 1e-5


def test_fast_transform_rejected_in_tf32x3():
    sk = _sk()
    s = sk.Sketch(SEED, "gaussian", 100, 8, mode="tf32x3", omega="fast")
    with pytest.raises(sk.SketchError) as e:
        s.apply(torch.zeros((4, 100), device="cuda"))
    assert e.value.name == "SK_ERR_UNSUPPORTED"


@pytest.mark.parametrize("mode", ["tf32", "bf16", "tf32x3"])
@pytest.mark.parametrize("omega", ["accurate", "fast"])
def test_cluster_sharing_bit_identical(mode, omega):
    """Sharing generated Omega halves between two CTA pairs changes which SM computes a row, not
    the MMA sequence a row sees: B must equal the unshared CTA-pair result bit for bit."""
    if mode == "tf32x3" and omega == "fast":
        pytest.skip("fast transform not allowed in tf32x3")
    sk = _sk()
    A = _dev(synth.uniform(21, 4100, 3000))
    outs = []
    for cg in (2, 4, 6, 8):
        s = sk.Sketch(SEED, "gaussian", 3000, 256, mode=mode, omega=omega, cta_group=cg, split_k=3)
        outs.append(s.apply(A))
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


@pytest.mark.parametrize("block_rows", [0, 100, 333])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_streaming_apply(block_rows, pinned):
    """sketch_apply_host: A in host memory, streamed in row blocks (double-buffered H2D/compute)."""
    sk = _sk()
    A = synth.uniform(31, 1000, 1502)  # lda not a multiple of 4: device staging pads rows
    At = torch.from_numpy(A)
    if pinned:
        At = At.pin_memory()
    s = sk.Sketch(SEED, "gaussian", 1502, 48, mode="tf32")
    B = s.apply_host(At, block_rows=block_rows).numpy()
    assert _relF(B, oracle.sketch(SEED, "gaussian", A, 48)) <= 5e-3
    # identical to the device-resident call (same kernels, same split per block size)
    Bd = s.apply(_dev(A)).cpu().numpy()
    if block_rows == 0:
        assert np.array_equal(B, Bd)


@pytest.mark.parametrize("block_rows", [0, 256, 777])
def test_host_streaming_nystrom_integer_exact(block_rows):
    sk = _sk()
    A, _ = synth.lowrank_psd(5, 2000, 8, -2, 2)
    s = sk.Sketch(SEED, "rademacher", 2000, 64, mode="tf32")
    B, C = s.nystrom_core_host(torch.from_numpy(A).pin_memory(), block_rows=block_rows)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, 64)
    assert np.array_equal(B.numpy().astype(np.float64), Bref)
    assert np.array_equal(C.numpy().astype(np.float64), Cref)


def test_nystrom_reconstruction_exact_rank():
    """f3: rank-20 PSD A, r = 40: B C^+ B^T recovers A (pinv tol 1e-12 PAPER.md:1020);
    the blocked error formula agrees with the explicit reconstruction."""
    sk = _sk()
    from paper_2603_20966_b200 import quality
    A, _ = synth.lowrank_psd(3, 1200, 20)
    Ad = _dev(A)
    s = sk.Sketch(SEED, "gaussian", 1200, 40, mode="tf32x3")
    B, C = s.nystrom_core(Ad)
    err = quality.reconstruction_error(Ad, B, C, block_rows=500)
    W = quality.pinv_sym(C)
    explicit = torch.linalg.norm(Ad.double() - B.double() @ W @ B.double().T) / torch.linalg.norm(Ad.double())
    assert err < 1e-4 and abs(err - float(explicit)) < 1e-6


def test_nystrom_error_decreases_with_rank_gpu():
    sk = _sk()
    from paper_2603_20966_b200 import quality
    Ad = _dev(synth.rbf_kernel(4, 1500, 8))
    errs = []
    for r in (16, 64, 192):
        s = sk.Sketch(SEED, "gaussian", 1500, r, mode="tf32x3")
        B, C = s.nystrom_core(Ad)
        errs.append(quality.reconstruction_error(Ad, B, C))
    assert errs[0] > errs[1] > errs[2]


@pytest.mark.parametrize("core", ["auto", "simt"])
@pytest.mark.parametrize("nb,r", [(1, 128), (7, 128), (64, 128), (100, 128), (300, 512), (520, 520)])
def test_core_block_cols(nb, r, core):
    """Column-block core for the Redist variant: C[:, cols] = Omega^T B[:, cols] (all r rows of C);
    r or nb > 256 take several 256 x 256 blocks of C."""
    sk = _sk()
    Bm = synth.int_matrix(17, 3000, nb, -8, 8)
    s = sk.Sketch(SEED, "rademacher", 5000, r, mode="tf32", core=core)
    Cc = s.core_block_cols(_dev(Bm), 77).cpu().numpy()
    Bpad = np.zeros((3000, r))
    Bpad[:, :nb] = Bm
    ref = oracle.core(SEED, "rademacher", Bpad, i0=77)[:, :nb]
    assert Cc.shape == (r, nb) and np.array_equal(Cc.astype(np.float64), ref)


# ----------------------------------------------------------------------------- stream-K decomposition
@pytest.mark.parametrize("dist,mode", [("gaussian", "bf16"), ("gaussian", "tf32"), ("rademacher", "tf32")])
def test_streamk_matches_oracle(dist, mode, capfd, monkeypatch):
    """A shape whose split-K waves would idle workers runs stream-K (equal K ranges per cluster / pair,
    m-blocks cut into pieces summed in K order): B equals the oracle (exactly in the integer regime)
    and reruns are bit-identical."""
    sk = _sk()
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    n1, n2, r = 6250, 16384, (256 if dist == "gaussian" else 128)
    A = synth.int_matrix(23, n1, n2, -4, 4) if dist == "rademacher" else synth.uniform(23, n1, n2)
    s = sk.Sketch(SEED, dist, n2, r, mode=mode)
    B1 = s.apply(_dev(A))
    B2 = s.apply(_dev(A))
    torch.cuda.synchronize()
    err = capfd.readouterr().err
    plans = [l for l in err.splitlines() if l.startswith("[sketch plan]") and f"n1={n1}" in l]
    assert plans and all("sk_len=0" not in l for l in plans), plans[:2]
    assert torch.equal(B1, B2)
    rows = np.linspace(0, n1 - 1, 32).astype(int)
    ref = oracle.sketch(SEED, dist, A[rows].astype(np.float64), r)
    got = B1.cpu().numpy()[rows]
    if dist == "rademacher":
        assert np.array_equal(got.astype(np.float64), ref)
    else:
        assert _relF(got, ref) <= TOL[mode]


# ----------------------------------------------------------------------------- clusters of 3 CTA pairs
@pytest.mark.parametrize("r", [48, 80, 200, 256])
def test_three_pair_clusters_auto(r, capfd, monkeypatch):
    """bf16 + fast transform at n1 >= 6144 runs clusters of 3 pairs automatically; each pair
    generates an uneven share of the Omega slice (r = 80: 13/13/14 of 40 rows, starting off the
    8-row swizzle atom).  B matches the oracle, and equals the unshared CTA pairs bit for bit (same
    split-K, so the same MMA sequence per row); a ragged last unit (6200 rows) is covered."""
    sk = _sk()
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    n1, n2 = 6200, 1500
    A = synth.uniform(27, n1, n2)
    Ad = _dev(A)
    s = sk.Sketch(SEED, "gaussian", n2, r, mode="bf16", omega="fast", split_k=2)
    B = s.apply(Ad)
    torch.cuda.synchronize()
    err = capfd.readouterr().err
    plans = [l for l in err.splitlines() if l.startswith("[sketch plan]") and f"n1={n1}" in l]
    assert plans and all(" cl=3 " in l for l in plans), plans[:2]
    ref_pairs = sk.Sketch(SEED, "gaussian", n2, r, mode="bf16", omega="fast", split_k=2, cta_group=2).apply(Ad)
    assert torch.equal(B, ref_pairs)
    rows = np.concatenate([np.arange(0, 40), np.linspace(40, n1 - 1, 40).astype(int), np.arange(n1 - 30, n1)])
    ref = oracle.sketch(SEED, "gaussian", A[rows].astype(np.float64), r)
    assert _relF(B.cpu().numpy()[rows], ref) <= TOL["bf16"]


@pytest.mark.parametrize("k0", [1, 333, 25000])
def test_three_pair_clusters_block_offsets(k0, capfd, monkeypatch):
    """The 2D-grid block form on clusters of 3 pairs (bf16 / fast, n1 >= 6144): a block of A whose
    column 0 is Omega row k0 (unaligned k0 makes every 4-row Philox chunk straddle two calls) matches
    the oracle on sampled rows and equals the unshared pairs bit for bit."""
    sk = _sk()
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    n1, k, r = 6400, 900, 256
    A = synth.uniform(29, n1, k)
    Ad = _dev(A)
    s = sk.Sketch(SEED, "gaussian", 40000, r, mode="bf16", omega="fast", split_k=1)
    Bp = s.apply_block(Ad, k0)
    torch.cuda.synchronize()
    plans = [l for l in capfd.readouterr().err.splitlines() if l.startswith("[sketch plan]") and f"n1={n1}" in l]
    assert plans and all(" cl=3 " in l for l in plans), plans[:2]
    ref_pairs = sk.Sketch(SEED, "gaussian", 40000, r, mode="bf16", omega="fast", split_k=1,
                          cta_group=2).apply_block(Ad, k0)
    assert torch.equal(Bp, ref_pairs)
    rows = np.concatenate([np.arange(0, 16), np.linspace(16, n1 - 1, 32).astype(int)])
    ref = oracle.sketch(SEED, "gaussian", A[rows], r, k0=k0)
    assert _relF(Bp.cpu().numpy()[rows], ref) <= TOL["bf16"]


# ----------------------------------------------------------------------------- in-GEMM Omega, elementwise
def _tf32_rna(x):
    """fp32 -> tf32 round-to-nearest, ties away from zero (cvt.rna.tf32.f32; reading R7)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)


def _bf16_rne(x):
    """fp32 -> bf16 round-to-nearest-even (reading R8)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("dist", ["gaussian", "uniform"])
@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
def test_identity_exposes_in_gemm_omega(dist, mode):
    """A = I makes B the Omega tiles the GEMM generated and multiplied, element by element:
    tf32: B == RNA_tf32(omega) exactly; bf16: B == RNE_bf16(omega) exactly; tf32x3 (Omega_hi + Omega_lo):
    within 4 ulp of the fp32 omega -- with omega from the oracle, so the Philox counters, the Box-Muller /
    uniform transform, the row/column mapping, the swizzled tile layout and the cluster sharing of the
    slices are all checked (n = 2100 takes clusters of 4 CTA pairs in tf32 / bf16; r = 300 two passes)."""
    sk = _sk()
    n, r = 2100, 300
    s = sk.Sketch(SEED, dist, n, r, mode=mode)
    B = s.apply(_dev(np.eye(n, dtype=np.float32))).cpu().numpy()
    om = oracle.omega(SEED, dist, 0, n, 0, r).astype(np.float32)
    if mode == "tf32x3":
        assert _ulp(B, om).max() <= 4
    else:
        rnd = _tf32_rna if mode == "tf32" else _bf16_rne
        if dist == "uniform":
            assert np.array_equal(B, rnd(om))  # uniforms are bit-exact, so their rounding is too
        else:
            # Gaussians: device value within 2 ulp, then rounded -> equal, or one rounding step apart
            step = 2.0 ** (-10 if mode == "tf32" else -7)
            err = np.abs(B.astype(np.float64) - rnd(om)) / np.maximum(np.abs(om), 2.0 ** -30)
            assert np.mean(B == rnd(om)) > 0.999
            assert err.max() <= step


@pytest.mark.parametrize("mode", ["tf32", "tf32x3", "bf16"])
def test_uniform_omega_sketch_and_core(mode):
    """The paper's experimental Omega is uniform Philox: B and C through the GEMMs, on
    an RBF kernel matrix as in the paper's experiments."""
    sk = _sk()
    n, r = 1500, 96
    A = synth.rbf_kernel(11, n, 64)
    s = sk.Sketch(SEED, "uniform", n, r, mode=mode)
    B, C = s.nystrom_core(_dev(A))
    Bref, Cref = oracle.nystrom_core(SEED, "uniform", A, r)
    assert _relF(B.cpu().numpy(), Bref) <= TOL[mode]
    assert _relF(C.cpu().numpy(), Cref) <= TOL[mode]
    B2 = s.apply(_dev(synth.uniform(12, 700, n))).cpu().numpy()
    assert _relF(B2, oracle.sketch(SEED, "uniform", synth.uniform(12, 700, n), r)) <= TOL[mode]


@pytest.mark.parametrize("mode,omega", [("bf16", "fast"), ("tf32", "accurate")])
def test_c4_shape_sampled_rows(mode, omega):
    """c4's shape class: short-wide A 2048 x 2^19, r = 512 Gaussian (the full c4 has K = 4,000,000),
    in the launch configuration the bench uses (clusters of CTA pairs over all 2048 rows); sampled
    rows of B against the oracle."""
    sk = _sk()
    n1, n2, r = 2048, 1 << 19, 512
    Ad = synth.uniform_device(4, n1, n2)
    s = sk.Sketch(SEED, "gaussian", n2, r, mode=mode, omega=omega)
    B = s.apply(Ad)
    torch.cuda.synchronize()
    rows = [0, 1, 127, 128, 511, 1024, 1500, 2047]
    Bref = oracle.sketch(SEED, "gaussian", Ad[rows].cpu().numpy(), r)
    assert _relF(B[rows].cpu().numpy(), Bref) <= TOL[mode]
    del Ad


@pytest.mark.parametrize("split", [1, 3])
def test_tf32x3_long_k_without_split(split):
    """tf32x3's fp32 accuracy must not depend on the split: K = 20,000 in ONE unit (split_k = 1) runs
    20 TMEM accumulation chunks of <= 1024 K, each promoted into the output in fp32 RN;
    the truncating TMEM accumulation alone would give ~1.4e-4 here."""
    sk = _sk()
    n1, n2, r = 640, 20000, 64
    A = synth.uniform(13, n1, n2)
    s = sk.Sketch(SEED, "gaussian", n2, r, mode="tf32x3", split_k=split)
    B = s.apply(_dev(A)).cpu().numpy()
    assert _relF(B, oracle.sketch(SEED, "gaussian", A, r)) <= 1e-5


@pytest.mark.parametrize("n1", [700, 1100, 2048])
@pytest.mark.parametrize("mode,omega", [("bf16", "fast"), ("tf32", "accurate"), ("bf16", "accurate")])
def test_wide_r_single_pass(n1, mode, omega):
    """256 < r <= 512 in ONE pass over A (two N = 256 Omega column blocks per CTA; clusters of 4 pairs
    for n1 <= 1024, of 8 pairs = 16 CTAs above): Gaussian and uniform Omega against the oracle."""
    sk = _sk()
    n2, r = 3000, 400
    A = synth.uniform(14, n1, n2)
    for dist in ("gaussian", "uniform"):
        if dist == "uniform" and omega == "fast":
            continue
        s = sk.Sketch(SEED, dist, n2, r, mode=mode, omega=omega)
        B = s.apply(_dev(A)).cpu().numpy()
        assert _relF(B, oracle.sketch(SEED, dist, A, r)) <= TOL[mode], dist


@pytest.mark.parametrize("mode,omega", [("bf16", "fast"), ("tf32", "accurate")])
def test_streamk_inplace_pieces(mode, omega, capfd, monkeypatch):
    """The 8-GPU per-rank shape of c2 (12,500 x 25,000): stream-K pieces of each m-block accumulated in
    place into B in descending piece order (no partials, no reduce kernel) -- sampled rows against the
    oracle, bit-identical reruns, and the same B as the partials + reduce path (SK_INPLACE=0) within
    fp32 rounding."""
    sk = _sk()
    n1, n2, r = 12500, 25000, 256
    Ad = synth.uniform_device(21, n1, n2)
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    s = sk.Sketch(SEED, "gaussian", n2, r, mode=mode, omega=omega)
    B1 = s.apply(Ad)
    B2 = s.apply(Ad)
    torch.cuda.synchronize()
    plan = capfd.readouterr().err
    if mode == "bf16":  # measured plan at this shape (profiles/r2_share_cluster_sweep.txt): stream-K
        assert "sk_len=0 " not in [l for l in plan.splitlines() if "sketch plan" in l][-1], plan
    assert torch.equal(B1, B2)
    rows = [0, 1, 1535, 1536, 6000, 12287, 12499]
    Bref = oracle.sketch(SEED, "gaussian", Ad[rows].cpu().numpy(), r)
    assert _relF(B1[rows].cpu().numpy(), Bref) <= TOL[mode]
    monkeypatch.setenv("SK_INPLACE", "0")
    B3 = sk.Sketch(SEED, "gaussian", n2, r, mode=mode, omega=omega).apply(Ad)
    assert _relF(B1.cpu().numpy(), B3.double().cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("mode,omega,n1", [("bf16", "fast", 6250), ("tf32", "accurate", 6250), ("bf16", "fast", 2100)])
def test_ragged_row_remainder(mode, omega, n1):
    """n1 = whole cluster units + a small remainder (6250 = 4 x 1536 + 106; 2100 = 2048 + 52): the last
    cluster unit is mostly empty rows (TMA zero fill, rows >= n1 never stored); every row against the
    oracle (Gaussian, relF), and bit-exact in the integer regime."""
    sk = _sk()
    n2, r = 3000, 256
    A = synth.uniform(23, n1, n2)
    B = sk.Sketch(SEED, "gaussian", n2, r, mode=mode, omega=omega).apply(_dev(A)).cpu().numpy()
    assert _relF(B, oracle.sketch(SEED, "gaussian", A, r)) <= TOL[mode]
    Ai = synth.int_matrix(24, n1, n2)
    Bi = sk.Sketch(SEED, "rademacher", n2, r, mode=mode).apply(_dev(Ai)).cpu().numpy()
    assert np.array_equal(Bi.astype(np.float64), oracle.sketch(SEED, "rademacher", Ai, r))


@pytest.mark.timeout(300)
def test_concurrent_inplace_launches_two_streams():
    """Two in-place (stream-K / split-K, waiting pieces) sketch launches in flight at once on one GPU from
    two streams and two threads: the launches are cooperative, so neither can hold SMs the other's
    waiting CTAs need; both results equal the serial ones bit for bit."""
    import threading
    sk = _sk()
    n1, n2, r = 12500, 25000, 256
    A1 = synth.uniform_device(31, n1, n2)
    A2 = synth.uniform_device(32, n1, n2)
    s1 = sk.Sketch(SEED, "gaussian", n2, r, mode="bf16", omega="fast")
    s2 = sk.Sketch(SEED + 1, "gaussian", n2, r, mode="bf16", omega="fast")
    ref1, ref2 = s1.apply(A1), s2.apply(A2)
    torch.cuda.synchronize()
    outs = [None, None]

    def run(i, s, A):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            B = None
            for _ in range(20):
                B = s.apply(A)
            st.synchronize()
        outs[i] = B

    ts = [threading.Thread(target=run, args=(0, s1, A1)), threading.Thread(target=run, args=(1, s2, A2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(240)
    assert not any(t.is_alive() for t in ts)
    assert torch.equal(outs[0], ref1) and torch.equal(outs[1], ref2)


@pytest.mark.parametrize("mode", ["tf32", "bf16", "tf32x3"])
def test_three_column_passes_with_pieces(mode):
    """r = 600 (three 256-column passes, none a 512-column pair) on a shape the planner splits into
    pieces: every pass accumulates its pieces (in place or through partials) into its own columns of B;
    integer regime bit-exact, Gaussian within tolerance."""
    sk = _sk()
    n1, n2, r = 1500, 9000, 600
    Ai = synth.int_matrix(41, n1, n2)
    Bi = sk.Sketch(SEED, "rademacher", n2, r, mode=mode).apply(_dev(Ai)).cpu().numpy()
    assert np.array_equal(Bi.astype(np.float64), oracle.sketch(SEED, "rademacher", Ai, r))
    A = synth.uniform(42, n1, n2)
    B = sk.Sketch(SEED, "gaussian", n2, r, mode=mode).apply(_dev(A)).cpu().numpy()
    assert _relF(B, oracle.sketch(SEED, "gaussian", A, r)) <= TOL[mode]


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_fast_transform_clusters_of_three(mode, capfd, monkeypatch):
    """With the fast transform, tf32 and bf16 both take clusters of 3 CTA pairs (uneven 42/43/43-row
    shares of each Omega slice) at n1 >= 6144: against the oracle."""
    sk = _sk()
    monkeypatch.setenv("SK_DEBUG_PLAN", "1")
    n1, n2, r = 6200, 2000, 256
    A = synth.uniform(51, n1, n2)
    B = sk.Sketch(SEED, "gaussian", n2, r, mode=mode, omega="fast").apply(_dev(A)).cpu().numpy()
    plan = [l for l in capfd.readouterr().err.splitlines() if "sketch plan" in l]
    assert plan and " cl=3 " in plan[-1], plan
    assert _relF(B, oracle.sketch(SEED, "gaussian", A, r)) <= TOL[mode]


@pytest.mark.parametrize("mode", ["bf16", "tf32x3"])
@pytest.mark.parametrize("m", [1, 200, 3000, 6250, 9000, 25000])
def test_core_block_offsets_fit_queried_workspace(m, mode):
    """The core plan is chosen per span (i0 % 128 widens it by up to 127 rows): with exactly the
    workspace sketch_workspace_size reports for m rows, every block offset runs, and C matches the
    oracle core (Alg. 2)."""
    sk = _sk()
    r = 256
    Bm = synth.uniform(11, m, r)
    s = sk.Sketch(SEED, "gaussian", 10**6, r, mode=mode)
    Bd = _dev(Bm)
    for i0 in (0, 1, 63, 64, 127, 128, 12345):
        C = s.core_block(Bd, i0).cpu().numpy()
        assert _relF(C, oracle.core(SEED, "gaussian", Bm.astype(np.float64), i0=i0)) <= TOL[mode], i0
