"""Every multi-GPU layout on ONE GPU through "virtual ranks" (SURVEY §4.2 fake backend).

`dist.run_virtual(P, fn)` runs P ranks as threads of this process, each on its own CUDA stream of
cuda:0, with a `VirtualComm` in place of the NCCL process group: every rank's block goes through the
real library calls (`sketch_apply_block`, `sketch_apply_block_rs` with the epilogue storing into the
other ranks' receive slots, `sketch_reduce_slots`, `core_apply_block`, `core_apply_block_cols`,
`sketch_pack_cols`), and the reductions are the library's fixed-order `sketch_sum_peers` kernel over
same-device pointers.  The results are compared with the fp64 oracle of the WHOLE problem:
bit-exact in the integer regime (integer A, +-1 Omega: every partial sum is exact in fp32), within
the north-star tolerance for Gaussian Omega.  Alg. 1, Alg. 2 No-Redist
(C by AllReduce PAPER.md:1836-1839) and Redist.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import synth

pytestmark = pytest.mark.gpu

SEED = 42


def _run(world, spec, n1, n2, r, dist, mode, A, rs="nccl", fused_ar=False, variant="noredist", steps=2,
         omega="accurate"):
    import paper_2603_20966_b200 as sk
    from paper_2603_20966_b200.dist import DistSketch, Layout, run_virtual

    def body(comm):
        layout = Layout.parse(spec, world)
        local = sk.Sketch(SEED, dist, n2, r, mode=mode, omega=omega)
        ds = DistSketch(SEED, dist, n1, n2, r, layout, local=local, fused_rs=rs, fused_ar=fused_ar, comm=comm)
        r0, r1, c0, c1 = ds.a_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).cuda()
        outs = []
        for _ in range(steps):  # repeated steps reuse (and alternate) the receive slots
            if n1 == n2:
                if variant == "redist":
                    Bp, (a, b), C = ds.nystrom_core_redist(Ablk)
                else:
                    Bp, (a, b), C = ds.nystrom_core(Ablk)
                Cn = C.cpu().numpy()
            else:
                Bp, (a, b) = ds.apply(Ablk)
                Cn = None
            torch.cuda.current_stream().synchronize()
            outs.append((a, b, Bp.cpu().numpy(), Cn))
        return {"outs": outs, "comm": ds.comm_bytes // steps, "rs_mode": ds.rs_mode, "fused_ar": ds.fused_ar,
                "fallbacks": list(ds.fallbacks)}

    torch.cuda.set_device(0)
    return run_virtual(world, body)


def _check_exact(res, Bref, Cref, n1):
    covered = np.zeros(n1, dtype=int)
    for rk in res:
        first = rk["outs"][0]
        for a, b, Bp, C in rk["outs"]:
            assert (a, b) == first[:2]
            assert np.array_equal(Bp.astype(np.float64), Bref[a:b]), (a, b)
            if Cref is not None:
                assert np.array_equal(C.astype(np.float64), Cref)
        covered[first[0]:first[1]] += 1
    assert np.all(covered == 1)  # the B pieces partition the rows exactly once


LAYOUTS = [(2, "row"), (2, "col"), (4, "row"), (4, "col"), (4, "2x2"), (8, "4x2"), (8, "2x4"), (8, "row")]


@pytest.mark.parametrize("world,spec", LAYOUTS)
@pytest.mark.parametrize("rs", ["nccl", "peer", "epilogue"])
def test_virtual_layouts_nystrom_exact(world, spec, rs):
    """Alg. 2 No-Redist on every grid, every reduce-scatter of partial B, fused (peer-sum) AllReduce
    of C: bit-exact B pieces and C against the oracle; bytes as Alg. 1's cost for the NCCL-style
    exchange."""
    from paper_2603_20966_b200.dist import Layout, predicted_bytes_per_rank
    if rs != "nccl" and Layout.parse(spec, world).p2 == 1:
        pytest.skip("no reduce-scatter in the row-block layout")
    n, r = 1120, 48  # n / p1 divisible by p2 on every grid: no padded rows in the exchanged pieces
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    res = _run(world, spec, n, n, r, "rademacher", "tf32", A, rs=rs, fused_ar=True)
    _check_exact(res, Bref, Cref, n)
    for rk in res:
        assert rk["rs_mode"] == rs and rk["fused_ar"] and not rk["fallbacks"]  # no silent fallback
        if rs in ("nccl", "peer"):
            assert rk["comm"] == predicted_bytes_per_rank(n, r, Layout.parse(spec, world), True)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["tf32", "bf16", "tf32x3"])
def test_virtual_redist_exact(world, mode):
    """Redist (All-to-All of B packed by `sketch_pack_cols`, column blocks of C regenerating Omega for
    all n rows, all-gather of C): the same exact B and C as the oracle, predicted bytes."""
    from paper_2603_20966_b200.dist import Layout, predicted_bytes_per_rank
    n, r = 1200, 48
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    res = _run(world, "row", n, n, r, "rademacher", mode, A, variant="redist")
    _check_exact(res, Bref, Cref, n)
    pred = predicted_bytes_per_rank(n, r, Layout(world, 1), True, "redist")
    assert all(rk["comm"] == pred for rk in res)


@pytest.mark.parametrize("world,spec", [(2, "col"), (4, "2x2"), (8, "4x2")])
def test_virtual_sketch_colblock_rectangular(world, spec):
    """Alg. 1 alone on a rectangular A with ragged blocks (B pieces only), epilogue reduce-scatter."""
    n1, n2, r = 1000, 2900, 40
    A = synth.int_matrix(3, n1, n2, -4, 4)
    Bref = oracle.sketch(SEED, "rademacher", A, r)
    res = _run(world, spec, n1, n2, r, "rademacher", "tf32", A, rs="epilogue")
    _check_exact(res, Bref, None, n1)


@pytest.mark.parametrize("world,spec,variant", [(4, "2x2", "noredist"), (4, "row", "redist"),
                                                (8, "4x2", "noredist")])
def test_virtual_gaussian_tf32x3_tolerance(world, spec, variant):
    """Gaussian Omega, fp32-accurate mode, on a float A: relF(B), relF(C) <= 1e-5 (north star)."""
    n, r = 1536, 64
    A = synth.symmetric_uniform(1, n)
    Bref, Cref = oracle.nystrom_core(SEED, "gaussian", A, r)
    res = _run(world, spec, n, n, r, "gaussian", "tf32x3", A, rs="peer", fused_ar=True, variant=variant, steps=1)
    B = np.zeros_like(Bref)
    for rk in res:
        a, b, Bp, C = rk["outs"][0]
        B[a:b] = Bp
        assert np.linalg.norm(C - Cref) / np.linalg.norm(Cref) <= 1e-5
    assert np.linalg.norm(B - Bref) / np.linalg.norm(Bref) <= 1e-5
    # C is replicated: every rank holds the same bits
    for rk in res[1:]:
        assert np.array_equal(rk["outs"][0][3], res[0]["outs"][0][3])


@pytest.mark.parametrize("world,spec", [(2, "col"), (4, "2x2")])
def test_virtual_epilogue_rs_tf32x3(world, spec):
    """tf32x3 with the reduce-scatter fused into the sketch epilogue: the promoted TMEM chunks are
    stored / added (ordered L2 reductions) straight into the owners' receive slots; exact in the
    integer regime, and K = 4,000 per rank spans several 1024-K chunks."""
    n1, n2, r = 900, 8000, 40
    A = synth.int_matrix(5, n1, n2, -4, 4)
    Bref = oracle.sketch(SEED, "rademacher", A, r)
    res = _run(world, spec, n1, n2, r, "rademacher", "tf32x3", A, rs="epilogue")
    _check_exact(res, Bref, None, n1)


@pytest.mark.parametrize("world,mode", [(2, "tf32"), (4, "bf16"), (8, "tf32")])
def test_virtual_balanced_rowblock_exact(world, mode):
    """Row-block cut at whole units of the library's own plan (Sketch.plan_info), the ragged tail split
    by columns and reduced onto the last rank through symmetric memory (real kernels): exact B and C."""
    import paper_2603_20966_b200 as sk
    from paper_2603_20966_b200.dist import DistSketch, Layout, run_virtual
    n, r = 4400, 48  # units of 512 rows (pairs, 2 accumulators): 2048 / 1024 / 512 rows per rank + 304 tail
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    torch.cuda.set_device(0)

    def body(comm):
        local = sk.Sketch(SEED, "rademacher", n, r, mode=mode)
        unit = local.plan_info(-(-n // world), n)["rows_per_unit"]
        ds = DistSketch(SEED, "rademacher", n, n, r, Layout.parse("row", world), local=local, fused_ar=True,
                        comm=comm, balance_unit=unit)
        r0, r1, c0, c1 = ds.a_block_range()
        t = ds.tail_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).cuda()
        At = torch.from_numpy(np.ascontiguousarray(A[t[0]:t[1], t[2]:t[3]])).cuda() if t else None
        outs = []
        for _ in range(3):
            Bp, (a, b), C = ds.nystrom_core(Ablk, At)
            torch.cuda.current_stream().synchronize()
            outs.append((a, b, Bp.cpu().numpy(), C.cpu().numpy()))
        return {"outs": outs, "tail": ds.tail is not None, "fallbacks": list(ds.fallbacks)}

    res = run_virtual(world, body)
    assert all(rk["tail"] for rk in res) and not any(rk["fallbacks"] for rk in res)
    _check_exact(res, Bref, Cref, n)
