"""CPU tests of the multi-GPU layouts (paper_2603_20966_b200/dist.py) with gloo process groups.

The per-rank compute is injected: an oracle-backed CPU stand-in (test infrastructure) replaces the
CUDA library so that partitioning, global Omega offsets, the reduce-scatter of partial B, the
AllReduce of C and the communication accounting (Alg. 1 cost) are checked on CPU.
The CUDA path of the same layer runs in bench.py under torchrun on the GPU box.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
from inputs import synth
from paper_2603_20966_b200.dist import DistSketch, Layout, balanced_split, predicted_bytes_per_rank

SEED = 42


class OracleLocal:
    """CPU stand-in for paper_2603_20966_b200.Sketch's block entry points (tests only)."""

    def __init__(self, seed, dist, r):
        self.seed, self.dist, self.r = seed, dist, r

    def apply_block(self, A_blk, k0, out=None):
        B = torch.from_numpy(oracle.sketch(self.seed, self.dist, A_blk.numpy(), self.r, k0=k0).astype(np.float32))
        if out is None:
            return B
        out.copy_(B)
        return out

    def core_block_cols(self, B_blk, i0, out=None):
        # C[:, cols] = Omega[i0:i0+m, :r]^T B_blk (nb columns): the oracle core on a zero-padded B
        m, nb = B_blk.shape
        Bpad = np.zeros((m, self.r), dtype=np.float64)
        Bpad[:, :nb] = B_blk.numpy()
        C = torch.from_numpy(oracle.core(self.seed, self.dist, Bpad, i0=i0)[:, :nb].astype(np.float32))
        if out is None:
            return C
        out.copy_(C)
        return out

    @staticmethod
    def pack_cols(B_blk, cb):
        return torch.cat([B_blk[:, cb[j]:cb[j + 1]].reshape(-1) for j in range(len(cb) - 1)])

    def core_block(self, B_blk, i0):
        return torch.from_numpy(oracle.core(self.seed, self.dist, B_blk.numpy().astype(np.float64), i0=i0).astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, n1, n2, r, dist, nystrom, q, variant="noredist"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layout = Layout.parse(spec, world)
        A = synth.int_matrix(7, n1, n2, -4, 4, symmetric=(n1 == n2))
        ds = DistSketch(SEED, dist, n1, n2, r, layout, local=OracleLocal(SEED, dist, r), col_align=128)
        r0, r1, c0, c1 = ds.a_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1]))
        if nystrom:
            Bp, (a, b), C = ds.nystrom_core_redist(Ablk) if variant == "redist" else ds.nystrom_core(Ablk)
            q.put((rank, a, b, Bp.numpy(), C.numpy(), ds.comm_bytes))
        else:
            Bp, (a, b) = ds.apply(Ablk)
            q.put((rank, a, b, Bp.numpy(), None, ds.comm_bytes))
    finally:
        tdist.destroy_process_group()


def _run(world, spec, n1, n2, r, dist, nystrom, variant="noredist"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, spec, n1, n2, r, dist, nystrom, q, variant))
             for i in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=90) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


@pytest.mark.parametrize("world,spec", [(2, "row"), (2, "col"), (4, "2x2"), (4, "row"), (4, "col")])
def test_layouts_reproduce_global_product(world, spec):
    n1 = n2 = 520
    r = 24
    res = _run(world, spec, n1, n2, r, "rademacher", True)
    A = synth.int_matrix(7, n1, n2, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    covered = np.zeros(n1, dtype=int)
    for rank, a, b, Bp, C, comm in res:
        # integer regime: every rank's B piece and the all-reduced C are exact
        assert np.array_equal(Bp.astype(np.float64), Bref[a:b])
        assert np.array_equal(C.astype(np.float64), Cref)
        covered[a:b] += 1
        layout = Layout.parse(spec, world)
        assert comm == predicted_bytes_per_rank(n1, r, layout, True)
    assert np.all(covered == 1)  # B pieces partition the rows exactly once


def test_rowblock_needs_no_b_communication():
    # Thm 4.2 case P <= n1: the row-block layout moves zero words for B
    res = _run(2, "row", 300, 700, 16, "gaussian", False)
    for rank, a, b, Bp, C, comm in res:
        assert comm == 0
    assert predicted_bytes_per_rank(300, 16, Layout(2, 1), False) == 0


def test_colblock_reduce_scatter_matches_alg1_cost():
    n1, n2, r = 256, 900, 32
    res = _run(2, "col", n1, n2, r, "gaussian", False)
    A = synth.int_matrix(7, n1, n2, -4, 4)
    Bref = oracle.sketch(SEED, "gaussian", A, r)
    for rank, a, b, Bp, C, comm in res:
        np.testing.assert_allclose(Bp, Bref[a:b], rtol=1e-6, atol=1e-4)
        # (1 - 1/p2) n1 r / p1 words of fp32 (p3 = 1)
        assert comm == predicted_bytes_per_rank(n1, r, Layout(1, 2), False) == 4 * (n1 * r // 2)


def test_balanced_split_alignment():
    b = balanced_split(50000, 4, 128)
    assert b[0] == 0 and b[-1] == 50000 and all(x % 128 == 0 for x in b[1:-1])
    assert max(b[i + 1] - b[i] for i in range(4)) - min(b[i + 1] - b[i] for i in range(4)) <= 128
    assert balanced_split(10, 3) == [0, 3, 6, 10]


@pytest.mark.parametrize("world", [2, 4])
def test_redist_variant_matches_noredist(world):
    """Redist (All-to-All of B, column blocks of C) returns the same exact B and C as
    the No-Redist variant in the integer regime, with the predicted All-to-All + all-gather bytes."""
    n, r = 520, 24
    res = _run(world, "row", n, n, r, "rademacher", True, "redist")
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    for rank, a, b, Bp, C, comm in res:
        assert np.array_equal(Bp.astype(np.float64), Bref[a:b])
        assert np.array_equal(C.astype(np.float64), Cref)
        pred = predicted_bytes_per_rank(n, r, Layout(world, 1), True, "redist")
        assert comm == pred


@pytest.mark.parametrize("world,spec,variant", [(2, "col", "noredist"), (4, "2x2", "noredist"),
                                                (8, "4x2", "noredist"), (4, "row", "redist")])
def test_virtual_comm_matches_oracle(world, spec, variant):
    """The single-process virtual-rank backend (VirtualComm) on CPU: same exact B pieces and
    C as the oracle of the whole problem, and the same byte accounting as the gloo process groups."""
    from paper_2603_20966_b200.dist import run_virtual
    n, r = 520, 24
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    layout = Layout.parse(spec, world)

    def body(comm):
        ds = DistSketch(SEED, "rademacher", n, n, r, layout, local=OracleLocal(SEED, "rademacher", r), comm=comm)
        r0, r1, c0, c1 = ds.a_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1]))
        Bp, (a, b), C = ds.nystrom_core_redist(Ablk) if variant == "redist" else ds.nystrom_core(Ablk)
        return a, b, Bp.numpy(), C.numpy(), ds.comm_bytes

    covered = np.zeros(n, dtype=int)
    for a, b, Bp, C, comm in run_virtual(world, body):
        assert np.array_equal(Bp.astype(np.float64), Bref[a:b])
        assert np.array_equal(C.astype(np.float64), Cref)
        assert comm == predicted_bytes_per_rank(n, r, layout, True, variant)
        covered[a:b] += 1
    assert np.all(covered == 1)


@pytest.mark.parametrize("world,unit,variant", [(2, 128, "noredist"), (4, 128, "noredist"), (4, 64, "redist"),
                                                (8, 32, "noredist")])
def test_balanced_rowblock_matches_oracle(world, unit, variant):
    """Row-block cut at whole units with the ragged tail split by columns and reduced onto the last rank
    (virtual ranks, oracle stand-in): B pieces partition the rows, B and C exact in the integer regime,
    bytes = the tail partial (+ r^2 for C, or the Redist exchange)."""
    from paper_2603_20966_b200.dist import run_virtual
    n, r = 1120, 24
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    layout = Layout.parse("row", world)

    def body(comm):
        ds = DistSketch(SEED, "rademacher", n, n, r, layout, local=OracleLocal(SEED, "rademacher", r), comm=comm,
                        balance_unit=unit)
        assert ds.tail is not None
        r0, r1, c0, c1 = ds.a_block_range()
        t0, t1, tc0, tc1 = ds.tail_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1]))
        At = torch.from_numpy(np.ascontiguousarray(A[t0:t1, tc0:tc1]))
        f = ds.nystrom_core_redist if variant == "redist" else ds.nystrom_core
        Bp, (a, b), C = f(Ablk, At)
        return a, b, Bp.numpy(), C.numpy(), ds.comm_bytes, ds.tail["R"]

    covered = np.zeros(n, dtype=int)
    for a, b, Bp, C, comm, R in run_virtual(world, body):
        assert np.array_equal(Bp.astype(np.float64), Bref[a:b])
        assert np.array_equal(C.astype(np.float64), Cref)
        if variant == "noredist":
            assert comm == predicted_bytes_per_rank(n, r, layout, True, tail_rows=R)
        covered[a:b] += 1
    assert np.all(covered == 1)
