"""Multi-GPU layouts on real GPUs (needs >= 2 CUDA devices; skipped otherwise).

The fused reduce-scatters (partial B stored from the GEMM epilogue into the owners'
symmetric-memory receive slots over NVLink, or written locally and summed by the owners with NVLink
peer reads; both fixed-order) must return exactly the B pieces of the NCCL reduce_scatter path in the integer regime (integer A, Rademacher Omega: every
partial sum is exact in fp32), and those must equal the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch

SEED = 42


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, n1, n2, r, q):
    import torch.distributed as tdist
    import paper_2603_20966_b200 as sk
    from inputs import synth
    from paper_2603_20966_b200.dist import DistSketch, Layout
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        layout = Layout.parse(spec, world)
        A = synth.int_matrix(7, n1, n2, -4, 4)
        out = {}
        for fused in ("nccl", "epilogue", "peer"):
            local = sk.Sketch(SEED, "rademacher", n2, r, mode="tf32")
            ds = DistSketch(SEED, "rademacher", n1, n2, r, layout, local=local, fused_rs=fused)
            r0, r1, c0, c1 = ds.a_block_range()
            Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).to(dev)
            for _ in range(2):  # twice: the second call reuses the receive slots
                Bp, (a, b) = ds.apply(Ablk)
            torch.cuda.synchronize()
            out[fused] = (a, b, Bp.cpu().numpy(), ds.comm_bytes, ds.rs_mode)
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("spec,n1,n2,r", [("col", 3000, 4096, 64), ("col", 2500, 2100, 256)])
def test_fused_reduce_scatter_matches_nccl_and_oracle(spec, n1, n2, r):
    import torch.multiprocessing as mp
    import oracle
    from inputs import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, spec, n1, n2, r, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = synth.int_matrix(7, n1, n2, -4, 4)
    Bref = oracle.sketch(SEED, "rademacher", A, r)
    for rank, out in res:
        a, b, Bn, _, _ = out["nccl"]
        for mode in ("epilogue", "peer"):
            af, bf, Bf, comm, rs_mode = out[mode]
            assert rs_mode == mode  # the symmetric-memory path ran (no silent NCCL fallback)
            assert (a, b) == (af, bf)
            assert np.array_equal(Bn, Bf), mode
            assert np.array_equal(Bf.astype(np.float64), Bref[a:b]), mode
            assert comm > 0


def _worker_ar(rank, world, port, n, r, q):
    import torch.distributed as tdist
    import paper_2603_20966_b200 as sk
    from inputs import synth
    from paper_2603_20966_b200.dist import DistSketch, Layout
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
        out = {}
        for fused in (False, True):
            local = sk.Sketch(SEED, "rademacher", n, r, mode="tf32")
            ds = DistSketch(SEED, "rademacher", n, n, r, Layout.parse("row", world), local=local, fused_ar=fused)
            r0, r1, c0, c1 = ds.a_block_range()
            Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).to(dev)
            for _ in range(3):  # both alternating slots, then the first again
                Bp, (a, b), C = ds.nystrom_core(Ablk)
            torch.cuda.synchronize()
            assert ds.fused_ar == fused  # no silent fallback to NCCL
            out[fused] = C.cpu().numpy()
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_fused_allreduce_of_core_matches_nccl_and_oracle():
    import torch.multiprocessing as mp
    import oracle
    from inputs import synth
    world, n, r = 2, 2100, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ar, args=(i, world, port, n, r, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    _, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    for rank, out in res:
        assert np.array_equal(out[False], out[True])
        assert np.array_equal(out[True].astype(np.float64), Cref)


def _has_multicast(ds):
    ar = getattr(ds, "_ar", None)
    return bool(ar and ar["sb"].multicast_ptr)


def _worker_layouts(rank, world, port, n, r, q):
    """Every Nystrom variant on real GPUs over NCCL + symmetric memory: No-Redist on the row-block and
    (for 4 ranks) 2 x 2 grids with the peer-read reduce-scatter and the fused AllReduce, and Redist."""
    import torch.distributed as tdist
    import paper_2603_20966_b200 as sk
    from inputs import synth
    from paper_2603_20966_b200.dist import DistSketch, Layout
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
        specs = ["row", "col"] + (["2x2"] if world == 4 else [])
        out = {}
        for spec in specs:
            for variant in ("noredist", "redist"):
                if variant == "redist" and spec != "row":
                    continue
                local = sk.Sketch(SEED, "rademacher", n, r, mode="tf32")
                ds = DistSketch(SEED, "rademacher", n, n, r, Layout.parse(spec, world), local=local,
                                fused_rs="peer", fused_ar=True)
                ds.nvls_min_ranks = 2  # exercise the in-switch path on every group that has it
                r0, r1, c0, c1 = ds.a_block_range()
                Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).to(dev)
                for _ in range(2):
                    Bp, (a, b), C = ds.nystrom_core_redist(Ablk) if variant == "redist" else ds.nystrom_core(Ablk)
                torch.cuda.synchronize()
                out[(spec, variant)] = (a, b, Bp.cpu().numpy(), C.cpu().numpy(), ds.rs_mode, ds.fused_ar,
                                        list(ds.fallbacks), ds.reduce_path, _has_multicast(ds))
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("world", [2, 4])
def test_all_variants_nccl_match_oracle(world):
    """Row-block / column-block / 2 x 2 No-Redist (peer-read reduce-scatter, fused AllReduce) and Redist
    (sketch_pack_cols + NCCL All-to-All + column blocks of C): exact B pieces and C against the oracle
    in the integer regime, with the symmetric-memory paths actually taken (no fallback)."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    import oracle
    from inputs import synth
    n, r = 2048, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_layouts, args=(i, world, port, n, r, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    for rank, out in res:
        for (spec, variant), (a, b, Bp, C, rs_mode, fused_ar, fallbacks, path, mc) in out.items():
            assert np.array_equal(Bp.astype(np.float64), Bref[a:b]), (spec, variant)
            assert np.array_equal(C.astype(np.float64), Cref), (spec, variant)
            assert not fallbacks, fallbacks
            if variant == "noredist":
                assert fused_ar
                # the in-switch (NVLS) reduction runs whenever the symmetric buffers have a multicast mapping
                assert path == ("nvls" if mc else "peer"), (path, mc)
                if spec != "row":
                    assert rs_mode == "peer"


def _worker_ar_epi(rank, world, port, n, r, q):
    import torch.distributed as tdist
    import paper_2603_20966_b200 as sk
    from inputs import synth
    from paper_2603_20966_b200.dist import DistSketch, Layout
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
        local = sk.Sketch(SEED, "rademacher", n, r, mode="tf32")
        ds = DistSketch(SEED, "rademacher", n, n, r, Layout.parse("row", world), local=local, fused_ar="epilogue")
        r0, r1, c0, c1 = ds.a_block_range()
        Ablk = torch.from_numpy(np.ascontiguousarray(A[r0:r1, c0:c1])).to(dev)
        Cs = []
        for _ in range(3):
            Bp, (a, b), C = ds.nystrom_core(Ablk)
            Cs.append(C.cpu().numpy())
        torch.cuda.synchronize()
        q.put((rank, Cs, ds.ar_mode, ds.reduce_path))
    finally:
        tdist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_epilogue_allreduce_multicast_matches_oracle():
    """The AllReduce of C issued from the core GEMM's epilogue (multimem.red through the multicast
    mapping): exact against the oracle in the integer regime on every rank, every step."""
    import torch.multiprocessing as mp
    import oracle
    from inputs import synth
    world, n, r = 2, 2100, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ar_epi, args=(i, world, port, n, r, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = synth.int_matrix(7, n, n, -4, 4, symmetric=True)
    _, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    for rank, Cs, mode, path in res:
        if mode != "epilogue":
            pytest.skip("no multicast mapping on this box")
        assert path == "nvls-epilogue"
        for C in Cs:
            assert np.array_equal(C.astype(np.float64), Cref)
