"""Multi-GPU layouts of the sketch and the Nystrom core (one process per GPU, torch.distributed/NCCL).

Implements Alg. 1 (RandMatMul) and the No-Redist variant of Alg. 2
(RandCompNys with Psi = Pi) for processor grids p1 x p2 x 1:

  * rank r <-> grid coordinates (i, j) = (r // p2, r % p2)
  * rank (i, j) owns A_ij = rows R_i x columns K_j of A
  * All-Gather of A is a no-op because p3 = 1
  * GenRandom: every rank regenerates Omega rows K_j itself (inside the kernel)
  * local product B-bar_i = A_ij Omega_Kj
  * Reduce-Scatter of B-bar_i over the row group {(i, *)}: rank (i, j) keeps
    rows piece j of R_i (skipped when p2 = 1: zero communication, Thm. 4.2 / Case 1,
    PAPER.md:350, 438-440)
  * Nystrom: C-bar = Omega^T_{rows} B_piece regenerated for the owned B rows
    then AllReduce of the r x r partials (the GPU variant replaces Reduce-Scatter
    of C by AllReduce; reading R11: full C on every rank).

Redist variant (Case 1 of the first grid-selection approach, p1 = q3 = P,
PAPER.md:665-687, 698): B is computed row-block (zero communication), redistributed by an All-to-All
so that rank k owns column block k of B over all n rows (bandwidth ~ n r / P words),
and rank k computes the column block C[:, cols_k] = Omega^T B[:, cols_k] with Omega regenerated for
all n rows.  The pack of the paper's exchange is the library's `sketch_pack_cols`
kernel; no unpack is needed because the row-major blocks arrive in global row order.  The paper
leaves C distributed; `nystrom_core_redist` all-gathers the column blocks so both variants return
the same replicated C.

Bandwidth accounting: predicted words per rank = (1 - 1/p2) n1 r / p1 for B (Alg. 1 cost,
PAPER.md:427 with p3 = 1) plus the AllReduce payload r^2 for C; measured = bytes handed to
the collectives.  Row splits are balanced; column splits are multiples of 128 (so each block's
Omega rows start on a Philox row-group boundary) except the last.

Communication goes through a `comm` object: `TorchComm` (torch.distributed process group + torch
symmetric memory over NVLink) in production, or `VirtualComm` -- P virtual ranks as threads of ONE
process on ONE device (SURVEY §4.2 "fake backend"): every rank's block runs through the same library
calls, symmetric buffers are plain same-device allocations, and the reductions are the library's own
fixed-order kernels (`sketch_sum_peers`, `sketch_reduce_slots`).  Nothing waits on the device for
another rank's kernel in the virtual mode (the barrier is host-side, after a stream sync).
"""
from __future__ import annotations

import os
import sys
import threading

from dataclasses import dataclass


def balanced_split(n: int, parts: int, align: int = 1) -> list:
    """Boundaries [b_0=0, ..., b_parts=n]; interior boundaries multiples of `align` when possible."""
    if align > 1 and n >= parts * align:
        units = -(-n // align)
        bnd = [min(n, (units * p // parts) * align) for p in range(parts + 1)]
    else:
        bnd = [n * p // parts for p in range(parts + 1)]
    bnd[-1] = n
    return bnd


@dataclass
class Layout:
    p1: int
    p2: int

    @property
    def P(self) -> int:
        return self.p1 * self.p2

    def coords(self, rank: int) -> tuple:
        return rank // self.p2, rank % self.p2

    @staticmethod
    def parse(spec: str, P: int) -> "Layout":
        """'row' -> P x 1, 'col' -> 1 x P, 'AxB' -> A x B (must multiply to P)."""
        if spec in ("row", "rowblock"):
            return Layout(P, 1)
        if spec in ("col", "colblock"):
            return Layout(1, P)
        a, b = (int(t) for t in spec.lower().split("x"))
        if a * b != P:
            raise ValueError(f"layout {spec} does not match world size {P}")
        return Layout(a, b)


def predicted_bytes_per_rank(n1: int, r: int, layout: Layout, nystrom: bool, variant: str = "noredist",
                             tail_rows: int = 0) -> int:
    """Alg. 1 reduce-scatter volume (1 - 1/p2) n1 r / p1 words (+ r^2 AllReduce payload), fp32.
    Redist (row-block only): All-to-All of B, (1 - 1/P) n r / P words sent per rank,
    plus the all-gather that replicates C, (P - 1) r ceil(r / P) words."""
    P = layout.P
    if variant == "redist" and nystrom and P > 1:
        return int(4 * ((n1 * r) // P - (n1 // P) * (r // P) + (P - 1) * r * (-(-r // P)))) if (n1 % P == 0 and r % P == 0) \
            else -1
    words = (1.0 - 1.0 / layout.p2) * n1 * r / layout.p1
    words += tail_rows * r  # balanced row-block: this rank's partial of the tail rows
    if nystrom and P > 1:
        words += r * r
    return int(round(4 * words))


# ============================================================================== communicators
class SymmBuf:
    """A buffer every rank of a group allocated together: `tensor` is this rank's, `ptrs[j]` the
    device address of rank j's (NVLink peer mappings, or same-device addresses for virtual ranks);
    `barrier()` orders every rank's prior writes before any rank's later reads."""

    def __init__(self, tensor, ptrs, barrier, multicast_ptr: int = 0):
        self.tensor, self.ptrs, self._barrier, self.multicast_ptr = tensor, list(ptrs), barrier, multicast_ptr

    def barrier(self):
        self._barrier()


class TorchComm:
    """torch.distributed process group; symmetric buffers from torch symmetric memory (NVLink)."""

    def __init__(self, group=None):
        import torch.distributed as tdist
        self.tdist = tdist
        self.group = group
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)

    def split(self, groups: list) -> "TorchComm":
        """Sub-communicator: `groups` lists the global ranks of every subgroup (all ranks call this with
        the same list); returns the one this rank belongs to."""
        me = self.tdist.get_rank()
        mine = None
        for g in groups:
            pg = self.tdist.new_group(g)
            if me in g:
                mine = pg
        return TorchComm(mine)

    def reduce_scatter(self, out, inp):
        self.tdist.reduce_scatter_tensor(out, inp, group=self.group)

    def all_reduce(self, t, op: str = "sum"):
        rop = {"sum": self.tdist.ReduceOp.SUM, "max": self.tdist.ReduceOp.MAX,
               "min": self.tdist.ReduceOp.MIN}[op]
        self.tdist.all_reduce(t, op=rop, group=self.group)

    def all_to_all(self, recv, send, out_splits, in_splits):
        self.tdist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)

    def all_gather(self, out, inp):
        self.tdist.all_gather_into_tensor(out, inp, group=self.group)

    def agree(self, ok: bool, device=None) -> bool:
        """Collective: True iff `ok` on every rank (so a fallback is taken by all ranks or none)."""
        import torch
        backend = self.tdist.get_backend(self.group)
        dev = device if (backend == "nccl" and device is not None) else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.tdist.all_reduce(t, op=self.tdist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))

    def symmetric(self, shape, dtype, device) -> SymmBuf:
        """Raises if symmetric memory cannot be set up here (the caller decides collectively)."""
        import torch.distributed._symmetric_memory as symm_mem
        grp = self.group if self.group is not None else self.tdist.group.WORLD
        buf = symm_mem.empty(shape, dtype=dtype, device=device)
        hdl = symm_mem.rendezvous(buf, grp.group_name)
        try:  # non-zero when the group's buffers have a multicast (NVLS) mapping
            mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
        except Exception:  # pragma: no cover - no multicast object on this box
            mc = 0
        return SymmBuf(buf, [int(x) for x in hdl.buffer_ptrs], lambda: hdl.barrier(channel=0), mc)


class VirtualWorld:
    """Shared state of P virtual ranks (threads of one process on one device)."""

    def __init__(self, world: int, timeout: float = 300.0):
        self.world = world
        self.timeout = timeout
        self._lock = threading.Lock()
        self._groups = {}  # members tuple -> (threading.Barrier, board dict)

    def group(self, members: tuple):
        with self._lock:
            g = self._groups.get(members)
            if g is None:
                g = (threading.Barrier(len(members), timeout=self.timeout), {})
                self._groups[members] = g
            return g


class VirtualComm:
    """One virtual rank of a `VirtualWorld` (SURVEY §4.2 single-GPU "virtual ranks" backend).

    Collectives: every member deposits its tensor after synchronising its own stream, a host barrier,
    then each member computes its result from the others' device buffers -- reductions with the
    library's fixed-order `sketch_sum_peers` kernel (rank order), data movement with device copies."""

    def __init__(self, vw: VirtualWorld, rank: int, members=None):
        self.vw = vw
        self.members = tuple(members) if members is not None else tuple(range(vw.world))
        self.grank = rank
        self.rank = self.members.index(rank)
        self.world = len(self.members)
        self._bar, self._board = vw.group(self.members)
        self._seq = 0

    def split(self, groups: list) -> "VirtualComm":
        for g in groups:
            if self.grank in g:
                return VirtualComm(self.vw, self.grank, g)
        raise ValueError("rank in no subgroup")

    @staticmethod
    def _sync():
        import torch
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()

    def _exchange(self, obj):
        """All members' `obj`, in rank order (host-side rendezvous after a stream sync)."""
        self._sync()
        key = self._seq
        self._seq += 1
        self._board[(key, self.rank)] = obj
        self._bar.wait()
        objs = [self._board[(key, j)] for j in range(self.world)]
        self._bar.wait()  # everyone has read: the slot may be dropped
        self._board.pop((key, self.rank), None)
        return objs

    def _sum_into(self, out, srcs):
        """out = srcs[0] + srcs[1] + ... (rank order) with the library's sum_peers kernel."""
        import torch
        if out.is_cuda and out.numel() % 4 == 0 and all(s.data_ptr() % 16 == 0 for s in srcs) \
                and out.data_ptr() % 16 == 0 and all(s.is_contiguous() for s in srcs) and out.is_contiguous():
            from . import sum_peers
            sum_peers([s.data_ptr() for s in srcs], out.numel(), out)
        else:
            acc = srcs[0].clone()
            for s in srcs[1:]:
                acc += s
            out.copy_(acc.view_as(out))

    def reduce_scatter(self, out, inp):
        ins = self._exchange(inp)
        n = out.numel()
        self._sum_into(out.view(-1), [t.reshape(-1)[self.rank * n:(self.rank + 1) * n] for t in ins])
        self._exchange(None)  # inputs may be reused after every member has read them

    def all_reduce(self, t, op: str = "sum"):
        ins = self._exchange(t.clone())
        if op == "sum":
            self._sum_into(t.view(-1), [x.reshape(-1) for x in ins])
        else:
            import torch
            acc = ins[0].clone()
            for x in ins[1:]:
                acc = torch.maximum(acc, x) if op == "max" else torch.minimum(acc, x)
            t.copy_(acc)
        self._exchange(None)  # every member's reads of the others' copies are done (stream-synced)

    def all_to_all(self, recv, send, out_splits, in_splits):
        ins = self._exchange((send, list(in_splits)))
        off = 0
        for j, (s, splits) in enumerate(ins):
            a = sum(splits[:self.rank])
            n = splits[self.rank]
            assert n == out_splits[j]
            recv[off:off + n].copy_(s[a:a + n])
            off += n
        self._exchange(None)

    def all_gather(self, out, inp):
        ins = self._exchange(inp)
        n = inp.numel()
        for j, x in enumerate(ins):
            out.view(-1)[j * n:(j + 1) * n].copy_(x.reshape(-1))
        self._exchange(None)

    def agree(self, ok: bool, device=None) -> bool:
        return all(self._exchange(bool(ok)))

    def symmetric(self, shape, dtype, device) -> SymmBuf:
        import torch
        buf = torch.empty(shape, dtype=dtype, device=device)
        ptrs = self._exchange(buf.data_ptr())
        return SymmBuf(buf, ptrs, lambda: self._exchange(None))


# ============================================================================== the layouts
class DistSketch:
    """B = A Omega and (optionally) C = Omega^T B on a p1 x p2 grid of ranks.

    `local` is the per-rank compute: by default the CUDA library (paper_2603_20966_b200.Sketch);
    CPU tests may inject an oracle stand-in to exercise partitioning and collectives with gloo.
    `comm` defaults to a TorchComm over `group`.
    """

    def __init__(self, seed: int, dist, n1: int, n2: int, r: int, layout: Layout, group=None,
                 mode: str = "tf32", omega: str = "accurate", local=None, col_align: int = 128,
                 fused_rs=False, fused_ar: bool = False, comm=None, balance_unit: int = 0):
        self.comm = comm if comm is not None else TorchComm(group)
        self.rank = self.comm.rank
        self.world = self.comm.world
        if layout.P != self.world:
            raise ValueError("layout size != world size")
        self.layout = layout
        self.n1, self.n2, self.r = n1, n2, r
        self.i, self.j = layout.coords(self.rank)
        self.row_bnd = balanced_split(n1, layout.p1)
        self.col_bnd = balanced_split(n2, layout.p2, col_align)
        # Row-block layout cut at whole cluster units (balance_unit = rows that share each generated
        # Omega slice in the library's plan, Sketch.plan_info): rank q owns rows [q M, (q+1) M), M a
        # multiple of the unit, and the ragged tail of R = n1 - P M rows is split by COLUMNS -- every
        # rank sketches the tail rows over its 1/P of K (Alg. 1 on a P x 1 grid for the bulk and a
        # 1 x P grid for the tail) and the partials are reduced onto the last rank,
        # whose B rows [(P-1) M, n1) stay contiguous.  Every rank then runs exactly M / unit units of
        # full-K work plus a small tail launch, instead of ceil((n1 / P) / unit) units.
        self.tail = None
        self._tail_slots = None
        self._tail_k = 0
        if balance_unit and layout.p2 == 1 and self.world > 1:
            U, P = int(balance_unit), self.world
            M = (n1 // (P * U)) * U
            R = n1 - P * M
            if M > 0 and R > 0:
                self.row_bnd = [q * M for q in range(P)] + [n1]
                self.tail = {"M": M, "R": R, "cols": balanced_split(n2, P, col_align)}
        if local is None:
            from . import Sketch
            local = Sketch(seed, dist, n2, r, mode=mode, omega=omega)
        self.local = local
        # row group {(i, *)} for the reduce-scatter of B
        self.row_comm = self.comm
        if layout.p2 > 1 and layout.p1 > 1:
            self.row_comm = self.comm.split([[ii * layout.p2 + jj for jj in range(layout.p2)]
                                             for ii in range(layout.p1)])
        self.comm_bytes = 0
        # reduce-scatter of partial B for p2 > 1: False / "nccl" = NCCL reduce_scatter;
        # "peer" = B-bar written into a symmetric-memory slot, one device barrier, each owner sums its
        # piece from the p2 slots over NVLink in rank order; True / "epilogue" = the GEMM epilogue
        # stores straight into the owners' slots
        mode = {False: "nccl", None: "nccl", True: "epilogue"}.get(fused_rs, fused_rs)
        if mode not in ("nccl", "peer", "epilogue"):
            raise ValueError(f"unknown reduce-scatter mode {fused_rs!r}")
        if mode == "peer" and r % 4:
            mode = "nccl"  # the peer-read sum works on float4
        self.rs_mode = mode if layout.p2 > 1 else "nccl"
        self.fused_rs = self.rs_mode != "nccl"
        self._rs = None
        self._rsp = None
        # f1: the AllReduce of C without NCCL (symmetric memory): True = every rank's core partial in its
        # slot, one barrier, a fixed-order sum (NVLink peer reads or NVLS ld_reduce; deterministic);
        # "epilogue" = the core GEMM's epilogue adds its partial tiles into C on every rank through the
        # multicast mapping (multimem.red; no partial workspace, no reduce kernel; not bit-reproducible)
        self.ar_mode = "epilogue" if fused_ar == "epilogue" else ("sum" if fused_ar else "nccl")
        self.fused_ar = bool(fused_ar) and r % 4 == 0
        self._ar = None
        self._arm = None
        self.fallbacks = []  # (what, error) of symmetric-memory setups that fell back to NCCL
        # f1 over NVLS: symmetric-memory reductions inside the NVSwitch when the buffers have a
        # multicast mapping (SK_NVLS=0: NVLink peer reads instead)
        self.nvls = os.environ.get("SK_NVLS", "1") != "0"
        # ... for groups of at least this many ranks (2 ranks: the NVLink peer read is as fast or faster,
        # r2j / r2p); SK_NVLS_MIN overrides
        self.nvls_min_ranks = int(os.environ.get("SK_NVLS_MIN", "4"))

        self.reduce_path = None  # "nvls" / "peer" once a symmetric-memory reduction ran

    # ------------------------------------------------------------------ symmetric memory setup
    def _symm(self, comm, shape, device, what):
        """Allocate + rendezvous a symmetric buffer on `comm`; the decision to fall back to NCCL is
        collective (all ranks of `comm` agree), so no rank is left waiting in a barrier.  Only the
        setup is guarded: failures of the compute calls propagate."""
        import torch
        buf, err = None, None
        try:
            buf = comm.symmetric(shape, torch.float32, device)
        except Exception as e:  # symmetric memory unavailable on this box
            err = e
        if comm.agree(buf is not None, device):
            return buf
        self.fallbacks.append((what, repr(err)))
        print(f"[dist] {what} over symmetric memory unavailable ({err!r}); using NCCL", file=sys.stderr)
        return None

    # ------------------------------------------------------------------ partition
    def a_block_range(self) -> tuple:
        """(row0, row1, col0, col1) of A_ij owned by this rank (the bulk block for a balanced layout)."""
        if self.tail is not None:
            M = self.tail["M"]
            return self.i * M, (self.i + 1) * M, 0, self.n2
        return (self.row_bnd[self.i], self.row_bnd[self.i + 1],
                self.col_bnd[self.j], self.col_bnd[self.j + 1])

    def tail_block_range(self):
        """(row0, row1, col0, col1) of this rank's block of the ragged tail rows (balanced row-block
        layout), or None."""
        if self.tail is None:
            return None
        P, M, cols = self.world, self.tail["M"], self.tail["cols"]
        return P * M, self.n1, cols[self.rank], cols[self.rank + 1]

    def b_piece_rows(self) -> tuple:
        """Global rows of B this rank owns after the reduce-scatter: piece j of R_i."""
        r0, r1 = self.row_bnd[self.i], self.row_bnd[self.i + 1]
        if self.layout.p2 == 1:
            return r0, r1
        per = -(-(r1 - r0) // self.layout.p2)
        a = min(r1, r0 + self.j * per)
        return a, min(r1, a + per)

    # ------------------------------------------------------------------ Alg. 1
    def apply(self, A_blk, A_tail=None):
        """Returns (B_piece, (row0, row1)): the rows of B = A Omega this rank owns.  A balanced row-block
        layout also takes this rank's block of the tail rows (tail_block_range)."""
        import torch
        if self.tail is not None:
            return self._apply_balanced(A_blk, A_tail)
        r0, r1, c0, c1 = self.a_block_range()
        assert tuple(A_blk.shape) == (r1 - r0, c1 - c0), (A_blk.shape, (r1 - r0, c1 - c0))
        p2 = self.layout.p2
        if p2 == 1:
            return self.local.apply_block(A_blk, c0), (r0, r1)
        rows = r1 - r0
        per = -(-rows // p2)
        if self.rs_mode == "epilogue":
            out = self._apply_fused_rs(A_blk, rows, per, c0)
            if out is not None:
                return out
        if self.rs_mode == "peer":
            out = self._apply_peer_rs(A_blk, rows, per, c0)
            if out is not None:
                return out
        Bbar = torch.zeros((per * p2, self.r), dtype=torch.float32, device=A_blk.device)
        self.local.apply_block(A_blk, c0, out=Bbar[:rows])
        piece = torch.empty((per, self.r), dtype=torch.float32, device=A_blk.device)
        self.row_comm.reduce_scatter(piece, Bbar)
        self.comm_bytes += Bbar.numel() * 4 * (p2 - 1) // p2
        a, b = self.b_piece_rows()
        return piece[: b - a], (a, b)

    def _apply_peer_rs(self, A_blk, rows, per, c0):
        """Alg. 1 line 415 over symmetric memory: B-bar (rows padded to p2 * per) is written into this
        rank's slot (two slots alternating per call), one device barrier over the row group, then the
        owner of piece j sums rows [j per, (j+1) per) of the p2 slots -- inside the NVSwitch (NVLS)
        when the slots have a multicast mapping, else over NVLink in rank order.
        Returns None (and switches to NCCL on every rank) if symmetric memory cannot be set up."""
        import torch
        p2, r = self.layout.p2, self.r
        key = (rows, per)
        if self._rsp is None or self._rsp["key"] != key:
            sb = self._symm(self.row_comm, (2, p2 * per, r), A_blk.device, "peer-read reduce-scatter")
            if sb is None:
                self.rs_mode, self.fused_rs = "nccl", False
                return None
            sb.tensor.zero_()  # padding rows of the last piece stay zero
            self._rsp = {"key": key, "sb": sb, "k": 0}
        st = self._rsp
        k = st["k"]
        st["k"] ^= 1
        sb = st["sb"]
        self.local.apply_block(A_blk, c0, out=sb.tensor[k][:rows])
        sb.barrier()  # every rank's B-bar is in its slot k
        a, b = self.b_piece_rows()
        piece = torch.empty((per, r), dtype=torch.float32, device=A_blk.device)
        off = (k * p2 * per + self.j * per) * r * 4
        self._reduce(sb, off, per * r, piece)
        self.comm_bytes += 4 * per * r * (p2 - 1)
        return piece[: b - a], (a, b)

    def _apply_balanced(self, A_blk, A_tail):
        """Balanced row-block (see __init__): the tail partial first (so every rank reaches the barrier
        together), then the bulk rows; the last rank sums the P tail partials into the end of its B."""
        import torch
        T, r, P = self.tail, self.r, self.world
        M, R = T["M"], T["R"]
        t0, t1, c0, c1 = self.tail_block_range()
        assert A_tail is not None and tuple(A_tail.shape) == (t1 - t0, c1 - c0), "tail block expected"
        assert tuple(A_blk.shape) == (M, self.n2), (A_blk.shape, (M, self.n2))
        owner = self.rank == P - 1
        dev = A_blk.device
        sb = None
        if r % 4 == 0 and getattr(A_blk, "is_cuda", False):
            if self._tail_slots is None:
                self._tail_slots = self._symm(self.comm, (2, R * r), dev, "tail reduction") or False
            sb = self._tail_slots or None
        if sb is not None:
            k = self._tail_k
            self._tail_k ^= 1
            part = sb.tensor[k].view(R, r)
            self.local.apply_block(A_tail, c0, out=part)
            sb.barrier()  # every rank's tail partial is in its slot k
        else:
            part = self.local.apply_block(A_tail, c0)
        Bp = torch.empty((M + R, r), dtype=torch.float32, device=dev) if owner else None
        if owner:
            self.local.apply_block(A_blk, 0, out=Bp[:M])
        else:
            Bp = self.local.apply_block(A_blk, 0)
        if sb is not None:
            if owner:
                self._reduce(sb, k * R * r * 4, R * r, Bp[M:])
        else:
            self.comm.all_reduce(part)
            if owner:
                Bp[M:].copy_(part)
        self.comm_bytes += 4 * R * r  # this rank's tail partial handed to the reduction
        return Bp, self.b_piece_rows()

    def _reduce(self, sb, off: int, elems: int, out):
        """out[:elems] = sum over the group of the symmetric buffers at byte offset `off`: inside the
        NVSwitch through the multicast mapping (NVLS, `sketch_multimem_sum`) when the group has one,
        else NVLink peer reads in rank order (`sketch_sum_peers`)."""
        from . import multimem_sum, sum_peers
        if self.nvls and sb.multicast_ptr and elems % 4 == 0 and len(sb.ptrs) >= self.nvls_min_ranks:
            multimem_sum(sb.multicast_ptr + off, elems, out)
            self.reduce_path = "nvls"
        else:
            sum_peers([p + off for p in sb.ptrs], elems, out)
            self.reduce_path = "peer"

    def _apply_fused_rs(self, A_blk, rows, per, c0):
        """Alg. 1 line 415 with the reduce-scatter fused into the GEMM epilogue: every
        rank's kernel stores its partial rows of piece j straight into rank (i, j)'s receive slot over
        NVLink; after a device-side barrier each owner sums its p2 * split slots in a fixed order."""
        import torch
        p2 = self.layout.p2
        npad = -(-self.r // 16) * 16
        k = A_blk.shape[1]
        if self._rs is None or self._rs["key"] != (rows, per, k):
            # split-K partials would each cross NVLink (S x the reduce-scatter bytes): default to no
            # split; SK_RS_SPLIT=auto takes the local plan's choice (max over the row group)
            env = os.environ.get("SK_RS_SPLIT", "1")
            split = 1 if env == "auto" else max(1, int(env))
            if env == "auto":
                t = torch.tensor([max(split, self.local.rs_split(rows, k))], dtype=torch.int32, device=A_blk.device)
                self.row_comm.all_reduce(t, op="max")  # same slot layout everywhere
                split = int(t.item())
            sb = self._symm(self.row_comm, (p2 * split * per * npad,), A_blk.device, "epilogue reduce-scatter")
            if sb is None:
                self.rs_mode, self.fused_rs = "nccl", False
                return None
            self._rs = {"key": (rows, per, k), "sb": sb, "split": split, "npad": npad}
        rs = self._rs
        sb, split = rs["sb"], rs["split"]
        sb.barrier()  # the owners have consumed the previous step's slots
        self.local.apply_block_rs(A_blk, c0, sb.ptrs[:p2], per, self.j, per * npad, split)
        sb.barrier()  # every rank's stores have landed
        a, b = self.b_piece_rows()
        piece = self.local.reduce_slots(sb.tensor, p2 * split, per * npad, b - a)
        # bytes this rank stored into other ranks' slots (split partials, rows padded to npad)
        mine = [min(rows, (jj + 1) * per) - min(rows, jj * per) for jj in range(p2)]
        self.comm_bytes += 4 * split * npad * (rows - mine[self.j])
        return piece, (a, b)

    # ------------------------------------------------------------------ Alg. 2 (Redist)
    def nystrom_core_redist(self, A_blk, A_tail=None):
        """Redist variant: returns (B_piece, rows, C) like nystrom_core (row-block layout only)."""
        import torch
        if self.layout.p2 != 1:
            raise ValueError("the Redist variant runs on the row-block grid Pi = (P, 1, 1)")
        Bp, (a, b) = self.apply(A_blk, A_tail)
        P, r = self.world, self.r
        if P == 1:
            return Bp, (a, b), self.local.core_block(Bp, a)
        cb = balanced_split(r, P)
        k = self.rank
        nbk = cb[k + 1] - cb[k]
        rows = [self.row_bnd[j + 1] - self.row_bnd[j] for j in range(P)]
        # pack by column block: block j = B[:, cb[j]:cb[j+1]] row-major, contiguous
        send = self.local.pack_cols(Bp, cb)
        in_splits = [(b - a) * (cb[j + 1] - cb[j]) for j in range(P)]
        out_splits = [rows[j] * nbk for j in range(P)]
        recv = torch.empty(sum(out_splits), dtype=torch.float32, device=Bp.device)
        self.comm.all_to_all(recv, send, out_splits, in_splits)
        self.comm_bytes += 4 * (sum(in_splits) - in_splits[k])
        Bcol = recv.view(self.n1, nbk)  # rows arrive in rank order = global row order: no unpack
        width = max(cb[j + 1] - cb[j] for j in range(P))
        # column block of C = Omega^T B[:, cols_k], Omega regenerated for all n rows, written into a
        # block padded to the widest column block for the all-gather that replicates C
        pad = torch.zeros((r, width), dtype=torch.float32, device=Bp.device)
        self.local.core_block_cols(Bcol, 0, out=pad[:, :nbk])
        gathered = torch.empty(P * r * width, dtype=torch.float32, device=Bp.device)
        self.comm.all_gather(gathered, pad.reshape(-1))
        gathered = gathered.view(P, r, width)
        self.comm_bytes += 4 * r * width * (P - 1)
        C = torch.cat([gathered[j, :, : cb[j + 1] - cb[j]] for j in range(P)], dim=1)
        return Bp, (a, b), C

    # ------------------------------------------------------------------ Alg. 2 (No-Redist)
    def nystrom_core(self, A_blk, A_tail=None):
        """Returns (B_piece, rows, C) with C = Omega^T A Omega replicated on every rank."""
        Bp, (a, b) = self.apply(A_blk, A_tail)
        if self.world > 1 and self.fused_ar and self.ar_mode == "epilogue":
            C = self._core_epilogue_allreduce(Bp, a)
            if C is not None:
                return Bp, (a, b), C
        if self.world > 1 and self.fused_ar:
            C = self._core_fused_allreduce(Bp, a)
            if C is not None:
                return Bp, (a, b), C
        C = self.local.core_block(Bp, a)
        if self.world > 1:
            self.comm.all_reduce(C)
            self.comm_bytes += C.numel() * 4
        return Bp, (a, b), C

    def _core_epilogue_allreduce(self, Bp, a):
        """AllReduce of C issued from the core GEMM's epilogue: every rank zeroes its copy
        of a symmetric r x r buffer, barrier, the core GEMM adds each partial tile into all ranks' copies
        through the multicast mapping (multimem.red inside the NVSwitch), barrier, C = this rank's copy.
        Returns None (and switches to the fixed-order sum) without a multicast mapping."""
        import torch
        r = self.r
        if self._arm is None:
            sb = self._symm(self.comm, (r * r,), Bp.device, "epilogue AllReduce")
            ok = self.comm.agree(sb is not None and bool(sb.multicast_ptr), Bp.device)
            if not ok:
                self.ar_mode = "sum"
                self.fallbacks.append(("epilogue AllReduce", "no multicast mapping"))
                return None
            self._arm = {"sb": sb}
        sb = self._arm["sb"]
        sb.tensor.zero_()
        sb.barrier()  # every rank's copy is zero (and every rank has read the previous C)
        self.local.core_block_mc(Bp, a, sb.multicast_ptr, r)
        sb.barrier()  # every rank's reductions have landed in every copy
        self.reduce_path = "nvls-epilogue"
        self.comm_bytes += r * r * 4
        return sb.tensor.view(r, r).clone()

    def _core_fused_allreduce(self, Bp, a):
        """AllReduce of the r x r core partials without NCCL: each rank's core GEMM
        writes its partial into its own symmetric-memory slot (two slots, alternating per call), one
        device barrier, then every rank sums all ranks' slots: in the NVSwitch (NVLS multimem
        ld_reduce) when the slots have a multicast mapping, else over NVLink in rank order."""
        import torch
        r = self.r
        if self._ar is None:
            sb = self._symm(self.comm, (2, r * r), Bp.device, "fused AllReduce")
            if sb is None:
                self.fused_ar = False
                return None
            self._ar = {"sb": sb, "k": 0}
        ar = self._ar
        k = ar["k"]
        ar["k"] ^= 1
        sb = ar["sb"]
        self.local.core_block(Bp, a, out=sb.tensor[k].view(r, r))
        sb.barrier()  # every rank's partial is in its slot k
        C = torch.empty((r, r), dtype=torch.float32, device=Bp.device)
        self._reduce(sb, k * r * r * 4, r * r, C)
        self.comm_bytes += r * r * 4
        return C


def run_virtual(world: int, fn, timeout: float = 600.0):
    """Runs fn(comm) for `world` virtual ranks (threads of this process on the current device when CUDA
    is available); returns the results in rank order, re-raising the first error.

    All virtual ranks enqueue on ONE shared CUDA stream: the persistent sketch kernel's CTAs may wait on
    one another inside a launch (in-place pieces, sketch_gemm.cu), which is safe only while the grid is
    co-resident -- two such launches running concurrently on one GPU could each hold the SMs the other
    waits for.  Serialising the ranks' kernels on one stream keeps every launch alone on the device."""
    import torch
    vw = VirtualWorld(world)
    res, errs = [None] * world, [None] * world
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None
    shared = torch.cuda.Stream(device=dev) if dev is not None else None

    def body(rank):
        try:
            if dev is not None:
                torch.cuda.set_device(dev)
                s = shared
                with torch.cuda.stream(s):
                    res[rank] = fn(VirtualComm(vw, rank))
                    s.synchronize()
            else:
                res[rank] = fn(VirtualComm(vw, rank))
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs[rank] = e
            for bar, _ in list(vw._groups.values()):
                bar.abort()

    ts = [threading.Thread(target=body, args=(i,)) for i in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return res
