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
so that rank k owns column block k of B over all n rows (bandwidth ~ n r / P words, PAPER.md:675;
the pack / unpack of the paper's column-major exchange, is a strided copy here), and
rank k computes the column block C[:, cols_k] = Omega^T B[:, cols_k] with Omega regenerated for all n
rows.  The paper leaves C distributed; `nystrom_core_redist` all-gathers the column blocks so both
variants return the same replicated C.

Bandwidth accounting: predicted words per rank = (1 - 1/p2) n1 r / p1 for B (Alg. 1 cost,
PAPER.md:427 with p3 = 1) plus the AllReduce payload r^2 for C; measured = bytes handed to
the collectives.  Row splits are balanced; column splits are multiples of 128 (so each block's
Omega rows start on a Philox row-group boundary) except the last.
"""
from __future__ import annotations

import os

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


def predicted_bytes_per_rank(n1: int, r: int, layout: Layout, nystrom: bool, variant: str = "noredist") -> int:
    """Alg. 1 reduce-scatter volume (1 - 1/p2) n1 r / p1 words (+ r^2 AllReduce payload), fp32.
    Redist (row-block only): All-to-All of B, (1 - 1/P) n r / P words sent per rank,
    plus the all-gather that replicates C, (P - 1) r ceil(r / P) words."""
    P = layout.P
    if variant == "redist" and nystrom and P > 1:
        return int(4 * ((n1 * r) // P - (n1 // P) * (r // P) + (P - 1) * r * (-(-r // P)))) if (n1 % P == 0 and r % P == 0) \
            else -1
    words = (1.0 - 1.0 / layout.p2) * n1 * r / layout.p1
    if nystrom and P > 1:
        words += r * r
    return int(round(4 * words))


class DistSketch:
    """B = A Omega and (optionally) C = Omega^T B on a p1 x p2 grid of ranks.

    `local` is the per-rank compute: by default the CUDA library (paper_2603_20966_b200.Sketch);
    tests may inject a CPU stand-in to exercise partitioning and collectives with gloo.
    """

    def __init__(self, seed: int, dist, n1: int, n2: int, r: int, layout: Layout, group=None,
                 mode: str = "tf32", omega: str = "accurate", local=None, col_align: int = 128,
                 fused_rs=False, fused_ar: bool = False):
        import torch.distributed as tdist
        self.tdist = tdist
        self.group = group
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)
        if layout.P != self.world:
            raise ValueError("layout size != world size")
        self.layout = layout
        self.n1, self.n2, self.r = n1, n2, r
        self.i, self.j = layout.coords(self.rank)
        self.row_bnd = balanced_split(n1, layout.p1)
        self.col_bnd = balanced_split(n2, layout.p2, col_align)
        if local is None:
            from . import Sketch
            local = Sketch(seed, dist, n2, r, mode=mode, omega=omega)
        self.local = local
        # row group {(i, *)} for the reduce-scatter of B
        self.row_group = group
        if layout.p2 > 1 and layout.p1 > 1:
            groups = [tdist.new_group([ii * layout.p2 + jj for jj in range(layout.p2)])
                      for ii in range(layout.p1)]
            self.row_group = groups[self.i]
        elif layout.p2 > 1:
            self.row_group = group
        self.comm_bytes = 0
        # f1: reduce-scatter of partial B fused into the GEMM epilogue (NVLink stores into the owners'
        # symmetric-memory receive buffers) instead of an NCCL reduce_scatter after the GEMM
        # reduce-scatter of partial B for p2 > 1: False / "nccl" = NCCL reduce_scatter; "peer" = B-bar
        # written into a symmetric-memory slot, one device barrier, each owner sums its piece from
        # the p2 slots over NVLink in rank order; True / "epilogue" = the GEMM epilogue stores
        # straight into the owners' slots
        mode = {False: "nccl", None: "nccl", True: "epilogue"}.get(fused_rs, fused_rs)
        if mode not in ("nccl", "peer", "epilogue"):
            raise ValueError(f"unknown reduce-scatter mode {fused_rs!r}")
        if mode == "peer" and r % 4:
            mode = "nccl"  # the peer-read sum works on float4
        self.rs_mode = mode if layout.p2 > 1 else "nccl"
        self.fused_rs = self.rs_mode != "nccl"
        self._rs = None
        self._rsp = None
        # f1: the AllReduce of C as one NVLink peer-read sum instead of NCCL (symmetric memory)
        self.fused_ar = bool(fused_ar)
        self._ar = None

    # ------------------------------------------------------------------ partition
    def a_block_range(self) -> tuple:
        """(row0, row1, col0, col1) of A_ij owned by this rank."""
        return (self.row_bnd[self.i], self.row_bnd[self.i + 1],
                self.col_bnd[self.j], self.col_bnd[self.j + 1])

    def b_piece_rows(self) -> tuple:
        """Global rows of B this rank owns after the reduce-scatter: piece j of R_i."""
        r0, r1 = self.row_bnd[self.i], self.row_bnd[self.i + 1]
        if self.layout.p2 == 1:
            return r0, r1
        per = -(-(r1 - r0) // self.layout.p2)
        a = min(r1, r0 + self.j * per)
        return a, min(r1, a + per)

    # ------------------------------------------------------------------ Alg. 1
    def apply(self, A_blk):
        """Returns (B_piece, (row0, row1)): the rows of B = A Omega this rank owns."""
        import torch
        r0, r1, c0, c1 = self.a_block_range()
        assert tuple(A_blk.shape) == (r1 - r0, c1 - c0), (A_blk.shape, (r1 - r0, c1 - c0))
        p2 = self.layout.p2
        if p2 == 1:
            return self.local.apply_block(A_blk, c0), (r0, r1)
        rows = r1 - r0
        per = -(-rows // p2)
        if self.rs_mode == "epilogue":
            return self._apply_fused_rs(A_blk, rows, per, c0)
        if self.rs_mode == "peer":
            try:
                return self._apply_peer_rs(A_blk, rows, per, c0)
            except Exception as e:  # symmetric memory unavailable: NCCL from now on (same results)
                self._fallback("peer-read reduce-scatter", e)
        Bbar = torch.zeros((per * p2, self.r), dtype=torch.float32, device=A_blk.device)
        self.local.apply_block(A_blk, c0, out=Bbar[:rows])
        piece = torch.empty((per, self.r), dtype=torch.float32, device=A_blk.device)
        self.tdist.reduce_scatter_tensor(piece, Bbar, group=self.row_group)
        self.comm_bytes += Bbar.numel() * 4 * (p2 - 1) // p2
        a, b = self.b_piece_rows()
        return piece[: b - a], (a, b)

    def _fallback(self, what, err):
        """Symmetric memory could not be set up (every rank hits the same condition): use NCCL."""
        import sys
        print(f"[dist] {what} over symmetric memory unavailable ({err!r}); using NCCL", file=sys.stderr)
        if self.rs_mode in ("peer", "epilogue"):
            self.rs_mode, self.fused_rs = "nccl", False
        self.fused_ar = False

    def _apply_peer_rs(self, A_blk, rows, per, c0):
        """Alg. 1 line 415 over symmetric memory: B-bar (rows padded to p2 * per) is written into this
        rank's slot (two slots alternating per call), one device barrier over the row group, then the
        owner of piece j sums rows [j per, (j+1) per) of the p2 slots over NVLink in rank order."""
        import torch
        from . import sum_peers
        p2, r = self.layout.p2, self.r
        key = (rows, per)
        if self._rsp is None or self._rsp["key"] != key:
            import torch.distributed._symmetric_memory as symm_mem
            grp = self.row_group if self.row_group is not None else self.tdist.group.WORLD
            try:
                symm_mem.enable_symm_mem_for_group(grp.group_name)
            except Exception:  # pragma: no cover
                pass
            buf = symm_mem.empty((2, p2 * per, r), dtype=torch.float32, device=A_blk.device)
            buf.zero_()  # padding rows of the last piece stay zero
            hdl = symm_mem.rendezvous(buf, grp.group_name)
            self._rsp = {"key": key, "buf": buf, "hdl": hdl, "ptrs": [int(x) for x in hdl.buffer_ptrs], "k": 0}
        st = self._rsp
        k = st["k"]
        st["k"] ^= 1
        self.local.apply_block(A_blk, c0, out=st["buf"][k][:rows])
        st["hdl"].barrier(channel=0)  # every rank's B-bar is in its slot k
        a, b = self.b_piece_rows()
        piece = torch.empty((per, r), dtype=torch.float32, device=A_blk.device)
        off = (k * p2 * per + self.j * per) * r * 4
        sum_peers([p + off for p in st["ptrs"]], per * r, piece)
        self.comm_bytes += 4 * per * r * (p2 - 1)
        return piece[: b - a], (a, b)

    def _apply_fused_rs(self, A_blk, rows, per, c0):
        """Alg. 1 line 415 with the reduce-scatter fused into the GEMM epilogue: every
        rank's kernel stores its partial rows of piece j straight into rank (i, j)'s receive slot over
        NVLink; after a device-side barrier each owner sums its p2 * split slots in a fixed order."""
        import torch
        p2 = self.layout.p2
        npad = -(-self.r // 16) * 16
        k = A_blk.shape[1]
        if self._rs is None or self._rs["key"] != (rows, per, k):
            import torch.distributed._symmetric_memory as symm_mem
            grp = self.row_group if self.row_group is not None else self.tdist.group.WORLD
            # split-K partials would each cross NVLink (S x the reduce-scatter bytes): default to no
            # split; RS_SPLIT=auto takes the local plan's choice (max over the row group)
            if os.environ.get("SK_RS_SPLIT", "1") == "auto":
                split = torch.tensor([self.local.rs_split(rows, k)], dtype=torch.int32, device=A_blk.device)
                self.tdist.all_reduce(split, op=self.tdist.ReduceOp.MAX, group=grp)  # same slot layout everywhere
                split = int(split.item())
            else:
                split = max(1, int(os.environ.get("SK_RS_SPLIT", "1")))
            try:
                symm_mem.enable_symm_mem_for_group(grp.group_name)
            except Exception:  # pragma: no cover - newer torch enables it implicitly
                pass
            buf = symm_mem.empty((p2 * split * per * npad,), dtype=torch.float32, device=A_blk.device)
            hdl = symm_mem.rendezvous(buf, grp.group_name)
            ptrs = [int(hdl.buffer_ptrs[j]) for j in range(p2)]
            self._rs = {"key": (rows, per, k), "buf": buf, "hdl": hdl, "ptrs": ptrs, "split": split, "npad": npad}
        rs = self._rs
        hdl, split = rs["hdl"], rs["split"]
        hdl.barrier(channel=0)  # the owners have consumed the previous step's slots
        self.local.apply_block_rs(A_blk, c0, rs["ptrs"], per, self.j, per * npad, split)
        hdl.barrier(channel=0)  # every rank's stores have landed
        a, b = self.b_piece_rows()
        piece = self.local.reduce_slots(rs["buf"], p2 * split, per * npad, b - a)
        # bytes this rank stored into other ranks' slots (split partials, rows padded to npad)
        mine = [min(rows, (jj + 1) * per) - min(rows, jj * per) for jj in range(p2)]
        self.comm_bytes += 4 * split * npad * (rows - mine[self.j])
        return piece, (a, b)

    # ------------------------------------------------------------------ Alg. 2 (Redist)
    def nystrom_core_redist(self, A_blk):
        """Redist variant: returns (B_piece, rows, C) like nystrom_core (row-block layout only)."""
        import torch
        if self.layout.p2 != 1:
            raise ValueError("the Redist variant runs on the row-block grid Pi = (P, 1, 1)")
        Bp, (a, b) = self.apply(A_blk)
        P, r = self.world, self.r
        if P == 1:
            return Bp, (a, b), self.local.core_block(Bp, a)
        cb = balanced_split(r, P)
        k = self.rank
        nbk = cb[k + 1] - cb[k]
        rows = [self.row_bnd[j + 1] - self.row_bnd[j] for j in range(P)]
        send = torch.cat([Bp[:, cb[j]:cb[j + 1]].reshape(-1) for j in range(P)])  # pack by column block
        in_splits = [(b - a) * (cb[j + 1] - cb[j]) for j in range(P)]
        out_splits = [rows[j] * nbk for j in range(P)]
        recv = torch.empty(sum(out_splits), dtype=torch.float32, device=Bp.device)
        self.tdist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)
        self.comm_bytes += 4 * (sum(in_splits) - in_splits[k])
        Bcol = recv.view(self.n1, nbk)  # rows arrive in rank order = global row order
        Ccol = self.local.core_block_cols(Bcol, 0)  # r x nbk, Omega regenerated for all n rows
        # replicate C: all-gather the column blocks (padded to the largest block)
        width = max(cb[j + 1] - cb[j] for j in range(P))
        pad = torch.zeros((r, width), dtype=torch.float32, device=Bp.device)
        pad[:, :nbk] = Ccol
        gathered = torch.empty(P * r * width, dtype=torch.float32, device=Bp.device)
        self.tdist.all_gather_into_tensor(gathered, pad.reshape(-1), group=self.group)
        gathered = gathered.view(P, r, width)
        self.comm_bytes += 4 * r * width * (P - 1)
        C = torch.cat([gathered[j, :, : cb[j + 1] - cb[j]] for j in range(P)], dim=1)
        return Bp, (a, b), C

    # ------------------------------------------------------------------ Alg. 2 (No-Redist)
    def nystrom_core(self, A_blk):
        """Returns (B_piece, rows, C) with C = Omega^T A Omega replicated on every rank."""
        Bp, (a, b) = self.apply(A_blk)
        if self.world > 1 and self.fused_ar:
            try:
                return Bp, (a, b), self._core_fused_allreduce(Bp, a)
            except Exception as e:  # symmetric memory unavailable: NCCL from now on (same results)
                self._fallback("fused AllReduce", e)
        C = self.local.core_block(Bp, a)
        if self.world > 1:
            self.tdist.all_reduce(C, group=self.group)
            self.comm_bytes += C.numel() * 4
        return Bp, (a, b), C

    def _core_fused_allreduce(self, Bp, a):
        """AllReduce of the r x r core partials without NCCL: each rank's core GEMM
        writes its partial into its own symmetric-memory slot (two slots, alternating per call), one
        device barrier, then every rank sums all ranks' slots over NVLink in rank order."""
        import torch
        from . import sum_peers
        r = self.r
        if self._ar is None:
            import torch.distributed._symmetric_memory as symm_mem
            grp = self.group if self.group is not None else self.tdist.group.WORLD
            try:
                symm_mem.enable_symm_mem_for_group(grp.group_name)
            except Exception:  # pragma: no cover
                pass
            buf = symm_mem.empty((2, r * r), dtype=torch.float32, device=Bp.device)
            hdl = symm_mem.rendezvous(buf, grp.group_name)
            self._ar = {"buf": buf, "hdl": hdl, "ptrs": [int(x) for x in hdl.buffer_ptrs], "k": 0}
        ar = self._ar
        k = ar["k"]
        ar["k"] ^= 1
        self.local.core_block(Bp, a, out=ar["buf"][k].view(r, r))
        ar["hdl"].barrier(channel=0)  # every rank's partial is in its slot k
        C = torch.empty((r, r), dtype=torch.float32, device=Bp.device)
        sum_peers([p + k * r * r * 4 for p in ar["ptrs"]], r * r, C)
        self.comm_bytes += r * r * 4
        return C
