"""paper_2603_20966_b200 -- B200-native sketch B = A*Omega and Nystrom core C = Omega^T*B.

Thin ctypes binding over ``libsketch.so`` (C ABI in ``include/sketch.h``).  This module only
marshals arguments: torch tensors -> device pointers, torch's current stream -> cudaStream_t,
workspace allocation.  Every step of the hot path runs in the library's CUDA kernels; there is
no CPU fallback -- without the extension or a GPU every compute call raises.

PAPER.md references: problem statement PAPER.md:106-122 (sec. 1); Omega regenerated from a
shared-seed counter-based Philox stream, PAPER.md:1185-1190 (sec. 6.3).
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["Sketch", "SketchError", "load_library", "library_path", "EXPORTED_SYMBOLS",
           "GAUSSIAN", "RADEMACHER", "UNIFORM", "MODES"]

GAUSSIAN, RADEMACHER, UNIFORM = 0, 1, 2
_DISTS = {"gaussian": GAUSSIAN, "rademacher": RADEMACHER, "uniform": UNIFORM}
MODES = {"tf32x3": 0, "tf32": 1, "bf16": 2}
_OMEGA = {"accurate": 0, "fast": 1}

EXPORTED_SYMBOLS = (
    "sketch_create", "sketch_destroy", "sketch_set_mode", "sketch_set_omega_transform",
    "sketch_set_split_k", "sketch_set_cta_group", "sketch_set_core_impl", "sketch_set_ablation", "sketch_set_trace",
    "sketch_workspace_size", "sketch_apply", "nystrom_core",
    "sketch_apply_block", "core_apply_block", "core_apply_block_mc", "core_apply_block_cols", "sketch_generate", "sketch_generate_bits",
    "sketch_rs_split", "sketch_plan_info", "sketch_apply_block_rs", "sketch_reduce_slots", "sketch_sum_peers", "sketch_multimem_sum", "sketch_pack_cols",
    "sketch_host_workspace_size", "sketch_apply_host", "nystrom_core_host",
    "sketch_debug_box_muller", "sketch_set_profiling", "sketch_profile_read", "sketch_launch_count",
    "sketch_status_string", "sketch_last_error", "sketch_build_info",
)
PHASES = ("sketch_gemm", "splitk_reduce", "core_gemm", "core_reduce", "generate")

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
_lock = threading.Lock()


class SketchError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


def library_path() -> str:
    return os.path.join(_HERE, "libsketch.so")


def load_library(build_if_missing: bool = True):
    """Load libsketch.so (building it in-tree with nvcc if absent or stale)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build as _build
        if build_if_missing:
            _build.build()
        path = library_path()
        if not os.path.exists(path):
            raise SketchError(-1, "SK_ERR_NOT_BUILT", f"{path} missing (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        i64, u64, i32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
        sz = ctypes.c_size_t
        lib.sketch_create.argtypes = [u64, ctypes.c_int, i64, i64, ctypes.POINTER(vp)]
        lib.sketch_destroy.argtypes = [vp]
        lib.sketch_set_mode.argtypes = [vp, ctypes.c_int]
        lib.sketch_set_omega_transform.argtypes = [vp, ctypes.c_int]
        lib.sketch_set_split_k.argtypes = [vp, i32]
        lib.sketch_set_cta_group.argtypes = [vp, i32]
        lib.sketch_set_ablation.argtypes = [vp, ctypes.c_uint32]
        lib.sketch_set_core_impl.argtypes = [vp, i32]
        lib.sketch_workspace_size.argtypes = [vp, i64, ctypes.POINTER(sz)]
        lib.sketch_apply.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, sz, vp]
        lib.nystrom_core.argtypes = [vp, vp, i64, i64, vp, i64, vp, i64, vp, sz, vp]
        lib.sketch_apply_block.argtypes = [vp, vp, i64, i64, i64, i64, vp, i64, vp, sz, vp]
        lib.core_apply_block.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, sz, vp]
        lib.core_apply_block_cols.argtypes = [vp, vp, i64, i64, i64, i64, vp, i64, vp, sz, vp]
        lib.sketch_host_workspace_size.argtypes = [vp, i64, i64, ctypes.POINTER(sz)]
        lib.sketch_apply_host.argtypes = [vp, vp, i64, i64, i64, vp, i64, i64, vp, sz, vp]
        lib.nystrom_core_host.argtypes = [vp, vp, i64, i64, vp, i64, vp, i64, i64, vp, sz, vp]
        lib.sketch_rs_split.argtypes = [vp, i64, i64, ctypes.POINTER(i32)]
        lib.sketch_apply_block_rs.argtypes = [vp, vp, i64, i64, i64, i64, ctypes.POINTER(vp), i32, i64, i32, i64,
                                              i32, vp]
        lib.sketch_reduce_slots.argtypes = [vp, vp, i32, i64, i64, vp, i64, vp]
        lib.sketch_sum_peers.argtypes = [ctypes.POINTER(vp), i32, i64, vp, vp]
        lib.sketch_multimem_sum.argtypes = [vp, i64, vp, vp, vp]
        lib.core_apply_block_mc.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, ctypes.c_size_t, vp]
        lib.sketch_plan_info.argtypes = [vp, i64, i64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        lib.sketch_pack_cols.argtypes = [vp, i64, i64, ctypes.POINTER(i64), i32, vp, vp]
        lib.sketch_set_trace.argtypes = [vp, vp, i32]
        lib.sketch_generate.argtypes = [vp, i64, i64, i64, i64, vp, i64, vp]
        lib.sketch_generate_bits.argtypes = [vp, i64, i64, i64, i64, vp, i64, vp]
        lib.sketch_debug_box_muller.argtypes = [vp, vp, i64, ctypes.c_int, vp, vp, vp]
        lib.sketch_set_profiling.argtypes = [vp, ctypes.c_int]
        lib.sketch_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        lib.sketch_launch_count.restype = ctypes.c_uint64
        lib.sketch_status_string.argtypes = [ctypes.c_int]
        lib.sketch_status_string.restype = ctypes.c_char_p
        lib.sketch_last_error.restype = ctypes.c_char_p
        lib.sketch_build_info.restype = ctypes.c_char_p
        for name in EXPORTED_SYMBOLS:
            if name not in ("sketch_status_string", "sketch_last_error", "sketch_build_info",
                            "sketch_launch_count"):
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def _check(status: int) -> None:
    if status != 0:
        lib = load_library()
        raise SketchError(status, lib.sketch_status_string(status).decode(),
                          lib.sketch_last_error().decode())


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _require_cuda(*tensors):
    torch = _torch()
    if not torch.cuda.is_available():
        raise SketchError(-1, "SK_ERR_NO_GPU", "no CUDA device: the sketch runs only on the GPU")
    for t in tensors:
        if t is not None and (not t.is_cuda or t.dtype != torch.float32):
            raise SketchError(1, "SK_ERR_INVALID_VALUE", "expected float32 CUDA tensors")
        if t is not None and t.dim() == 2 and t.stride(1) != 1:
            raise SketchError(1, "SK_ERR_INVALID_VALUE", "expected row-major tensors (stride(1) == 1)")


def _tma_ready(A):
    """A with a 16-byte-aligned base and row stride (TMA's requirement, SK_ERR_ALIGNMENT in the ABI).

    Contiguous inputs whose row length is not a multiple of 4 fp32 are copied once into a padded
    buffer (argument marshalling; pass an aligned A to avoid the extra pass over HBM)."""
    if A.dim() == 2 and A.shape[0] > 0 and (A.stride(0) % 4 != 0 or A.data_ptr() % 16 != 0):
        torch = _torch()
        n1, n2 = A.shape
        buf = torch.empty((n1, (n2 + 3) // 4 * 4), dtype=A.dtype, device=A.device)[:, :n2]
        buf.copy_(A)
        return buf
    return A


class Sketch:
    """Omega in R^{n2 x r} drawn from ``dist`` with ``seed``; never materialised on the hot path.

    mode: 'tf32x3' (fp32-accurate), 'tf32', 'bf16'; omega: 'accurate' | 'fast' Box-Muller.
    """

    def __init__(self, seed: int, dist, n2: int, r: int, mode: str = "tf32x3",
                 omega: str = "accurate", split_k: int = 0, cta_group: int = 0,
                 core: str = "auto"):
        self._lib = load_library()
        self.seed, self.n2, self.r = int(seed), int(n2), int(r)
        self.dist = _DISTS[dist] if isinstance(dist, str) else int(dist)
        self.mode, self.omega = mode, omega
        h = ctypes.c_void_p()
        _check(self._lib.sketch_create(self.seed, self.dist, self.n2, self.r, ctypes.byref(h)))
        self._h = h
        _check(self._lib.sketch_set_mode(h, MODES[mode]))
        _check(self._lib.sketch_set_omega_transform(h, _OMEGA[omega]))
        _check(self._lib.sketch_set_split_k(h, int(split_k)))
        _check(self._lib.sketch_set_cta_group(h, int(cta_group)))
        _check(self._lib.sketch_set_core_impl(h, 1 if core == "simt" else 0))
        self._ws = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.sketch_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    def set_ablation(self, flags: int) -> None:
        """Measurement-only switches (see sketch_set_ablation in include/sketch.h); results are wrong while set."""
        _check(self._lib.sketch_set_ablation(self._h, int(flags)))

    def set_trace(self, buf=None, stages: int = 0) -> None:
        """Pipeline trace (measurements only): `buf` a CUDA (or pinned host) int64 tensor of >= 1280*stages entries."""
        ptr = ctypes.c_void_p(buf.data_ptr() if buf is not None else 0)
        _check(self._lib.sketch_set_trace(self._h, ptr, int(stages)))

    # ------------------------------------------------------------------ profiling
    def set_profiling(self, enable: bool = True) -> None:
        _check(self._lib.sketch_set_profiling(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{phase: (device ms summed over launches, launch count)}; clears the record."""
        ms = (ctypes.c_double * len(PHASES))()
        cnt = (ctypes.c_int64 * len(PHASES))()
        _check(self._lib.sketch_profile_read(self._h, ms, cnt))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(PHASES)}

    # ------------------------------------------------------------------ workspace
    def workspace_size(self, n1: int) -> int:
        n = ctypes.c_size_t()
        _check(self._lib.sketch_workspace_size(self._h, int(n1), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, n1: int, device=None):
        """Device workspace for n1 rows (cached per (device, n1): no ABI query on the hot path)."""
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        key = (dev.index, int(n1))
        ws = self._ws.get(key)
        if ws is None:
            nbytes = self.workspace_size(n1)
            ws = torch.empty(max(nbytes, 16) // 4 + 4, dtype=torch.float32, device=dev)
            if len(self._ws) > 8:
                self._ws.clear()
            self._ws[key] = ws
        return ws

    # ------------------------------------------------------------------ hot path
    def apply(self, A, out=None, stream=None):
        """B = A Omega for A (n1 x n2) fp32 CUDA, row-major."""
        torch = _torch()
        _require_cuda(A, out)
        n1, n2 = A.shape
        A = _tma_ready(A)
        if out is None:
            out = torch.empty((n1, self.r), dtype=torch.float32, device=A.device)
        ws = self.workspace(n1, A.device)
        _check(self._lib.sketch_apply(self._h, A.data_ptr(), n1, n2, A.stride(0), out.data_ptr(),
                                      out.stride(0), ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)))
        return out

    def apply_block(self, A_blk, k0: int, out=None, stream=None):
        """B_part = A_blk Omega[k0:k0+k] (block form of Alg. 1)."""
        torch = _torch()
        _require_cuda(A_blk, out)
        m, k = A_blk.shape
        A_blk = _tma_ready(A_blk)
        if out is None:
            out = torch.empty((m, self.r), dtype=torch.float32, device=A_blk.device)
        ws = self.workspace(m, A_blk.device)
        _check(self._lib.sketch_apply_block(self._h, A_blk.data_ptr(), m, k, A_blk.stride(0), int(k0),
                                            out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel() * 4,
                                            _stream_ptr(stream)))
        return out

    # ------------------------------------------------------------------ fused reduce-scatter (f1)
    def rs_split(self, m: int, k: int) -> int:
        v = ctypes.c_int32(0)
        _check(self._lib.sketch_rs_split(self._h, ctypes.c_int64(m), ctypes.c_int64(k), ctypes.byref(v)))
        return int(v.value)

    def plan_info(self, m: int, k: int) -> dict:
        """The library's launch plan for an m x k block (sketch_plan_info): rows_per_unit, split,
        cluster_pairs, grid.  Host-side query, no GPU work."""
        v = [ctypes.c_int32(0) for _ in range(4)]
        _check(self._lib.sketch_plan_info(self._h, ctypes.c_int64(m), ctypes.c_int64(k), *[ctypes.byref(x) for x in v]))
        return dict(zip(("rows_per_unit", "split", "cluster_pairs", "grid"), (int(x.value) for x in v)))

    def apply_block_rs(self, A_blk, k0: int, dst_ptrs, piece_rows: int, slot: int, slot_elems: int, split: int,
                       stream=None):
        """Partial B = A_blk Omega[k0:k0+k] stored by the GEMM epilogue into the owners' receive
        buffers (device pointers dst_ptrs, e.g. symmetric-memory peers); see sketch_apply_block_rs."""
        _require_cuda(A_blk)
        m, k = A_blk.shape
        A_blk = _tma_ready(A_blk)
        arr = (ctypes.c_void_p * len(dst_ptrs))(*[ctypes.c_void_p(int(x)) for x in dst_ptrs])
        _check(self._lib.sketch_apply_block_rs(self._h, ctypes.c_void_p(A_blk.data_ptr()), ctypes.c_int64(m),
                                               ctypes.c_int64(k), ctypes.c_int64(A_blk.stride(0)),
                                               ctypes.c_int64(k0), arr, ctypes.c_int32(len(dst_ptrs)),
                                               ctypes.c_int64(piece_rows), ctypes.c_int32(slot),
                                               ctypes.c_int64(slot_elems), ctypes.c_int32(split),
                                               _stream_ptr(stream)))

    def reduce_slots(self, slots, nslots: int, slot_elems: int, rows: int, out=None, stream=None):
        """out[rows x r] = sum of the nslots receive slots, fixed order (owner side of the fused RS)."""
        torch = _torch()
        _require_cuda(slots, out)
        if out is None:
            out = torch.empty((rows, self.r), dtype=torch.float32, device=slots.device)
        _check(self._lib.sketch_reduce_slots(self._h, ctypes.c_void_p(slots.data_ptr()), ctypes.c_int32(nslots),
                                             ctypes.c_int64(slot_elems), ctypes.c_int64(rows),
                                             ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(out.stride(0)),
                                             _stream_ptr(stream)))
        return out

    def core_block(self, B_blk, i0: int, out=None, stream=None):
        """C_part = Omega[i0:i0+m]^T B_blk (Alg. 2 second product)."""
        torch = _torch()
        _require_cuda(B_blk, out)
        m = B_blk.shape[0]
        if out is None:
            out = torch.empty((self.r, self.r), dtype=torch.float32, device=B_blk.device)
        ws = self.workspace(m, B_blk.device)
        _check(self._lib.core_apply_block(self._h, B_blk.data_ptr(), m, B_blk.stride(0), int(i0),
                                          out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel() * 4,
                                          _stream_ptr(stream)))
        return out

    def core_block_mc(self, B_blk, i0: int, c_mc: int, ldc: int, stream=None):
        """Adds Omega[i0:i0+m]^T B_blk into C on every rank of a multicast group (core_apply_block_mc)."""
        _require_cuda(B_blk)
        m = B_blk.shape[0]
        ws = self.workspace(m, B_blk.device)
        _check(self._lib.core_apply_block_mc(self._h, ctypes.c_void_p(B_blk.data_ptr()), ctypes.c_int64(m),
                                             ctypes.c_int64(B_blk.stride(0) if m else self.r), ctypes.c_int64(i0),
                                             ctypes.c_void_p(int(c_mc)), ctypes.c_int64(ldc),
                                             ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel() * 4),
                                             _stream_ptr(stream)))

    def core_block_cols(self, B_blk, i0: int, out=None, stream=None):
        """C[:, cols] = Omega[i0:i0+m]^T B_blk for a column block of B (Redist variant)."""
        torch = _torch()
        _require_cuda(B_blk, out)
        m, nb = B_blk.shape
        if out is None:
            out = torch.empty((self.r, nb), dtype=torch.float32, device=B_blk.device)
        ws = self.workspace(m, B_blk.device)
        _check(self._lib.core_apply_block_cols(self._h, B_blk.data_ptr(), m, nb, B_blk.stride(0), int(i0),
                                               out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel() * 4,
                                               _stream_ptr(stream)))
        return out

    def pack_cols(self, B_blk, col_bounds, out=None, stream=None):
        """Column blocks of B_blk packed back to back (Redist All-to-All send buffer, sketch_pack_cols)."""
        torch = _torch()
        _require_cuda(B_blk, out)
        rows = B_blk.shape[0]
        nblk = len(col_bounds) - 1
        if out is None:
            out = torch.empty(rows * int(col_bounds[-1]), dtype=torch.float32, device=B_blk.device)
        cb = (ctypes.c_int64 * len(col_bounds))(*[int(x) for x in col_bounds])
        _check(self._lib.sketch_pack_cols(ctypes.c_void_p(B_blk.data_ptr()), ctypes.c_int64(rows),
                                          ctypes.c_int64(B_blk.stride(0) if rows else 1), cb, ctypes.c_int32(nblk),
                                          ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def nystrom_core(self, A, B=None, C=None, stream=None):
        """(B, C) = (A Omega, Omega^T A Omega) for square A."""
        torch = _torch()
        _require_cuda(A, B, C)
        n = A.shape[0]
        A = _tma_ready(A)
        if B is None:
            B = torch.empty((n, self.r), dtype=torch.float32, device=A.device)
        if C is None:
            C = torch.empty((self.r, self.r), dtype=torch.float32, device=A.device)
        ws = self.workspace(n, A.device)
        _check(self._lib.nystrom_core(self._h, A.data_ptr(), n, A.stride(0), B.data_ptr(), B.stride(0),
                                      C.data_ptr(), C.stride(0), ws.data_ptr(), ws.numel() * 4,
                                      _stream_ptr(stream)))
        return B, C

    # ------------------------------------------------------------------ host buffers / out-of-core
    def _host_ws(self, n1: int, block_rows: int):
        torch = _torch()
        n = ctypes.c_size_t()
        _check(self._lib.sketch_host_workspace_size(self._h, int(n1), int(block_rows), ctypes.byref(n)))
        key = ("host", torch.cuda.current_device(), int(n1), int(block_rows))
        ws = self._ws.get(key)
        if ws is None:
            ws = torch.empty(max(n.value, 16) // 4 + 4, dtype=torch.float32, device="cuda")
            self._ws[key] = ws
        return ws

    def apply_host(self, A, out=None, block_rows: int = 0, stream=None, sync: bool = True):
        """B = A Omega for a HOST (CPU) fp32 A, streamed through the GPU in row blocks.

        Pin A (A.pin_memory()) for full PCIe bandwidth.  Returns a CPU tensor (pinned if out is None)."""
        torch = _torch()
        _require_cuda()
        if A.is_cuda or A.dtype != torch.float32 or A.stride(1) != 1:
            raise SketchError(1, "SK_ERR_INVALID_VALUE", "expected a row-major fp32 CPU tensor")
        n1, n2 = A.shape
        if out is None:
            out = torch.empty((n1, self.r), dtype=torch.float32, pin_memory=True)
        ws = self._host_ws(n1, block_rows)
        _check(self._lib.sketch_apply_host(self._h, A.data_ptr(), n1, n2, A.stride(0), out.data_ptr(),
                                           out.stride(0), int(block_rows), ws.data_ptr(), ws.numel() * 4,
                                           _stream_ptr(stream)))
        if sync:
            (stream or torch.cuda.current_stream()).synchronize()
        return out

    def nystrom_core_host(self, A, B=None, C=None, block_rows: int = 0, stream=None, sync: bool = True):
        """(B, C) for a HOST square A streamed in row blocks (out-of-core Nystrom core)."""
        torch = _torch()
        _require_cuda()
        if A.is_cuda or A.dtype != torch.float32 or A.stride(1) != 1:
            raise SketchError(1, "SK_ERR_INVALID_VALUE", "expected a row-major fp32 CPU tensor")
        n = A.shape[0]
        if B is None:
            B = torch.empty((n, self.r), dtype=torch.float32, pin_memory=True)
        if C is None:
            C = torch.empty((self.r, self.r), dtype=torch.float32, pin_memory=True)
        ws = self._host_ws(n, block_rows)
        _check(self._lib.nystrom_core_host(self._h, A.data_ptr(), n, A.stride(0), B.data_ptr(), B.stride(0),
                                           C.data_ptr(), C.stride(0), int(block_rows), ws.data_ptr(),
                                           ws.numel() * 4, _stream_ptr(stream)))
        if sync:
            (stream or torch.cuda.current_stream()).synchronize()
        return B, C

    # ------------------------------------------------------------------ test / debug
    def generate(self, row0: int, nrows: int, col0: int = 0, ncols=None, stream=None):
        torch = _torch()
        _require_cuda()
        ncols = self.r - col0 if ncols is None else ncols
        out = torch.empty((nrows, ncols), dtype=torch.float32, device="cuda")
        _check(self._lib.sketch_generate(self._h, row0, nrows, col0, ncols, out.data_ptr(),
                                         max(ncols, 1), _stream_ptr(stream)))
        return out

    def generate_bits(self, row0: int, nrows: int, col0: int = 0, ncols=None, stream=None):
        torch = _torch()
        _require_cuda()
        ncols = self.r - col0 if ncols is None else ncols
        out = torch.empty((nrows, ncols), dtype=torch.int32, device="cuda")
        _check(self._lib.sketch_generate_bits(self._h, row0, nrows, col0, ncols, out.data_ptr(),
                                              max(ncols, 1), _stream_ptr(stream)))
        return out


def sum_peers(src_ptrs, elems: int, out, stream=None):
    """out[:elems] = sum of the float32 buffers at the device pointers src_ptrs, in list order
    (the fused AllReduce of C; see sketch_sum_peers)."""
    _require_cuda(out)
    arr = (ctypes.c_void_p * len(src_ptrs))(*[ctypes.c_void_p(int(x)) for x in src_ptrs])
    _check(load_library().sketch_sum_peers(arr, ctypes.c_int32(len(src_ptrs)), ctypes.c_int64(elems),
                                           ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out


def multimem_sum(mc_src: int, elems: int, out=None, mc_out: int = 0, stream=None):
    """out[:elems] = sum over the multicast group's ranks of element i at the multicast address mc_src
    (NVLS in-switch reduction; see sketch_multimem_sum); optionally broadcast to mc_out."""
    _require_cuda(out)
    _check(load_library().sketch_multimem_sum(ctypes.c_void_p(int(mc_src)), ctypes.c_int64(elems),
                                              ctypes.c_void_p(out.data_ptr() if out is not None else 0),
                                              ctypes.c_void_p(int(mc_out)), _stream_ptr(stream)))
    return out


def launch_count() -> int:
    """Kernels launched by libsketch.so in this process so far."""
    return int(load_library().sketch_launch_count())


def debug_box_muller(w1, w2, transform: str = "accurate", stream=None):
    """Device Box-Muller on word pairs (int32 CUDA tensors holding uint32 bits)."""
    torch = _torch()
    lib = load_library()
    _require_cuda()
    n = w1.numel()
    oe = torch.empty(n, dtype=torch.float32, device=w1.device)
    oo = torch.empty(n, dtype=torch.float32, device=w1.device)
    _check(lib.sketch_debug_box_muller(w1.data_ptr(), w2.data_ptr(), n, _OMEGA[transform],
                                       oe.data_ptr(), oo.data_ptr(), _stream_ptr(stream)))
    return oe, oo
