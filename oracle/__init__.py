"""oracle/ -- TEST INFRASTRUCTURE ONLY (not part of the product path).

Plain, slow, obviously-correct fp64 CPU reference for B = A*Omega and
C = Omega^T*B with Omega regenerated from Philox4x32-10 (reading O1 in
DESIGN.md; sec. 1, sec. 6.3).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2603_20966_b200`` (the CUDA path) and never
imports it.

Parity status per function:
  philox4x32_10   pinned: Random123 known-answer vectors (tests/golden/philox_kat.txt)
  omega_words     pinned: zero-KAT by construction; SURVEY Appendix A worked values
  box_muller      pinned: closed forms (u2 = 0, 1/4, 1/2, 3/4; u1 = 1; max |z|),
                  moments / KS against N(0,1) (scipy), E[Omega Omega^T]/r = I
  omega (values)  pinned: as above + Rademacher balance, diag(Omega^T Omega) = n2
  sketch          pinned: numpy matmul on materialised Omega, A = I / e_i e_j^T / 0,
                  brute force on tiny inputs, integer-exact regime
  core            pinned: associativity (Omega^T A) Omega, symmetry, A = I,
                  closed form for A = X X^T, exact Nystrom recovery
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GAUSSIAN, RADEMACHER, UNIFORM = 0, 1, 2
DISTS = {"gaussian": GAUSSIAN, "rademacher": RADEMACHER, "uniform": UNIFORM}


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp, no -ffast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            f32p = ctypes.POINTER(ctypes.c_float)
            f64p = ctypes.POINTER(ctypes.c_double)
            i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
            lib.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
            lib.oracle_omega_word.argtypes = [u64, i32, u64, u64]
            lib.oracle_omega_word.restype = ctypes.c_uint32
            lib.oracle_omega_value.argtypes = [u64, i32, u64, u64]
            lib.oracle_omega_value.restype = ctypes.c_float
            lib.oracle_box_muller.argtypes = [ctypes.c_uint32, ctypes.c_uint32, f64p, f64p]
            lib.oracle_omega.argtypes = [u64, i32, i64, i64, i64, i64, f32p, i64]
            lib.oracle_omega_words.argtypes = [u64, i32, i64, i64, i64, i64, u32p, i64]
            lib.oracle_sketch.argtypes = [u64, i32, f32p, i64, i64, i64, i64, i64, f64p, i64]
            lib.oracle_core.argtypes = [u64, i32, f64p, i64, i64, i64, i64, f64p, i64]
            lib.oracle_box_muller_many.argtypes = [u32p, u32p, i64, f32p, f32p]
            lib.oracle_num_threads.restype = i32
            lib.oracle_set_num_threads.argtypes = [i32]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _dist(d) -> int:
    return DISTS[d] if isinstance(d, str) else int(d)


def philox4x32_10(ctr, key) -> tuple:
    lib = _load()
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib.oracle_philox4x32_10(_ptr(c, ctypes.c_uint32), _ptr(k, ctypes.c_uint32), _ptr(out, ctypes.c_uint32))
    return tuple(int(v) for v in out)


def box_muller(w1: int, w2: int) -> tuple:
    """fp64 (z_even, z_odd) from the two raw words of a pair (not rounded)."""
    lib = _load()
    ze, zo = ctypes.c_double(), ctypes.c_double()
    lib.oracle_box_muller(ctypes.c_uint32(w1), ctypes.c_uint32(w2), ctypes.byref(ze), ctypes.byref(zo))
    return ze.value, zo.value


def box_muller_many(w1: np.ndarray, w2: np.ndarray) -> tuple:
    """Correctly rounded fp32 (z_even, z_odd) for arrays of word pairs."""
    lib = _load()
    w1 = np.ascontiguousarray(w1, dtype=np.uint32)
    w2 = np.ascontiguousarray(w2, dtype=np.uint32)
    n = w1.size
    ze = np.empty(n, dtype=np.float32)
    zo = np.empty(n, dtype=np.float32)
    if n:
        lib.oracle_box_muller_many(_ptr(w1, ctypes.c_uint32), _ptr(w2, ctypes.c_uint32), n,
                                   _ptr(ze, ctypes.c_float), _ptr(zo, ctypes.c_float))
    return ze, zo


def omega(seed: int, dist, row0: int, nrows: int, col0: int, ncols: int) -> np.ndarray:
    """fp32 Omega[row0:row0+nrows, col0:col0+ncols] (each entry rounded once from fp64)."""
    lib = _load()
    out = np.empty((nrows, ncols), dtype=np.float32)
    if nrows and ncols:
        lib.oracle_omega(seed, _dist(dist), row0, nrows, col0, ncols, _ptr(out, ctypes.c_float), ncols)
    return out


def omega_words(seed: int, dist, row0: int, nrows: int, col0: int, ncols: int) -> np.ndarray:
    """Raw Philox word each entry is derived from (x[j&3] for tag 0, x[(j>>5)&3] for tag 1)."""
    lib = _load()
    out = np.empty((nrows, ncols), dtype=np.uint32)
    if nrows and ncols:
        lib.oracle_omega_words(seed, _dist(dist), row0, nrows, col0, ncols, _ptr(out, ctypes.c_uint32), ncols)
    return out


def sketch(seed: int, dist, A: np.ndarray, r: int, k0: int = 0) -> np.ndarray:
    """fp64 B = A * Omega[k0:k0+n2, :r] for fp32 A (n1 x n2)."""
    lib = _load()
    A = np.ascontiguousarray(A, dtype=np.float32)
    n1, n2 = A.shape
    B = np.zeros((n1, r), dtype=np.float64)
    if n1 and n2 and r:
        lib.oracle_sketch(seed, _dist(dist), _ptr(A, ctypes.c_float), n1, n2, n2, k0, r,
                          _ptr(B, ctypes.c_double), r)
    return B


def core(seed: int, dist, B: np.ndarray, i0: int = 0) -> np.ndarray:
    """fp64 C = Omega[i0:i0+n, :r]^T * B for fp64 B (n x r)."""
    lib = _load()
    B = np.ascontiguousarray(B, dtype=np.float64)
    n, r = B.shape
    C = np.zeros((r, r), dtype=np.float64)
    if r:
        lib.oracle_core(seed, _dist(dist), _ptr(B, ctypes.c_double), n, r, i0, r,
                        _ptr(C, ctypes.c_double), r)
    return C


def nystrom_core(seed: int, dist, A: np.ndarray, r: int) -> tuple:
    """(B, C) = (A Omega, Omega^T A Omega) for square A."""
    B = sketch(seed, dist, A, r)
    return B, core(seed, dist, B)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))
