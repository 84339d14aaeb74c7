"""Seeded synthetic inputs shared by tests/ and bench.py.

This module holds NONE of the method's arithmetic (no Philox, no Omega, no
products with Omega): only the matrices A that the sketch is applied to, with
the shapes and value distributions of the paper's workloads (DESIGN.md
"Input recipe"):

  * ``uniform``      iid U[-1/2, 1/2) fp32, the data-matrix stand-in for the
                     tall-skinny / short-wide configs ("different
                     dimensions and aspect ratios").
  * ``rbf_kernel``   RBF kernel exp(-|x_i - x_j|^2 / (2 sigma^2)) of X ~ U[0,1)^{n x d},
                     sigma = |X|_F / sqrt(n) -- the synthetic analogue of the
                     CIFAR-10 kernel matrices of PAPER.md:1013-1024 (sigma rule of
                     Table 2); symmetric PSD.
  * ``int_matrix``   integers in [lo, hi] (the integer-exact regime).
  * ``lowrank_psd``  X X^T with integer X (exact, PSD, rank <= d).

Host versions return numpy arrays (used for parity tests, where the very same
array is handed to the oracle and uploaded to the GPU); ``*_device`` versions
build large inputs directly in HBM with torch (bench only).
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform(seed: int, n1: int, n2: int) -> np.ndarray:
    return (_rng(seed).random((n1, n2), dtype=np.float32) - np.float32(0.5)).astype(np.float32)


def symmetric_uniform(seed: int, n: int) -> np.ndarray:
    g = uniform(seed, n, n)
    return ((g + g.T) * np.float32(0.5)).astype(np.float32)


def int_matrix(seed: int, n1: int, n2: int, lo: int = -4, hi: int = 4, symmetric: bool = False) -> np.ndarray:
    a = _rng(seed).integers(lo, hi + 1, size=(n1, n2)).astype(np.float32)
    if symmetric:
        assert n1 == n2
        a = np.triu(a) + np.triu(a, 1).T
    return a


def lowrank_psd(seed: int, n: int, d: int, lo: int = -2, hi: int = 2) -> tuple:
    """Returns (A, X) with A = X X^T, X integer n x d (exact in fp32 when n*d*hi^2 < 2^24)."""
    X = _rng(seed).integers(lo, hi + 1, size=(n, d)).astype(np.float64)
    A = X @ X.T
    return A.astype(np.float32), X


def rbf_kernel(seed: int, n: int, d: int) -> np.ndarray:
    X = _rng(seed).random((n, d))
    sigma = np.linalg.norm(X) / np.sqrt(n)
    sq = (X * X).sum(1)
    D2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * (X @ X.T), 0.0)
    A = np.exp(-D2 / (2.0 * sigma * sigma)).astype(np.float32)
    return np.triu(A) + np.triu(A, 1).T


# ----------------------------------------------------------------------------
# Device-side generators (bench: inputs created in HBM, never on the host).
# ----------------------------------------------------------------------------

def uniform_device(seed: int, n1: int, n2: int, device="cuda", out=None):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if out is None:
        out = torch.empty((n1, n2), dtype=torch.float32, device=device)
    # fill in row chunks to bound the temporary footprint
    step = max(1, (1 << 28) // max(n2, 1))
    for i in range(0, n1, step):
        blk = out[i:i + step]
        blk.uniform_(-0.5, 0.5, generator=g)
    return out


def int_matrix_device(seed: int, n1: int, n2: int, lo: int = -4, hi: int = 4, device="cuda", out=None):
    """iid integers in [lo, hi] as fp32, generated in HBM in row chunks (full-size integer-regime tests)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if out is None:
        out = torch.empty((n1, n2), dtype=torch.float32, device=device)
    step = max(1, (1 << 27) // max(n2, 1))
    for i in range(0, n1, step):
        blk = out[i:i + step]
        blk.copy_(torch.randint(lo, hi + 1, blk.shape, generator=g, device=device, dtype=torch.int32))
    return out


def rbf_kernel_device(seed: int, n: int, d: int, device="cuda", out=None, chunk: int = 8192):
    """RBF kernel of X ~ U[0,1)^{n x d} built in row blocks on the GPU (fp64 distances)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    X = torch.rand((n, d), generator=g, device=device, dtype=torch.float64)
    sigma2 = float((X * X).sum()) / n
    sq = (X * X).sum(1)
    if out is None:
        out = torch.empty((n, n), dtype=torch.float32, device=device)
    for i in range(0, n, chunk):
        xi = X[i:i + chunk]
        d2 = (sq[i:i + chunk, None] + sq[None, :] - 2.0 * (xi @ X.T)).clamp_min_(0.0)
        out[i:i + chunk] = torch.exp(-d2 / (2.0 * sigma2)).to(torch.float32)
    # exact symmetry (upper triangle mirrored), as in the host recipe
    for i in range(0, n, chunk):
        for j in range(0, i, chunk):
            out[i:i + chunk, j:j + chunk] = out[j:j + chunk, i:i + chunk].T
    del X, sq
    return out
