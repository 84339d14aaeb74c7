"""Nyström reconstruction and its error (post-processing, not on the timed path).

The paper forms the Nyström approximation  A~ = (A Omega)(Omega^T A Omega)^+ (A Omega)^T
 and, for its accuracy table, builds the pseudoinverse of the core with a numerical
tolerance of 1e-12 and measures the relative error of the explicit reconstruction
(Table 2).

Here B and C come from the sketch kernels; the r x r pseudoinverse and the error use torch linear
algebra in fp64 (library routines on tiny / blocked problems, like the paper's own post-processing).
The error is evaluated block by block without materialising the n x n approximation: for each row
block A_i, E_i = A_i - (B_i W) B^T (W = C^+) is formed and ||E_i||_F^2 accumulated in fp64.  (The
trace identity ||A||^2 - 2 tr(W B^T A B) + tr(W G W G) cancels catastrophically when the error is
small and C^+ is ill-conditioned, so it is not used.)
"""
from __future__ import annotations


def pinv_sym(C, rtol: float = 1e-12):
    """Moore-Penrose pseudoinverse of the (symmetrised) core, eigenvalues below rtol * max|lambda|
    dropped.  Returns fp64."""
    import torch
    Cs = 0.5 * (C.double() + C.double().T)
    lam, V = torch.linalg.eigh(Cs)
    cut = rtol * lam.abs().max()
    inv = torch.where(lam.abs() > cut, 1.0 / lam, torch.zeros_like(lam))
    return (V * inv) @ V.T


def reconstruction_error(A, B, C, rtol: float = 1e-12, block_rows: int = 8192) -> float:
    """Relative Frobenius error ||A - B C^+ B^T||_F / ||A||_F (fp64 accumulation, blocked over A)."""
    import torch
    W = pinv_sym(C, rtol)
    Bd = B.double()
    BW = Bd @ W
    a2 = 0.0
    e2 = 0.0
    n = A.shape[0]
    for i in range(0, n, block_rows):
        Ai = A[i:i + block_rows].double()
        a2 += float((Ai * Ai).sum())
        Ei = Ai - BW[i:i + block_rows] @ Bd.T
        e2 += float((Ei * Ei).sum())
    return e2 ** 0.5 / max(a2, 1e-300) ** 0.5
