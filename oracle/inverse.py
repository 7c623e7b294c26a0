"""Oracle for the iterative inverse of the 3D DRT, fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and nothing on the
product path.  Shares no code with paper_2501_13664_b200/.

What the paper fixes (§"Radon and John 3D inverse transforms"):
  * the adjoint (backprojection, eq:invmap3Dsummation) is "an approximate inverse operator of
    the DRT in the theory of iterative improvement of a solution to linear equations"
    (Press, Numerical Recipes §2.5): x <- x + B (b - A x);
  * the 3D high-pass filter h: centre 7/8, face neighbours -1/16, edge
    neighbours -1/32, corner neighbours -1/64 (zero DC response);
  * a prolongation/restriction multigrid accelerator (eq. after), cycle unspecified.

Readings taken here (R15-R18):
  R15  B r = alpha * h * (A^T r): the filtered backprojection; A = the stacked DRT over the
       dodecants of `mask`, A^T its adjoint (sum of the per-dodecant backprojections).
  R16  the scale alpha, which the paper leaves to the method, is the residual-minimising step
       alpha_k = <r_k, A p_k> / <A p_k, A p_k> with p_k = h * A^T r_k, recomputed every iteration
       (so ||r_k|| never increases); the residual is updated as r <- r - alpha A p.
  R17  h is applied with zero padding outside the cube.
  R18  the multigrid cycle (unspecified) is a recursive approximate inverse B (mg_apply): restrict
       the residual with S, solve the half-size problem recursively, prolongate with P, then one
       R16 filtered-backprojection step on the remaining residual at this size; the coarsest size
       n_min uses the R16 step alone.  n_min = N is the single-grid iteration (press_refine).
Every step is written in the order of the iteration above; the DRT / adjoint steps call the
pinned oracle transforms (oracle.drt_planes, oracle.drt_planes_adjoint).
"""
from __future__ import annotations

import numpy as np

from . import drt_planes, drt_planes_adjoint, tables

# h(1,1,1) = 7/8, then by the number of non-centre coordinates: 1 -> -1/16, 2 -> -1/32, 3 -> -1/64
#
H_WEIGHTS = {0: 7.0 / 8.0, 1: -1.0 / 16.0, 2: -1.0 / 32.0, 3: -1.0 / 64.0}


def highpass_kernel() -> np.ndarray:
    """The 3x3x3 filter h of PAPER.md:576-591 as an array h[a][b][c], a,b,c in {0,1,2}."""
    h = np.zeros((3, 3, 3), np.float64)
    for a in range(3):
        for b in range(3):
            for c in range(3):
                h[a, b, c] = H_WEIGHTS[(a != 1) + (b != 1) + (c != 1)]
    return h


def highpass(g: np.ndarray) -> np.ndarray:
    """(h * g)[x,y,z] = sum_{a,b,c} h[a][b][c] g[x+a-1, y+b-1, z+c-1], zero outside the cube (R17)."""
    g = np.asarray(g, np.float64)
    N = g.shape[0]
    pad = np.zeros((N + 2, N + 2, N + 2), np.float64)
    pad[1:-1, 1:-1, 1:-1] = g
    h = highpass_kernel()
    out = np.zeros_like(g)
    for a in range(3):
        for b in range(3):
            for c in range(3):
                out += h[a, b, c] * pad[a:a + N, b:b + N, c:c + N]
    return out


def press_refine(coef: np.ndarray, iters: int, mask: int = 0xFFF, table: int = tables.TABLE_HEMISPHERE,
                 x0: np.ndarray | None = None):
    """Iterative improvement x <- x + alpha_k h*(A^T r_k) (R15-R17) for `iters` iterations.

    coef: stacked DRT coefficients [K][N][N][3N] (the b of A x = b).  Returns (x, rnorm) with
    rnorm[k] = ||r_k||_2 before iteration k and rnorm[iters] after the last one.
    """
    b = np.asarray(coef, np.float64)
    N = b.shape[1]
    x = np.zeros((N, N, N), np.float64) if x0 is None else np.array(x0, np.float64)
    r = b - drt_planes(x, mask, table) if x0 is not None else b.copy()
    rnorm = [float(np.sqrt(np.sum(r * r)))]
    for _ in range(iters):
        g = drt_planes_adjoint(r, mask, table)      # A^T r
        p = highpass(g)                             # h * A^T r
        q = drt_planes(p, mask, table)              # A p
        qq = float(np.sum(q * q))
        alpha = float(np.sum(r * q)) / qq if qq > 0 else 0.0
        x = x + alpha * p
        r = r - alpha * q
        rnorm.append(float(np.sqrt(np.sum(r * r))))
    return x, np.array(rnorm)


def nrmsd(x: np.ndarray, f: np.ndarray) -> float:
    """Normalised root-mean-square deviation: ||x - f||_2 / ||f||_2."""
    f = np.asarray(f, np.float64)
    return float(np.linalg.norm(np.asarray(x, np.float64) - f) / np.linalg.norm(f))


# ---------------------------------------------------------------- multigrid

def prolong(xc: np.ndarray) -> np.ndarray:
    """P: f^N_{i+a, j+b, k+c} = f^{N/2}_{floor(i/2), floor(j/2), floor(k/2)}, i.e.
    every coarse voxel fills its 2x2x2 block of the fine cube."""
    xc = np.asarray(xc, np.float64)
    return xc.repeat(2, axis=0).repeat(2, axis=1).repeat(2, axis=2)


def restrict(coef: np.ndarray) -> np.ndarray:
    """S, per dodecant: R^{N/2}(s1, s2, d) = 1/8 [R^N(2 s1, 2 s2, 2 d) + R^N(2 s1, 2 s2, 2 d + 1)]
    on the stacked layout [K][N][N][3N] -> [K][N/2][N/2][3N/2]."""
    c = np.asarray(coef, np.float64)
    return 0.125 * (c[:, 0::2, 0::2, 0::2] + c[:, 0::2, 0::2, 1::2])


def _min_residual_step(r, mask, table):
    """p = h * A^T r and the step alpha = <r, A p> / <A p, A p> (R15-R16); returns (alpha p, alpha A p)."""
    p = highpass(drt_planes_adjoint(r, mask, table))
    q = drt_planes(p, mask, table)
    qq = float(np.sum(q * q))
    alpha = float(np.sum(r * q)) / qq if qq > 0 else 0.0
    return alpha * p, alpha * q


def mg_apply(r: np.ndarray, mask: int = 0xFFF, table: int = tables.TABLE_HEMISPHERE, n_min: int = 2):
    """Multigrid approximate inverse B r (reading R18): at the coarsest size n_min
    B r = alpha h*(A^T r); above it
        e  = P B_{N/2}(S r)                    (coarse correction, prolongated)
        r' = r - A e
        e  = e + alpha' h*(A^T r')             (fine-level filtered backprojection, R16 step)
    Returns (e, A e) so the caller can update its residual without another transform."""
    r = np.asarray(r, np.float64)
    N = r.shape[1]
    if N <= n_min:
        return _min_residual_step(r, mask, table)
    ec, _ = mg_apply(restrict(r), mask, table, n_min)
    e = prolong(ec)
    ae = drt_planes(e, mask, table)
    dp, dq = _min_residual_step(r - ae, mask, table)
    return e + dp, ae + dq


def press_multigrid(coef: np.ndarray, iters: int, mask: int = 0xFFF, table: int = tables.TABLE_HEMISPHERE,
                    n_min: int = 2):
    """Iterative improvement x <- x + B (b - A x) with the multigrid B of `mg_apply` (PAPER.md:575,
    R18), x_0 = 0.  Returns (x, rnorm) with rnorm[k] = ||b - A x_k||."""
    b = np.asarray(coef, np.float64)
    N = b.shape[1]
    x = np.zeros((N, N, N), np.float64)
    r = b.copy()
    rnorm = [float(np.sqrt(np.sum(r * r)))]
    for _ in range(iters):
        e, ae = mg_apply(r, mask, table, n_min)
        x = x + e
        r = r - ae
        rnorm.append(float(np.sqrt(np.sum(r * r))))
    return x, np.array(rnorm)
