"""Oracle for the applications of SURVEY §8(f) F-4, integer arithmetic (int64 / exact).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and nothing on the
product path.  Shares no code with paper_2501_13664_b200/.

* Ray denoising (PAPER.md:448 and the caption of fig:output3DDJT): "a thresholding of the highest
  amplitude coefficients, and subsequent backprojection, eliminates most of the noise":
  denoise(f) = A_J^T threshold(A_J f).
* Plane detection: "the plane that accumulated the greatest number of voxels is
  detected in the transformed space, and then those that are orthogonal to it, and simultaneously
  are relative maxima and exceed a threshold".

Readings (R19-R22):
  R19  threshold: keep c when c * den >= num * max(c) (max over the whole call), an exact integer
       test of c >= (num/den) max; other coefficients become 0.
  R20  "the plane that accumulated the greatest number of voxels": the global argmax over all
       dodecants' coefficients, ties to the smallest index in the stacked layout [k][s1][s2][D].
  R21  "relative maxima": c >= every neighbour in the 26-neighbourhood of (s1, s2, D) inside the
       same dodecant, and c > the neighbours with a smaller linear index (one representative per
       plateau).
  R22  plane normals: the dodecant-k plane z' = l_{s1}(x') + l_{s2}(y') + delta has slope s/(N-1)
       per axis (l_s(N-1) = s, eq:digitalLine), so its oriented normal is (s1, s2, -(N-1)); the
       orientation (reading A) is a signed axis permutation, which maps it to
       the original axes: n[|p_j| - 1] = sign(p_j) n'_j.  "Orthogonal": |cos| <= onum/oden, tested
       exactly as (n . m)^2 oden^2 <= onum^2 |n|^2 |m|^2 in integers.
"""
from __future__ import annotations

import numpy as np

from . import djt_lines, djt_lines_adjoint, tables


def threshold(coef: np.ndarray, num: int, den: int) -> np.ndarray:
    """R19: c if c * den >= num * max(c) else 0."""
    c = np.asarray(coef).astype(np.int64)
    mx = int(c.max())
    return np.where(c * den >= num * mx, c, 0)


def denoise_rays(cube: np.ndarray, mask: int, num: int, den: int, table: int = tables.TABLE_HEMISPHERE):
    """A_J^T threshold(A_J f) for one cube [N][N][N]: returns (kept coefficients,
    backprojection), int64."""
    c = djt_lines(cube, mask, table)
    kept = threshold(c, num, den)
    return kept, djt_lines_adjoint(kept, mask, table)


def argmax(coef: np.ndarray) -> int:
    """R20: flat index of the largest coefficient, smallest index among ties."""
    return int(np.argmax(np.asarray(coef).reshape(-1)))


def plane_normal(k: int, s1: int, s2: int, N: int, table: int = tables.TABLE_HEMISPHERE):
    """R22: integer normal, in the original axes, of the plane family (k, s1, s2)."""
    row = tables.table(table, "drt")[k]
    npr = (s1, s2, -(N - 1))
    n = [0, 0, 0]
    for j, p in enumerate(row):
        n[abs(p) - 1] = (1 if p > 0 else -1) * npr[j]
    return n


def is_relative_max(c: np.ndarray, j: int, s1: int, s2: int, D: int) -> bool:
    """R21 on c[k] = c[j] of shape [N][N][3N]."""
    a = c[j]
    v = a[s1, s2, D]
    N, W = a.shape[0], a.shape[2]
    for d1 in (-1, 0, 1):
        for d2 in (-1, 0, 1):
            for d3 in (-1, 0, 1):
                if d1 == d2 == d3 == 0:
                    continue
                t1, t2, t3 = s1 + d1, s2 + d2, D + d3
                if not (0 <= t1 < N and 0 <= t2 < N and 0 <= t3 < W):
                    continue
                u = a[t1, t2, t3]
                smaller_index = (d1, d2, d3) < (0, 0, 0)        # lexicographic = linear order
                if u > v or (smaller_index and u == v):
                    return False
    return True


def detect_planes(coef: np.ndarray, mask: int, num: int, den: int, onum: int, oden: int,
                  table: int = tables.TABLE_HEMISPHERE):
    """PAPER.md:669-679 on stacked DRT coefficients [K][N][N][3N] (K = popcount(mask)):
    returns (flags uint8 [K][N][N][3N], argmax flat index).  flags = 1 for the argmax plane and
    for every coefficient that exceeds the R19 threshold, is a relative maximum (R21) and whose
    plane is orthogonal to the argmax plane (R22)."""
    c = np.asarray(coef).astype(np.int64)
    K, N = c.shape[0], c.shape[1]
    ks = [k for k in range(12) if (mask >> k) & 1]
    am = argmax(c)
    j0, s10, s20, _ = np.unravel_index(am, c.shape)
    m = plane_normal(ks[j0], int(s10), int(s20), N, table)
    mm = sum(x * x for x in m)
    mx = int(c.reshape(-1)[am])
    flags = np.zeros(c.shape, np.uint8)
    flags.reshape(-1)[am] = 1
    cand = np.argwhere(c * den >= num * mx)
    for j, s1, s2, D in cand:
        n = plane_normal(ks[j], int(s1), int(s2), N, table)
        dot = sum(a * b for a, b in zip(n, m))
        nn = sum(x * x for x in n)
        if dot * dot * oden * oden > onum * onum * nn * mm:
            continue
        if is_relative_max(c, int(j), int(s1), int(s2), int(D)):
            flags[j, s1, s2, D] = 1
    return flags, am
