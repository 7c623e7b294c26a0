"""CPU oracle for arXiv 2501.13664 (3D DRT of planes, 3D DJT of lines).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / `--impl reference` legs of bench.py, never by the product path
(paper_2501_13664_b200/).  Shares no code with the CUDA library.

The arithmetic lives in oracle.c (plain single-threaded C, int64 / fp64), a
transcription of PAPER.md's definitions and algorithms; this module only
marshals numpy arrays, applies the orientation (reading A: numpy transpose and
flip, Alg. 2) and assembles the stacked / mosaic layouts.

Parity status per function: every function below is
pinned by tests/test_oracle_*.py; `mosaic` by its block placement and by the
seams of fig:shapeOutput (the shared boundary planes of
neighbouring dodecants sit on facing block edges, reading R13).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import tables

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, no fast-math) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, dbl, p = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        L.oracle_line.restype = i64
        L.oracle_line.argtypes = [ctypes.c_int, i64, i64]
        L.oracle_line_closed.restype = i64
        L.oracle_line_closed.argtypes = [ctypes.c_int, i64, i64, ctypes.c_int]
        for name in ("oracle_drt_brute_f64", "oracle_drt_separable_f64", "oracle_drt_alg1_i64",
                     "oracle_drt_alg1_f64", "oracle_drt_adjoint_f64", "oracle_djt_brute_f64",
                     "oracle_djt_alg3_i64", "oracle_djt_alg3_f64", "oracle_djt_adjoint_f64"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [p, i64, p]
        for name in ("oracle_drt_point_f64", "oracle_drt_point_abs_f64"):
            f = getattr(L, name)
            f.restype = dbl
            f.argtypes = [p, i64, i64, i64, i64]
        L.oracle_djt_point_f64.restype = dbl
        L.oracle_djt_point_f64.argtypes = [p, i64, i64, i64, i64, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _is_float(a) -> bool:
    return np.asarray(a).dtype.kind == "f"


def _as(a, dt):
    return np.ascontiguousarray(np.asarray(a), dtype=dt)


def _n(N: int) -> int:
    n = int(N).bit_length() - 1
    if N < 1 or (1 << n) != N:
        raise ValueError("N must be a power of two")
    return n


# ------------------------------------------------------------------ L0 ----

def line(n: int, s: int, u: int) -> int:
    """l^n_s(u), recursive eq:digitalLine."""
    return int(lib().oracle_line(n, s, u))


def line_closed(n: int, s: int, u: int, real_division: bool) -> int:
    """Closed form of eq:digitalLine, either division reading."""
    return int(lib().oracle_line_closed(n, s, u, int(real_division)))


# --------------------------------------------------------- orientation ----

def orient(f: np.ndarray, row) -> np.ndarray:
    """Alg. 2 permute + flip, reading A:
    oriented axis j = original axis |row[j]|, reversed if row[j] < 0.
    Each row applies to the ORIGINAL cube (reading C-amb-5)."""
    g = np.transpose(f, [abs(p) - 1 for p in row])
    for j, p in enumerate(row):
        if p < 0:
            g = np.flip(g, axis=j)
    return np.ascontiguousarray(g)


# ------------------------------------------------------------- planes ----

def drt_alg1(f: np.ndarray) -> np.ndarray:
    """Alg. 1 basicDRT3D on an (already oriented) cube: [N][N][3N].
    int64 for integer input, fp64 for float input."""
    N = f.shape[0]
    _n(N)
    if _is_float(f):
        g = _as(f, np.float64)
        out = np.zeros((N, N, 3 * N), np.float64)
        lib().oracle_drt_alg1_f64(_ptr(g), N, _ptr(out))
    else:
        g = _as(f, np.int64)
        out = np.zeros((N, N, 3 * N), np.int64)
        lib().oracle_drt_alg1_i64(_ptr(g), N, _ptr(out))
    return out


def drt_brute(f: np.ndarray) -> np.ndarray:
    """eq:3DfDRT by brute force, fp64, O(N^5)."""
    N = f.shape[0]
    _n(N)
    g = _as(f, np.float64)
    out = np.zeros((N, N, 3 * N), np.float64)
    lib().oracle_drt_brute_f64(_ptr(g), N, _ptr(out))
    return out


def drt_separable(f: np.ndarray) -> np.ndarray:
    """eq:3DfDRT as two 2D DRT definitions, fp64, O(5 N^4)."""
    N = f.shape[0]
    _n(N)
    g = _as(f, np.float64)
    out = np.zeros((N, N, 3 * N), np.float64)
    lib().oracle_drt_separable_f64(_ptr(g), N, _ptr(out))
    return out


def drt_point(f: np.ndarray, s1: int, s2: int, D: int, absolute: bool = False) -> float:
    """One eq:3DfDRT output (O(N^2)); absolute=True sums |f| instead."""
    g = _as(f, np.float64)
    fn = lib().oracle_drt_point_abs_f64 if absolute else lib().oracle_drt_point_f64
    return float(fn(_ptr(g), g.shape[0], s1, s2, D))


def drt_adjoint(coef: np.ndarray) -> np.ndarray:
    """Backprojection of one dodecant by eq:invmap3Dsummation."""
    N = coef.shape[0]
    c = _as(coef, np.float64)
    g = np.zeros((N, N, N), np.float64)
    lib().oracle_drt_adjoint_f64(_ptr(c), N, _ptr(g))
    return g


def drt_planes(cube: np.ndarray, mask: int = 0xFFF, table: int = tables.TABLE_HEMISPHERE) -> np.ndarray:
    """Alg. 2 dodecant loop in the stacked layout:
    cube [B][N][N][N] (or [N][N][N]) -> [B][K][N][N][3N], K = popcount(mask),
    dodecants in increasing k."""
    c = np.asarray(cube)
    single = c.ndim == 3
    if single:
        c = c[None]
    rows = tables.table(table, "drt")
    ks = [k for k in range(12) if (mask >> k) & 1]
    out = np.stack([np.stack([drt_alg1(orient(c[b], rows[k])) for k in ks]) for b in range(c.shape[0])])
    return out[0] if single else out


def mosaic(stacked: np.ndarray) -> np.ndarray:
    """Alg. 2 placement of the 12 stacked dodecants
    [12][N][N][3N] into the 4N x 4N x (3N-2) mosaic: block
    DodecantCoords[k], OutOrder[k] applied to (s1, s2) by reading A (permute,
    then flip the permuted axis), d = D - 2.  OutOrder rows 0-3 are the
    repaired rows of reading R13 (tables.MOSAIC_OUT_ORDER), which make the
    dodecants "fit accurately" (fig:shapeOutput)."""
    K, N = stacked.shape[0], stacked.shape[1]
    assert K == 12
    out = np.zeros((4 * N, 4 * N, 3 * N - 2), stacked.dtype)
    for k in range(12):
        o = tables.MOSAIC_OUT_ORDER[k]
        blk = stacked[k][:, :, 2:]
        # permute the (s1, s2) axes by |o0|,|o1| and flip negative ones
        blk = np.transpose(blk, [abs(o[0]) - 1, abs(o[1]) - 1, 2])
        if o[0] < 0:
            blk = blk[::-1]
        if o[1] < 0:
            blk = blk[:, ::-1]
        bi, bj = tables.DODECANT_COORDS[k]
        out[bi * N:(bi + 1) * N, bj * N:(bj + 1) * N, :] = blk
    return out


# -------------------------------------------------------------- lines ----

def djt_alg3(f: np.ndarray) -> np.ndarray:
    """Alg. 3 basicDJT3D on an (already oriented) cube: [N][N][2N][2N]."""
    N = f.shape[0]
    _n(N)
    if _is_float(f):
        g = _as(f, np.float64)
        out = np.zeros((N, N, 2 * N, 2 * N), np.float64)
        lib().oracle_djt_alg3_f64(_ptr(g), N, _ptr(out))
    else:
        g = _as(f, np.int64)
        out = np.zeros((N, N, 2 * N, 2 * N), np.int64)
        lib().oracle_djt_alg3_i64(_ptr(g), N, _ptr(out))
    return out


def djt_brute(f: np.ndarray) -> np.ndarray:
    """eq:3DfDJT by brute force, fp64, O(4 N^5)."""
    N = f.shape[0]
    _n(N)
    g = _as(f, np.float64)
    out = np.zeros((N, N, 2 * N, 2 * N), np.float64)
    lib().oracle_djt_brute_f64(_ptr(g), N, _ptr(out))
    return out


def djt_point(f: np.ndarray, s1: int, s2: int, D1: int, D2: int) -> float:
    g = _as(f, np.float64)
    return float(lib().oracle_djt_point_f64(_ptr(g), g.shape[0], s1, s2, D1, D2))


def djt_adjoint(coef: np.ndarray) -> np.ndarray:
    """Backprojection of one DJT dodecant by eq:invmap3DJsummation."""
    N = coef.shape[0]
    c = _as(coef, np.float64)
    g = np.zeros((N, N, N), np.float64)
    lib().oracle_djt_adjoint_f64(_ptr(c), N, _ptr(g))
    return g


def djt_lines(cube: np.ndarray, mask: int = 0x001, table: int = tables.TABLE_HEMISPHERE) -> np.ndarray:
    """DJT over the dodecants of `mask`: [B][K][N][N][2N][2N]."""
    c = np.asarray(cube)
    single = c.ndim == 3
    if single:
        c = c[None]
    rows = tables.table(table, "djt")
    ks = [k for k in range(12) if (mask >> k) & 1]
    out = np.stack([np.stack([djt_alg3(orient(c[b], rows[k])) for k in ks]) for b in range(c.shape[0])])
    return out[0] if single else out


# ------------------------------------------------- adjoints (F-1) ----

def unorient(h: np.ndarray, row) -> np.ndarray:
    """Transpose of `orient` (a voxel permutation, so its inverse): undo the flips
    of reading A, then the axis permutation."""
    g = np.asarray(h)
    for j, p in enumerate(row):
        if p < 0:
            g = np.flip(g, axis=j)
    perm = [abs(p) - 1 for p in row]
    inv = [perm.index(a) for a in range(3)]
    return np.ascontiguousarray(np.transpose(g, inv))


def drt_planes_adjoint(coef: np.ndarray, mask: int = 0xFFF, table: int = tables.TABLE_HEMISPHERE) -> np.ndarray:
    """Backprojection of the stacked DRT coefficients [B][K][N][N][3N] (or [K][N][N][3N]):
    sum over the dodecants k of unorient_k(adjoint of Alg. 1), fp64."""
    c = np.asarray(coef)
    single = c.ndim == 4
    if single:
        c = c[None]
    rows = tables.table(table, "drt")
    ks = [k for k in range(12) if (mask >> k) & 1]
    out = np.stack([sum(unorient(drt_adjoint(c[b][j]), rows[k]) for j, k in enumerate(ks)) for b in range(c.shape[0])])
    return out[0] if single else out


def djt_lines_adjoint(coef: np.ndarray, mask: int = 0x001, table: int = tables.TABLE_HEMISPHERE) -> np.ndarray:
    """Backprojection of stacked DJT coefficients [B][K][N][N][2N][2N] (or [K]...):
    sum over the dodecants of unorient_k(adjoint of Alg. 3), fp64."""
    c = np.asarray(coef)
    single = c.ndim == 5
    if single:
        c = c[None]
    rows = tables.table(table, "djt")
    ks = [k for k in range(12) if (mask >> k) & 1]
    out = np.stack([sum(unorient(djt_adjoint(c[b][j]), rows[k]) for j, k in enumerate(ks)) for b in range(c.shape[0])])
    return out[0] if single else out
