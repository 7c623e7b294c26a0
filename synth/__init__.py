"""Seeded synthetic inputs shared by the tests, bench.py and the oracle checks.

This module holds NONE of the method's arithmetic (no discrete lines, no
dodecant tables, no transform).  It only draws random voxels with a
counter-based SplitMix64 generator (Steele, Lea & Flood, OOPSLA 2014) and
rasterises simple geometric clutter (planar sheets, line segments) with plain
rational (floor-division) digital geometry, which is deliberately *not* the
paper's dyadic line of eq:digitalLine.

Recipes mirror BASELINE.json `configs`:
  cfg1  N=16  int32 uniform [0,255]                         (one cube)
  cfg2  N=64  uint8 uniform [0,255] + 50 planar sheets = 255 (walls)
  cfg3  N=256 uint8, each voxel != 0 w.p. 0.3, value U{1..255}
  cfg4  N=64  uint8 uniform [0,255] + 200 line segments = 255 (rays)
  cfg5  256 cubes N=32 float32 ~ N(0,1) (Box-Muller, cosine branch)
The paper's own volumes (MRI, depth maps, phantoms)
are not available, so these seeded synthetic cubes stand in for them.
All cubes are C-ordered [batch][x][y][z] (z contiguous).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

SEEDS = {1: 0xD47C0001, 2: 0xD47C0002, 3: 0xD47C0003, 4: 0xD47C0004, 5: 0xD47C0005}


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """Counter-based SplitMix64: draw i is mix(seed + (i+1)*golden)."""

    def __init__(self, seed: int):
        self.seed = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.counter = 0

    def draw(self, count: int) -> np.ndarray:
        idx = np.arange(self.counter + 1, self.counter + 1 + count, dtype=np.uint64)
        self.counter += count
        with np.errstate(over="ignore"):
            return _mix(self.seed + idx * _GOLDEN)

    def uint(self, count: int, lo: int, hi: int) -> np.ndarray:
        """Uniform integers in [lo, hi] as a + (r mod (b-a+1)) (int64)."""
        span = np.uint64(hi - lo + 1)
        return (self.draw(count) % span).astype(np.int64) + lo

    def unit(self, count: int) -> np.ndarray:
        """Uniform doubles in [0, 1): (r >> 11) * 2^-53."""
        return (self.draw(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def normal(self, count: int) -> np.ndarray:
        """N(0,1) doubles, Box-Muller cosine branch, two draws per value."""
        r = self.draw(2 * count)
        u1 = ((r[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        u2 = (r[1::2] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def _floordiv(a, b):
    return np.floor_divide(a, b)


# ---------------------------------------------------------------- basic cubes

def uniform_cube(N: int, seed: int, dtype=np.uint8, lo: int = 0, hi: int = 255,
                 batch: int | None = None) -> np.ndarray:
    g = SplitMix64(seed)
    b = 1 if batch is None else batch
    v = g.uint(b * N * N * N, lo, hi).astype(dtype).reshape(b, N, N, N)
    return v[0] if batch is None else v


def sparse_cube(N: int, seed: int, p: float = 0.3, batch: int | None = None) -> np.ndarray:
    """uint8: each voxel non-zero with probability p, value U{1..255}."""
    g = SplitMix64(seed)
    b = 1 if batch is None else batch
    cnt = b * N * N * N
    keep = g.unit(cnt) < p
    val = g.uint(cnt, 1, 255)
    v = np.where(keep, val, 0).astype(np.uint8).reshape(b, N, N, N)
    return v[0] if batch is None else v


def normal_cube(N: int, seed: int, batch: int | None = None) -> np.ndarray:
    g = SplitMix64(seed)
    b = 1 if batch is None else batch
    v = g.normal(b * N * N * N).astype(np.float32).reshape(b, N, N, N)
    return v[0] if batch is None else v


# ------------------------------------------------------- geometric clutter

def _axes(a: int):
    return [(a + 1) % 3, (a + 2) % 3]


def add_sheets(cube: np.ndarray, count: int, seed: int, value: int = 255) -> list:
    """Draw `count` digital planar sheets into `cube` (in place).

    Sheet: driven axis a, the other two axes (b, c), integer slopes
    p, q in [-(N-1), N-1] and an anchor voxel C; the sheet is every voxel with
    u_a = C_a + floor((p (u_b - C_b) + q (u_c - C_c)) / (N-1)) inside the cube.
    Returns the list of (a, p, q, C) tuples.
    """
    N = cube.shape[0]
    g = SplitMix64(seed ^ 0x5EE75)
    out = []
    ub, uc = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    for _ in range(count):
        a = int(g.uint(1, 0, 2)[0])
        p, q = (int(t) for t in g.uint(2, -(N - 1), N - 1))
        C = [int(t) for t in g.uint(3, 0, N - 1)]
        b, c = _axes(a)
        ua = C[a] + _floordiv(p * (ub - C[b]) + q * (uc - C[c]), max(N - 1, 1))
        ok = (ua >= 0) & (ua < N)
        idx = [None, None, None]
        idx[a], idx[b], idx[c] = ua[ok], ub[ok], uc[ok]
        cube[idx[0], idx[1], idx[2]] = value
        out.append((a, p, q, tuple(C)))
    return out


def add_segments(cube: np.ndarray, count: int, seed: int, value: int = 255) -> list:
    """Draw `count` digital line segments into `cube` (in place).

    Segment: driving axis a, slopes p, q in [-(N-1), N-1], anchor voxel C and
    a driving range [u0, u1]; voxel at u is (u, C_b + floor(p (u - C_a)/(N-1)),
    C_c + floor(q (u - C_a)/(N-1))) in (a, b, c) order, kept if inside.
    """
    N = cube.shape[0]
    g = SplitMix64(seed ^ 0x5E6E)
    out = []
    for _ in range(count):
        a = int(g.uint(1, 0, 2)[0])
        p, q = (int(t) for t in g.uint(2, -(N - 1), N - 1))
        C = [int(t) for t in g.uint(3, 0, N - 1)]
        u0, u1 = sorted(int(t) for t in g.uint(2, 0, N - 1))
        b, c = _axes(a)
        u = np.arange(u0, u1 + 1)
        vb = C[b] + _floordiv(p * (u - C[a]), max(N - 1, 1))
        vc = C[c] + _floordiv(q * (u - C[a]), max(N - 1, 1))
        ok = (vb >= 0) & (vb < N) & (vc >= 0) & (vc < N)
        idx = [None, None, None]
        idx[a], idx[b], idx[c] = u[ok], vb[ok], vc[ok]
        cube[idx[0], idx[1], idx[2]] = value
        out.append((a, p, q, tuple(C), u0, u1))
    return out


# ------------------------------------------------------------ the 5 configs

CONFIGS = {
    1: dict(name="cfg1_drt_n16_i32_dodecant0", transform="drt", N=16, batch=1,
            mask=0x001, in_dtype="i32", out_dtype="i32"),
    2: dict(name="cfg2_drt_n64_u8_sheets_12dod", transform="drt", N=64, batch=1,
            mask=0xFFF, in_dtype="u8", out_dtype="i32"),
    3: dict(name="cfg3_drt_n256_u8_sparse30_12dod", transform="drt", N=256, batch=1,
            mask=0xFFF, in_dtype="u8", out_dtype="i32"),
    4: dict(name="cfg4_djt_n64_u8_segments_dodecant0", transform="djt", N=64, batch=1,
            mask=0x001, in_dtype="u8", out_dtype="i32"),
    5: dict(name="cfg5_drt_batch256_n32_f32_12dod", transform="drt", N=32, batch=256,
            mask=0xFFF, in_dtype="f32", out_dtype="f32"),
}


def config_input(cfg: int) -> np.ndarray:
    """The seeded input of BASELINE.json config `cfg`, shape [batch][N][N][N]."""
    s = SEEDS[cfg]
    if cfg == 1:
        return uniform_cube(16, s, np.int32, 0, 255, batch=1)
    if cfg == 2:
        c = uniform_cube(64, s, np.uint8)
        add_sheets(c, 50, s)
        return c[None]
    if cfg == 3:
        return sparse_cube(256, s, 0.3, batch=1)
    if cfg == 4:
        c = uniform_cube(64, s, np.uint8)
        add_segments(c, 200, s)
        return c[None]
    if cfg == 5:
        return normal_cube(32, s, batch=256)
    raise ValueError(cfg)
