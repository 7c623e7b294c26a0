"""Pins of the application oracle (oracle/apps.py).

Threshold decisions are checked against exact rational arithmetic (fractions.Fraction); the
plane normals against the geometry of digital planes built point by point from eq:digitalLine
and the orientation table; the relative-maximum test against scipy's maximum filter; the two
applications by what the paper claims they do (walls detected as mutually orthogonal maxima;
a ray buried in stronger noise recovered by threshold + backprojection)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import apps, tables


def test_threshold_exact_rational():
    rng = np.random.default_rng(1)
    c = rng.integers(-50, 1000, 500)
    for num, den in ((0, 1), (1, 3), (2, 3), (7, 10), (1, 1)):
        t = apps.threshold(c, num, den)
        mx = int(c.max())
        for v, w in zip(c, t):
            keep = Fraction(int(v)) >= Fraction(num, den) * mx
            assert w == (v if keep else 0)
    assert np.count_nonzero(apps.threshold(c, 1, 1)) == np.count_nonzero(c == c.max())


def _oriented_plane_voxels(N, k, s1, s2, delta, table=tables.TABLE_HEMISPHERE):
    """Original-cube voxels of the dodecant-k digital plane z' = l_s1(x') + l_s2(y') + delta."""
    g = np.zeros((N, N, N), np.int64)
    for x in range(N):
        for y in range(N):
            z = oracle.line(N.bit_length() - 1, s1, x) + oracle.line(N.bit_length() - 1, s2, y) + delta
            if 0 <= z < N:
                g[x, y, z] = 1
    return oracle.unorient(g, tables.table(table, "drt")[k])


@pytest.mark.parametrize("k,s1,s2", [(0, 5, 9), (3, 13, 2), (6, 7, 7), (10, 0, 11), (11, 15, 15)])
def test_plane_normal_is_normal(k, s1, s2):
    """n . p is constant up to the digitisation (|spread| <= 4 (N-1)) over every voxel p of the
    plane in the ORIGINAL axes; swapping two normal components breaks it."""
    N = 16
    f = _oriented_plane_voxels(N, k, s1, s2, 0)
    pts = np.argwhere(f)
    n = np.array(apps.plane_normal(k, s1, s2, N))
    proj = pts @ n
    assert proj.max() - proj.min() <= 4 * (N - 1)
    if s1 != s2:
        nb = n.copy()
        a = [abs(p) - 1 for p in tables.table(tables.TABLE_HEMISPHERE, "drt")[k]]
        nb[a[0]], nb[a[1]] = n[a[1]], n[a[0]]
        pb = pts @ nb
        assert pb.max() - pb.min() > 4 * (N - 1)


def test_relative_max_matches_maximum_filter():
    ndimage = pytest.importorskip("scipy.ndimage")
    rng = np.random.default_rng(2)
    c = rng.permutation(2 * 6 * 6 * 18).reshape(2, 6, 6, 18)          # distinct values: no ties
    for j in range(2):
        mf = ndimage.maximum_filter(c[j], size=3, mode="constant", cval=-1)
        for s1 in range(6):
            for s2 in range(6):
                for D in range(18):
                    assert apps.is_relative_max(c, j, s1, s2, D) == (c[j, s1, s2, D] == mf[s1, s2, D])


def test_relative_max_plateau_one_representative():
    c = np.zeros((1, 3, 3, 5), np.int64)
    c[0, 1, 1, 1:4] = 7                                               # a plateau of three
    got = [D for D in range(5) if apps.is_relative_max(c, 0, 1, 1, D)]
    assert got == [1]


def _room(N, seed=0):
    f = np.zeros((N, N, N), np.int64)
    f[3, :, :] = 1                     # wall x = 3
    f[:, N - 4, :] = 1                 # wall y = N - 4
    f[:, :, 2] = 1                     # floor z = 2
    f[N // 3:N // 2, N // 3:N // 2, N // 3:N // 2] = 1                # a box
    rng = np.random.default_rng(seed)
    return f + (rng.random((N, N, N)) < 0.02)


def test_detect_room_walls():
    """the strongest plane and the relative maxima orthogonal to it are the walls."""
    N = 32
    c = oracle.drt_planes(_room(N))
    flags, am = apps.detect_planes(c, 0xFFF, 1, 3, 1, 10)
    j0, a1, a2, _ = np.unravel_index(am, c.shape)
    m = np.array(apps.plane_normal(int(j0), int(a1), int(a2), N))
    assert np.count_nonzero(m) == 1                                    # an axis plane wins
    axes = set()
    for j, s1, s2, D in np.argwhere(flags):
        n = np.array(apps.plane_normal(int(j), int(s1), int(s2), N))
        if (j, s1, s2, D) != (j0, a1, a2, _):
            assert (n @ m) ** 2 * 100 <= (n @ n) * (m @ m)              # orthogonal (R22)
            assert c[j, s1, s2, D] * 3 >= c.reshape(-1)[am]             # above threshold (R19)
            assert apps.is_relative_max(c, int(j), int(s1), int(s2), int(D))
        if np.count_nonzero(n) == 1:
            axes.add(int(np.argmax(np.abs(n))))
    assert axes == {0, 1, 2}                                           # all three walls found


def test_denoise_recovers_buried_ray():
    """a ray in noise of larger amplitude stands out in the John domain; keeping the
    top coefficients and backprojecting brings the ray back."""
    N, n = 32, 5
    s1, s2, d1, d2 = 7, 12, N + 5, N + 3
    rng = np.random.default_rng(3)
    f = rng.integers(0, 201, (N, N, N)).astype(np.int64)            # noise amplitude 200
    ray = np.zeros_like(f)
    for u in range(N):
        ray[u, oracle.line(n, s1, u) + d1 - N, oracle.line(n, s2, u) + d2 - N] = 1
    f += 100 * ray                                                     # ray amplitude 100
    kept, back = apps.denoise_rays(f, 0x001, 9, 10)
    assert apps.argmax(kept) == np.ravel_multi_index((0, s1, s2, d1, d2), kept.shape)
    top = np.argsort(back.reshape(-1))[::-1][:N]
    assert set(top.tolist()) == set(np.flatnonzero(ray).tolist())
