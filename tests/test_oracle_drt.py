"""Pins for the oracle's 3D DRT of planes (eq:3DfDRT, Alg. 1, Alg. 2).

Each test pins the oracle to something other than itself: hand-derived
goldens, the brute-force definition vs the recursion (two independent
routes), the separable Wu-Brady route, closed forms, invariants (mass,
support), special cases and the exact adjoint identity.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import tables
from conftest import load_golden


def _rand(N, seed, lo=0, hi=255):
    return synth.uniform_cube(N, seed, np.int64, lo, hi)


def test_golden_n2():
    x, y, z = np.meshgrid(np.arange(2), np.arange(2), np.arange(2), indexing="ij")
    f = 1 + 4 * x + 2 * y + z
    out = oracle.drt_alg1(f)
    for row in load_golden("drt_n2_dodecant0.txt"):
        s1, s2, vals = row[0], row[1], row[2:]
        assert list(out[s1, s2]) == vals


@pytest.mark.parametrize("N,seed", [(2, 1), (4, 2), (4, 3), (8, 4), (16, 5)])
def test_alg1_equals_brute_force(N, seed):
    # Alg. 1 read literally == eq:3DfDRT cell for cell.
    f = _rand(N, seed)
    assert np.array_equal(oracle.drt_alg1(f), oracle.drt_brute(f).astype(np.int64))


@pytest.mark.parametrize("N,seed", [(16, 6), (32, 7)])
def test_alg1_equals_separable(N, seed):
    # the Wu-Brady separable route.
    f = _rand(N, seed)
    assert np.array_equal(oracle.drt_alg1(f), oracle.drt_separable(f).astype(np.int64))


def test_alg1_float_equals_int():
    f = _rand(8, 8)
    assert np.array_equal(oracle.drt_alg1(f.astype(np.float64)), oracle.drt_alg1(f).astype(np.float64))


@pytest.mark.parametrize("N", [4, 16, 64])
def test_mass_and_support(N):
    # Planes at fixed slopes partition the cube, and the
    # non-zero displacements are exactly D in [2N - s1 - s2, 3N-1]
    # ("N + s1 + s2" displacements).
    f = _rand(N, 10 + N, 1, 255)          # strictly positive voxels
    out = oracle.drt_alg1(f)
    assert np.all(out.sum(axis=2) == f.sum())
    s1 = np.arange(N)[:, None, None]
    s2 = np.arange(N)[None, :, None]
    D = np.arange(3 * N)[None, None, :]
    inside = D >= 2 * N - s1 - s2
    assert np.all(out[~np.broadcast_to(inside, out.shape)] == 0)
    assert np.all(out[np.broadcast_to(inside, out.shape)] > 0)


def test_spec_examples():
    # delta at (0,0,0) -> 1 at (s1, s2, 2N) for all slopes.
    N = 8
    f = np.zeros((N, N, N), np.int64)
    f[0, 0, 0] = 1
    out = oracle.drt_alg1(f)
    exp = np.zeros_like(out)
    exp[:, :, 2 * N] = 1
    assert np.array_equal(out, exp)
    # all-ones N=4, s1=s2=0 -> 16 at D = 8..11.
    out = oracle.drt_alg1(np.ones((4, 4, 4), np.int64))
    assert list(out[0, 0]) == [0] * 8 + [16] * 4


def test_z_slices_and_diagonal_closed_forms():
    # s1 = s2 = 0: horizontal planes z = D - 2N, i.e. z-slice sums.
    # s1 = s2 = N-1: l(u) = u exactly, plane z = x + y + D - 2N.
    N = 16
    f = _rand(N, 11)
    out = oracle.drt_alg1(f)
    assert np.array_equal(out[0, 0, 2 * N:], f.sum(axis=(0, 1)))
    x, y = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    for D in range(3 * N):
        z = x + y + D - 2 * N
        ok = (z >= 0) & (z < N)
        assert out[N - 1, N - 1, D] == f[x[ok], y[ok], z[ok]].sum()


def test_y_invariant_reduces_to_2d_drt():
    # f(x,y,z) = h(x,z) for every y -> out[s1][0][D] = N * DRT2D(h)(s1, D - 2N),
    # with the 2D DRT of eq:GotzfDRT written out directly.
    N, n = 16, 4
    h = synth.uniform_cube(N, 12, np.int64)[:, 0, :]
    f = np.repeat(h[:, None, :], N, axis=1)
    out = oracle.drt_alg1(f)
    for s in range(N):
        L = [oracle.line(n, s, u) for u in range(N)]
        for D in range(3 * N):
            d = D - 2 * N
            exp = sum(h[u, L[u] + d] for u in range(N) if 0 <= L[u] + d < N)
            assert out[s, 0, D] == N * exp


def test_linearity():
    f, g = _rand(8, 13), _rand(8, 14)
    assert np.array_equal(oracle.drt_alg1(3 * f - 2 * g), 3 * oracle.drt_alg1(f) - 2 * oracle.drt_alg1(g))


def test_point_equals_alg1():
    f = _rand(32, 15)
    out = oracle.drt_alg1(f)
    rng = np.random.default_rng(0)
    for _ in range(50):
        s1, s2, D = rng.integers(0, 32), rng.integers(0, 32), rng.integers(0, 96)
        assert oracle.drt_point(f, s1, s2, D) == out[s1, s2, D]


# ------------------------------------------------------------ 12 dodecants

def test_orient_semantics():
    # row (-2,1,3) maps a delta at (0,0,0) to (3,0,0) at N = 4.
    f = np.zeros((4, 4, 4), np.int64)
    f[0, 0, 0] = 1
    g = oracle.orient(f, (-2, 1, 3))
    assert g[3, 0, 0] == 1 and g.sum() == 1
    # a voxel at (1,2,3): new axis 0 = old axis 2 reversed -> 3-2 = 1, new axis 1 = old x = 1
    f[:] = 0
    f[1, 2, 3] = 1
    assert oracle.orient(f, (-2, 1, 3))[1, 1, 3] == 1


def _det(row):
    M = np.zeros((3, 3), int)
    for j, p in enumerate(row):
        M[j, abs(p) - 1] = 1 if p > 0 else -1
    return round(np.linalg.det(M))


def test_tables_right_handed():
    # right-hand rule (p1-p0) x (p2-p0) = d: every row is a
    # proper rotation (det = +1) of the basic dodecant.
    for T in (tables.DRT_PRINTED, tables.DRT_HEMISPHERE, tables.DJT_HEMISPHERE, tables.SHARED):
        assert len(T) == 12 and all(_det(r) == 1 for r in T)
        assert all(sorted(abs(p) for p in r) == [1, 2, 3] for r in T)


def test_centre_delta_every_dodecant():
    # a delta at the centre lies on exactly one plane per slope
    # pair in every dodecant -> N^2 ones per dodecant.
    N = 8
    f = np.zeros((N, N, N), np.int64)
    f[N // 2, N // 2, N // 2] = 1
    out = oracle.drt_planes(f, 0xFFF)
    assert out.shape == (12, N, N, 3 * N)
    assert np.all(out.sum(axis=3) == 1)
    assert np.all(out.max(axis=3) == 1)


def _plane_sets(N, T):
    """Voxel sets of every discrete plane of each dodecant (by pushing unit
    deltas through the oracle)."""
    fam = []
    for k in range(12):
        sets = {}
        for x in range(N):
            for y in range(N):
                for z in range(N):
                    f = np.zeros((N, N, N), np.int64)
                    f[x, y, z] = 1
                    out = oracle.drt_alg1(oracle.orient(f, T[k]))
                    for idx in zip(*np.nonzero(out)):
                        sets.setdefault(idx, set()).add((x, y, z))
        fam.append({frozenset(v) for v in sets.values()})
    return fam


@pytest.mark.slow
def test_hemisphere_table_complete_printed_duplicates():
    # the printed InOrder gives dodecant 5 == 7 and 9 == 11 as plane
    # families; the repaired (HEMISPHERE) table gives 12 distinct families.
    N = 4
    fam = _plane_sets(N, tables.DRT_PRINTED)
    assert fam[5] == fam[7] and fam[9] == fam[11]
    famh = _plane_sets(N, tables.DRT_HEMISPHERE)
    assert len({frozenset(F) for F in famh}) == 12
    assert len(set().union(*famh)) > len(set().union(*fam))


def test_printed_duplicate_relation():
    # SURVEY F4 exact relation: out5[s1][s2][D] = out7[s2][s1][5N-1-s1-s2-D].
    N = 8
    f = _rand(N, 16)
    out = oracle.drt_planes(f, 0xFFF, tables.TABLE_PRINTED)
    for s1 in range(N):
        for s2 in range(N):
            for D in range(3 * N):
                D2 = 5 * N - 1 - s1 - s2 - D
                v = out[7, s2, s1, D2] if 0 <= D2 < 3 * N else 0
                assert out[5, s1, s2, D] == v
                v = out[11, s2, s1, D2] if 0 <= D2 < 3 * N else 0
                assert out[9, s1, s2, D] == v


def test_hemisphere_outputs_distinct():
    N = 8
    out = oracle.drt_planes(_rand(N, 17), 0xFFF)
    for a in range(12):
        for b in range(a + 1, 12):
            assert not np.array_equal(out[a], out[b])


@pytest.mark.parametrize("N,S0,S1,S2,table", [
    (4, 1098240, 1268203776, 1299219764, 0),
    (4, 1098240, 1268437632, 1304432436, 1),
    (8, 45957120, 423765843968, 268380499636, 0),
    (8, 45957120, 423769395200, 269831660916, 1),
    (16, 1578369024, 116384106938368, 38082645501420, 0),
    (16, 1578369024, 116384167493632, 38159905160620, 1),
])
def test_survey_checksums(N, S0, S1, S2, table):
    # Cross-check against the survey's independent scratch brute force
    # (SURVEY.md §8(c) "Checksums"): f = (37x + 11y + 3z + 5xyz) mod 256.
    x, y, z = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    f = (37 * x + 11 * y + 3 * z + 5 * x * y * z) % 256
    v = oracle.drt_planes(f, 0xFFF, table).reshape(-1).astype(np.int64)
    i = np.arange(1, v.size + 1, dtype=np.int64)
    assert (int(v.sum()), int((v * i).sum()), int((v * v).sum())) == (S0, S1, S2)


def test_mosaic_placement():
    # Alg. 2: 4N x 4N x (3N-2), 12 populated blocks, 4 empty.
    N = 4
    st = oracle.drt_planes(_rand(N, 18, 1, 255), 0xFFF)
    M = oracle.mosaic(st)
    assert M.shape == (4 * N, 4 * N, 3 * N - 2)
    filled = {(i, j) for i in range(4) for j in range(4) if M[i * N:(i + 1) * N, j * N:(j + 1) * N].any()}
    assert filled == set(tables.DODECANT_COORDS)
    for k, (i, j) in enumerate(tables.DODECANT_COORDS):
        blk = M[i * N:(i + 1) * N, j * N:(j + 1) * N]
        assert sorted(blk.reshape(-1)) == sorted(st[k][:, :, 2:].reshape(-1))


# ----------------------------------------------------------------- adjoint

@pytest.mark.parametrize("N", [4, 8, 16])
def test_adjoint_identity(N):
    # eq:invmap3Dsummation is the exact transpose
    # of Alg. 1: <A f, g> == <f, A^T g> in exact integer arithmetic.
    f = _rand(N, 20 + N, -50, 50)
    g = synth.uniform_cube(N, 30 + N, np.int64, -50, 50)
    g = np.concatenate([g, g, g], axis=2)[:, :, :3 * N]
    lhs = int((oracle.drt_alg1(f) * g).sum())
    rhs = int(round((f * oracle.drt_adjoint(g.astype(np.float64))).sum()))
    assert lhs == rhs


def test_round_trip_cg():
    # "exact round trip through the fast inverse on tiny N" (BASELINE north_star):
    # CG on the normal equations A^T A x = A^T b with the paper's adjoint
    # (PAPER.md:573-575 uses the adjoint as the approximate inverse) recovers
    # the integer input exactly after rounding.
    N = 4
    f = _rand(N, 40, 0, 9).astype(np.float64)
    b = oracle.drt_alg1(f)
    A = lambda v: oracle.drt_alg1(v.reshape(N, N, N))
    At = lambda r: oracle.drt_adjoint(r)
    x = np.zeros_like(f)
    r = At(b) - At(A(x))
    p = r.copy()
    rs = (r * r).sum()
    for _ in range(400):
        Ap = At(A(p))
        a = rs / (p * Ap).sum()
        x += a * p
        r -= a * Ap
        rsn = (r * r).sum()
        if rsn < 1e-20:
            break
        p = r + (rsn / rs) * p
        rs = rsn
    assert np.array_equal(np.rint(x), f)
