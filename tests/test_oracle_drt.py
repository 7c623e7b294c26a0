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


# ------------------------------------------------ mosaic seams (R13)
# Shared boundary planes of neighbouring dodecants of one normal set (HEMISPHERE table): the
# slope-0 edge of one is the same set of discrete planes as the slope-0 edge of the other
# (e.g. k=0 at s2=0 is z = l_s1(x) + d for every y; k=1 at s1=0 is z = l_s2(x) + d, reading A).
# The identities follow from the geometry, not from any mosaic code.
SHARED_EDGES = [
    (0, "s2=0", 1, "s1=0"), (0, "s1=0", 3, "s2=0"), (1, "s2=0", 2, "s1=0"), (2, "s2=0", 3, "s1=0"),
    (4, "s1=0", 5, "s2=0"), (4, "s2=0", 6, "s1=0"), (5, "s1=0", 7, "s2=0"), (6, "s2=0", 7, "s1=0"),
    (8, "s2=0", 9, "s1=0"), (8, "s1=0", 10, "s2=0"), (9, "s2=0", 11, "s1=0"), (10, "s1=0", 11, "s2=0"),
]


def _edge(out_k, e):
    return out_k[0] if e == "s1=0" else out_k[:, 0]


@pytest.mark.parametrize("N,seed", [(4, 41), (8, 42), (16, 43)])
def test_shared_boundary_identities(N, seed):
    st = oracle.drt_planes(_rand(N, seed), 0xFFF)
    for k, e, kk, ee in SHARED_EDGES:
        assert np.array_equal(_edge(st[k], e), _edge(st[kk], ee)), (k, e, kk, ee)
    # the slope-0 edges of dodecants of different sets are different planes
    assert not np.array_equal(_edge(st[0], "s1=0"), _edge(st[4], "s1=0"))


def _block(M, N, k):
    bi, bj = tables.DODECANT_COORDS[k]
    return M[bi * N:(bi + 1) * N, bj * N:(bj + 1) * N]


def _facing(M, N, k, kk):
    """Facing edge lines of the blocks of k and kk, which must be neighbours on the 4 x 4 block
    torus (the y- and x-sets meet across the hemisphere's wrap); None if they are not."""
    (bi, bj), (ci, cj) = tables.DODECANT_COORDS[k], tables.DODECANT_COORDS[kk]
    A, B = _block(M, N, k), _block(M, N, kk)
    if bj == cj and (ci - bi) % 4 == 1:
        return A[N - 1], B[0]
    if bj == cj and (bi - ci) % 4 == 1:
        return A[0], B[N - 1]
    if bi == ci and (cj - bj) % 4 == 1:
        return A[:, N - 1], B[:, 0]
    if bi == ci and (bj - cj) % 4 == 1:
        return A[:, 0], B[:, N - 1]
    return None


@pytest.mark.parametrize("N,seed", [(4, 44), (8, 45), (16, 46)])
def test_mosaic_seams_fit(N, seed):
    # fig:shapeOutput: "Each individual dodecant output is rotated so that all
    # of them fit accurately".  Every shared boundary of SHARED_EDGES lies on the facing edges of
    # the two blocks, column for column, and those edges hold exactly the shared planes.
    st = oracle.drt_planes(_rand(N, seed, 1, 255), 0xFFF)
    M = oracle.mosaic(st)
    for k, e, kk, ee in SHARED_EDGES:
        f = _facing(M, N, k, kk)
        assert f is not None, (k, kk)
        a, b = f
        assert np.array_equal(a, b), (k, kk)
        line = _edge(st[k], e)[:, 2:]
        assert sorted(map(tuple, a)) == sorted(map(tuple, line)), (k, kk)


@pytest.mark.parametrize("N", [4, 8])
def test_mosaic_null_normals(N):
    # fig:shapeOutput: "The black dots mark the position of x, y, and z null normals": the
    # (s1, s2) = (0, 0) columns of the z-set meet at the mosaic centre, those of the y-set at the
    # middles of the top and bottom edges, those of the x-set at the middles of the left and
    # right edges.
    st = oracle.drt_planes(_rand(N, 47, 1, 255), 0xFFF)
    M = oracle.mosaic(st)
    dots = {0: (2 * N - 1, 2 * N - 1), 1: (2 * N - 1, 2 * N), 2: (2 * N, 2 * N), 3: (2 * N, 2 * N - 1),
            4: (0, 2 * N), 5: (0, 2 * N - 1), 6: (4 * N - 1, 2 * N), 7: (4 * N - 1, 2 * N - 1),
            8: (2 * N, 0), 9: (2 * N - 1, 0), 10: (2 * N, 4 * N - 1), 11: (2 * N - 1, 4 * N - 1)}
    for k, (i, j) in dots.items():
        assert np.array_equal(M[i, j], st[k][0, 0, 2:]), k


def test_mosaic_orientation_is_forced():
    # With DodecantCoords verbatim, exactly one of the 8 square symmetries per dodecant closes all
    # four seams of its normal set (R13): the mosaic's within-block orientation is not a choice.
    N = 4
    st = oracle.drt_planes(_rand(N, 48, 1, 255), 0xFFF)
    syms = [(p, f0, f1) for p in (0, 1) for f0 in (0, 1) for f1 in (0, 1)]

    def orient_block(b, sym):
        p, f0, f1 = sym
        b = np.transpose(b, (1, 0, 2)) if p else b
        b = b[::-1] if f0 else b
        return b[:, ::-1] if f1 else b

    import itertools
    for S in ((0, 1, 2, 3), (4, 5, 6, 7), (8, 9, 10, 11)):
        pairs = [p for p in SHARED_EDGES if p[0] in S]
        good = []
        for choice in itertools.product(range(8), repeat=4):
            M = np.zeros((4 * N, 4 * N, 3 * N - 2), st.dtype)
            for k, c in zip(S, choice):
                bi, bj = tables.DODECANT_COORDS[k]
                M[bi * N:(bi + 1) * N, bj * N:(bj + 1) * N] = orient_block(st[k][:, :, 2:], syms[c])
            if all(np.array_equal(*_facing(M, N, k, kk)) for k, _, kk, _ in pairs):
                good.append(choice)
        assert len(good) == 1, (S, good)
        M = oracle.mosaic(st)
        for k, c in zip(S, good[0]):
            assert np.array_equal(_block(M, N, k), orient_block(st[k][:, :, 2:], syms[c])), k


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
