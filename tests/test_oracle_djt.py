"""Pins for the oracle's 3D DJT of lines (eq:3DfDJT, Alg. 3)."""
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
    out = oracle.djt_alg3(f)
    for row in load_golden("djt_n2_dodecant0.txt"):
        s1, s2, D1, vals = row[0], row[1], row[2], row[3:]
        assert list(out[s1, s2, D1]) == vals


@pytest.mark.parametrize("N,seed", [(2, 1), (4, 2), (8, 3), (16, 4)])
def test_alg3_equals_brute_force(N, seed):
    # Alg. 3 read literally == eq:3DfDJT.
    f = _rand(N, seed)
    assert np.array_equal(oracle.djt_alg3(f), oracle.djt_brute(f).astype(np.int64))


@pytest.mark.parametrize("N", [4, 16])
def test_mass(N):
    # lines at fixed slopes partition the cube
    f = _rand(N, 50 + N)
    out = oracle.djt_alg3(f)
    assert np.all(out.sum(axis=(2, 3)) == f.sum())


def test_spec_examples():
    N = 8
    # delta at (0,0,0) -> 1 at (s1, s2, N, N) for all slopes
    f = np.zeros((N, N, N), np.int64)
    f[0, 0, 0] = 1
    out = oracle.djt_alg3(f)
    exp = np.zeros_like(out)
    exp[:, :, N, N] = 1
    assert np.array_equal(out, exp)
    # all ones, s1 = s2 = 0 -> N at (0, 0, N+y, N+z)
    out = oracle.djt_alg3(np.ones((4, 4, 4), np.int64))
    assert np.all(out[0, 0, 4:, 4:] == 4) and out[0, 0].sum() == 64
    # the diagonal ray u -> (u,u,u): N at (N-1, N-1, N, N), unique max
    for N in (4, 8):
        f = np.zeros((N, N, N), np.int64)
        for u in range(N):
            f[u, u, u] = 1
        out = oracle.djt_alg3(f)
        assert out[N - 1, N - 1, N, N] == N
        assert (out == N).sum() == 1


def test_axis_lines_closed_form():
    # s1 = s2 = 0: lines parallel to x: out[0][0][N+y][N+z] = sum_x f(x,y,z);
    # s1 = s2 = N-1: exact diagonals (l(u) = u).
    N = 16
    f = _rand(N, 60)
    out = oracle.djt_alg3(f)
    assert np.array_equal(out[0, 0, N:, N:], f.sum(axis=0))
    u = np.arange(N)
    for D1 in range(2 * N):
        for D2 in range(0, 2 * N, 3):
            y, z = u + D1 - N, u + D2 - N
            ok = (y >= 0) & (y < N) & (z >= 0) & (z < N)
            assert out[N - 1, N - 1, D1, D2] == f[u[ok], y[ok], z[ok]].sum()


def test_point_and_linearity():
    f, g = _rand(16, 61), _rand(16, 62)
    out = oracle.djt_alg3(f)
    rng = np.random.default_rng(1)
    for _ in range(50):
        s1, s2, D1, D2 = (int(t) for t in rng.integers(0, [16, 16, 32, 32]))
        assert oracle.djt_point(f, s1, s2, D1, D2) == out[s1, s2, D1, D2]
    assert np.array_equal(oracle.djt_alg3(2 * f - g), 2 * out - oracle.djt_alg3(g))


@pytest.mark.parametrize("N", [4, 8])
def test_adjoint_identity(N):
    # eq:invmap3DJsummation is the exact transpose of Alg. 3.
    f = _rand(N, 70 + N, -50, 50)
    rng = np.random.default_rng(N)
    g = rng.integers(-50, 50, size=(N, N, 2 * N, 2 * N)).astype(np.int64)
    lhs = int((oracle.djt_alg3(f) * g).sum())
    rhs = int(round((f * oracle.djt_adjoint(g.astype(np.float64))).sum()))
    assert lhs == rhs


def test_djt_table_complete():
    # the DJT table gives 12 distinct line families (N = 4).
    N = 4
    fams = []
    for k in range(12):
        lines = {}
        for x in range(N):
            for y in range(N):
                for z in range(N):
                    f = np.zeros((N, N, N), np.int64)
                    f[x, y, z] = 1
                    out = oracle.djt_alg3(oracle.orient(f, tables.DJT_HEMISPHERE[k]))
                    for idx in zip(*np.nonzero(out)):
                        lines.setdefault(idx, set()).add((x, y, z))
        fams.append(frozenset(frozenset(v) for v in lines.values()))
    assert len(set(fams)) == 12


def test_survey_checksums():
    # SURVEY.md §8(c) checksums (independent scratch brute force).
    exp = {(4, 1): (91520, 47874112, 26454578), (8, 1): (3829760, 31514388480, 2693652920),
           (16, 1): (131530752, 17258756440064, 190836777728),
           (4, 0xFFF): (1098240, 6760109568, 358152088), (8, 0xFFF): (45957120, 4519516487680, 34730771616)}
    for (N, mask), want in exp.items():
        x, y, z = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
        f = (37 * x + 11 * y + 3 * z + 5 * x * y * z) % 256
        v = oracle.djt_lines(f, mask).reshape(-1).astype(np.int64)
        i = np.arange(1, v.size + 1, dtype=np.int64)
        assert (int(v.sum()), int((v * i).sum()), int((v * v).sum())) == want
