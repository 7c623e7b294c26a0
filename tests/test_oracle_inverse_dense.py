"""Dense-matrix pins of the inverse oracle (oracle/inverse.py, readings R15-R18 of DESIGN.md).

The DRT is linear, so at N = 2 and 4 it can be written out as an explicit 0/1 matrix A built
voxel by voxel from the definition eq:3DfDRT: voxel v lies on plane
(k, s1, s2, D) of dodecant k iff its oriented coordinates satisfy z' = l_s1(x') + l_s2(y') + D - 2N,
with the recursive digital line of eq:digitalLine and reading A of the
orientation rows.  Nothing here calls the oracle's transforms: A^T is the
matrix transpose, h is scipy's correlate, P and S are explicit matrices.  The oracle's iterative
improvement (press_refine) and multigrid approximate inverse (mg_apply, press_multigrid) must
equal the same iteration computed with these matrices.
"""
import numpy as np
import pytest
from scipy import ndimage

import oracle
from oracle import inverse, tables


def _line(n, s, u):
    """eq:digitalLine, recursive: l^k_s(u) = l^{k-1}_{floor(s/2)}(u mod 2^{k-1}) + u_{k-1} ceil(s/2)."""
    if n == 0:
        return 0
    return _line(n - 1, s >> 1, u & ((1 << (n - 1)) - 1)) + ((u >> (n - 1)) & 1) * ((s + 1) >> 1)


def _dense_drt(N, mask=0xFFF, table=tables.TABLE_HEMISPHERE):
    """A[(j, s1, s2, D), voxel] over the dodecants j of `mask` (stacked layout, C order)."""
    n = N.bit_length() - 1
    rows = tables.table(table, "drt")
    ks = [k for k in range(12) if (mask >> k) & 1]
    A = np.zeros((len(ks) * N * N * 3 * N, N ** 3))
    for j, k in enumerate(ks):
        p = rows[k]
        for x in range(N):
            for y in range(N):
                for z in range(N):
                    v = (x, y, z)
                    o = [v[abs(a) - 1] if a > 0 else N - 1 - v[abs(a) - 1] for a in p]   # reading A
                    for s1 in range(N):
                        for s2 in range(N):
                            D = o[2] - _line(n, s1, o[0]) - _line(n, s2, o[1]) + 2 * N
                            A[((j * N + s1) * N + s2) * 3 * N + D, (x * N + y) * N + z] += 1.0
    return A


def _h(g):
    """The high-pass filter of PAPER.md:576-591 with zero padding (R17), by scipy."""
    return ndimage.correlate(g, inverse.highpass_kernel(), mode="constant", cval=0.0)


def _step(A, r, N):
    """R15-R16 with explicit matrices: p = h * (A^T r), alpha = <r, Ap> / <Ap, Ap>."""
    p = _h((A.T @ r).reshape(N, N, N)).reshape(-1)
    q = A @ p
    alpha = float(r @ q) / float(q @ q)
    return alpha * p, alpha * q


@pytest.fixture(scope="module")
def mats():
    return {N: _dense_drt(N) for N in (2, 4)}


def test_dense_matrix_is_the_oracle_transform(mats):
    rng = np.random.default_rng(3)
    for N, A in mats.items():
        f = rng.standard_normal((N, N, N))
        assert np.allclose(A @ f.reshape(-1), oracle.drt_planes(f).reshape(-1), atol=1e-12)
        c = rng.standard_normal(A.shape[0])
        assert np.allclose(A.T @ c, oracle.drt_planes_adjoint(c.reshape(12, N, N, 3 * N)).reshape(-1), atol=1e-10)


def test_press_refine_equals_dense_iteration(mats):
    # R15-R16: x_{k+1} = x_k + alpha_k h*(A^T r_k), r_{k+1} = r_k - alpha_k A h*(A^T r_k)
    N, A = 4, mats[4]
    f = np.random.default_rng(4).integers(0, 9, (N, N, N)).astype(np.float64)
    b = A @ f.reshape(-1)
    x, r = np.zeros(N ** 3), b.copy()
    norms = [np.linalg.norm(r)]
    for _ in range(3):
        dx, dq = _step(A, r, N)
        x, r = x + dx, r - dq
        norms.append(np.linalg.norm(r))
    xo, ro = inverse.press_refine(b.reshape(12, N, N, 3 * N), 3)
    assert np.allclose(xo.reshape(-1), x, atol=1e-10)
    assert np.allclose(ro, norms, rtol=1e-12, atol=1e-12)


def _dense_restrict(N):
    """S as a matrix on stacked coefficients: 1/8 [c(2 s1, 2 s2, 2 d) + c(., ., 2 d + 1)]."""
    M, W, Wh = N // 2, 3 * N, 3 * N // 2
    S = np.zeros((12 * M * M * Wh, 12 * N * N * W))
    for j in range(12):
        for s1 in range(M):
            for s2 in range(M):
                for d in range(Wh):
                    row = ((j * M + s1) * M + s2) * Wh + d
                    for dd in (2 * d, 2 * d + 1):
                        S[row, ((j * N + 2 * s1) * N + 2 * s2) * W + dd] = 0.125
    return S


def _dense_prolong(M):
    """P as a matrix: every coarse voxel fills its 2 x 2 x 2 fine block."""
    N = 2 * M
    P = np.zeros((N ** 3, M ** 3))
    for x in range(N):
        for y in range(N):
            for z in range(N):
                P[(x * N + y) * N + z, ((x // 2) * M + y // 2) * M + z // 2] = 1.0
    return P


def test_multigrid_equals_dense_recursion(mats):
    # R18: B_N r = e + alpha' h*(A^T (r - A e)) with e = P B_{N/2}(S r); B_{n_min} = the R16 step
    A4, A2 = mats[4], mats[2]
    S, P = _dense_restrict(4), _dense_prolong(2)
    f = np.random.default_rng(5).standard_normal((4, 4, 4))
    r = A4 @ f.reshape(-1)
    ec, _ = _step(A2, S @ r, 2)
    e = P @ ec
    ae = A4 @ e
    dp, dq = _step(A4, r - ae, 4)
    e_dense, ae_dense = e + dp, ae + dq
    e_o, ae_o = inverse.mg_apply(r.reshape(12, 4, 4, 12), n_min=2)
    assert np.allclose(e_o.reshape(-1), e_dense, atol=1e-10)
    assert np.allclose(ae_o.reshape(-1), ae_dense, atol=1e-10)
    # and the restriction / prolongation operators themselves
    assert np.allclose(inverse.restrict(r.reshape(12, 4, 4, 12)).reshape(-1), S @ r)
    assert np.allclose(inverse.prolong(ec.reshape(2, 2, 2)).reshape(-1), P @ ec)


def test_press_multigrid_two_iterations_dense(mats):
    A4, A2 = mats[4], mats[2]
    S, P = _dense_restrict(4), _dense_prolong(2)
    f = np.random.default_rng(6).integers(0, 5, (4, 4, 4)).astype(np.float64)
    b = A4 @ f.reshape(-1)
    x, r = np.zeros(64), b.copy()
    for _ in range(2):
        ec, _ = _step(A2, S @ r, 2)
        e = P @ ec
        ae = A4 @ e
        dp, dq = _step(A4, r - ae, 4)
        x, r = x + e + dp, r - ae - dq
    xo, ro = inverse.press_multigrid(b.reshape(12, 4, 4, 12), 2, n_min=2)
    assert np.allclose(xo.reshape(-1), x, atol=1e-10)
    assert np.isclose(ro[-1], np.linalg.norm(r), rtol=1e-12)
