"""Pins of the iterative-inverse oracle (oracle/inverse.py).

The filter is pinned to the values the paper prints (tests/golden/highpass_h.txt) and to
properties fixed by the mathematics (zero DC response, the 48 cube symmetries, annihilation of
affine functions away from the border, agreement with scipy's correlation).  The iteration is
pinned by properties that any correct implementation of R15-R16 has and that a wrong adjoint,
sign or step breaks: the exact solution is a fixed point, the residual never increases, the step
minimises the residual along its direction, and the iterate converges to the true cube."""
import itertools
from fractions import Fraction
import os

import numpy as np
import pytest

import oracle
from oracle import inverse as inv

GOLD = os.path.join(os.path.dirname(__file__), "golden", "highpass_h.txt")


def _golden_h():
    h = np.zeros((3, 3, 3))
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        a, b, *v = line.split()
        for c, t in enumerate(v):
            h[int(a), int(b), c] = float(Fraction(t))
    return h


def _phantom(N, seed=0):
    x, y, z = np.meshgrid(*[np.arange(N)] * 3, indexing="ij")
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.3 * N, 0.7 * N, 3)
    w = rng.uniform(0.1 * N * N, 0.2 * N * N, 3)
    return np.exp(-((x - c[0]) ** 2 / w[0] + (y - c[1]) ** 2 / w[1] + (z - c[2]) ** 2 / w[2]))


def test_filter_matches_paper():
    assert np.array_equal(inv.highpass_kernel(), _golden_h())


def test_filter_zero_dc_and_symmetry():
    h = inv.highpass_kernel()
    assert abs(h.sum()) < 1e-15                       # zero DC response
    for perm in itertools.permutations(range(3)):
        for flips in itertools.product([False, True], repeat=3):
            g = np.transpose(h, perm)
            for ax, f in enumerate(flips):
                if f:
                    g = np.flip(g, ax)
            assert np.array_equal(g, h)


def test_highpass_kills_affine_interior():
    N = 8
    x, y, z = np.meshgrid(*[np.arange(N)] * 3, indexing="ij")
    f = 3.0 + 2.0 * x - 1.5 * y + 0.25 * z
    out = inv.highpass(f)
    assert np.allclose(out[1:-1, 1:-1, 1:-1], 0.0, atol=1e-12)
    assert not np.allclose(out[0], 0.0)             # zero padding: the border sees the cut


def test_highpass_equals_library_correlation():
    ndimage = pytest.importorskip("scipy.ndimage")
    g = np.random.default_rng(3).normal(size=(9, 9, 9))
    ref = ndimage.correlate(g, _golden_h(), mode="constant", cval=0.0)
    assert np.allclose(inv.highpass(g), ref, atol=1e-12)


def test_exact_solution_is_fixed_point():
    N = 8
    f = _phantom(N, 1)
    b = oracle.drt_planes(f)
    x, rn = inv.press_refine(b, 2, x0=f)
    assert rn[0] < 1e-9 * np.linalg.norm(b)
    assert np.allclose(x, f, atol=1e-9)


@pytest.mark.parametrize("mask", [0xFFF, 0x00F])
def test_residual_monotone_and_step_minimises(mask):
    N = 8
    f = np.random.default_rng(5).uniform(0, 1, (N, N, N))
    b = oracle.drt_planes(f, mask)
    x, rn = inv.press_refine(b, 6, mask)
    assert np.all(np.diff(rn) <= 1e-9 * rn[0])
    # the step of one iteration minimises ||r - a A p|| over a (perturbing a increases it)
    r = b - oracle.drt_planes(x, mask)
    p = inv.highpass(oracle.drt_planes_adjoint(r, mask))
    q = oracle.drt_planes(p, mask)
    a = float(np.sum(r * q) / np.sum(q * q))
    best = np.linalg.norm(r - a * q)
    for e in (0.9, 1.1):
        assert np.linalg.norm(r - e * a * q) > best


def test_converges_to_the_cube():
    """the iteration recovers the input (NRMSD falls; residual ~1e-2 after 20)."""
    N = 16
    f = _phantom(N, 0)
    b = oracle.drt_planes(f)
    x5, _ = inv.press_refine(b, 5)
    x20, rn = inv.press_refine(b, 20)
    assert inv.nrmsd(x20, f) < 0.12
    assert inv.nrmsd(x20, f) < 0.5 * inv.nrmsd(x5, f)
    assert rn[-1] < 0.02 * rn[0]


# ---------------------------------------------------------------- multigrid (R18)

def test_prolong_delta_fills_block():
    xc = np.zeros((4, 4, 4))
    xc[1, 2, 3] = 5.0
    x = inv.prolong(xc)
    assert x.shape == (8, 8, 8) and x.sum() == 8 * 5.0
    assert np.all(x[2:4, 4:6, 6:8] == 5.0)


def test_restrict_mass_identity():
    """Sum over (s1, s2, d) of S(A_N P x) equals that of A_{N/2} x exactly: each (s1, s2) family
    sums to the cube's mass, P multiplies mass by 8, S keeps (N/2)^2 of the N^2
    fine families and divides by 8 -- the 1/8 of PAPER.md:599 is exactly mass-preserving."""
    for N in (4, 8, 16):
        xc = np.random.default_rng(N).integers(0, 9, (N // 2,) * 3).astype(np.float64)
        lhs = inv.restrict(oracle.drt_planes(inv.prolong(xc)))
        rhs = oracle.drt_planes(xc)
        assert lhs.shape == rhs.shape
        assert np.array_equal(lhs.sum(axis=(1, 2, 3)), rhs.sum(axis=(1, 2, 3)))


def test_restrict_first_order_consistency():
    """S A_N P = A_{N/2} up to O(1/N) on smooth cubes (the coarse grid sees the same planes)."""
    prev = None
    for N in (8, 16, 32):
        xc = _phantom(N // 2, 4)
        lhs = inv.restrict(oracle.drt_planes(inv.prolong(xc)))
        rhs = oracle.drt_planes(xc)
        e = np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs)
        assert e < 1.0 / N
        if prev is not None:
            assert e < 0.6 * prev
        prev = e


def test_multigrid_at_full_size_is_single_grid():
    N = 8
    b = oracle.drt_planes(_phantom(N, 2))
    x1, r1 = inv.press_multigrid(b, 3, n_min=N)
    x2, r2 = inv.press_refine(b, 3)
    assert np.allclose(x1, x2, atol=1e-12) and np.allclose(r1, r2, rtol=1e-12)


@pytest.mark.parametrize("N", [16, 32])
def test_multigrid_converges(N):
    """a half-dozen multigrid iterations give good results; faster than single grid."""
    f = _phantom(N, 0)
    b = oracle.drt_planes(f)
    x6, rn = inv.press_multigrid(b, 6)
    assert np.all(np.diff(rn) < 0)
    assert inv.nrmsd(x6, f) < 0.15
    xs, _ = inv.press_refine(b, 6)
    assert inv.nrmsd(x6, f) < 0.5 * inv.nrmsd(xs, f)
