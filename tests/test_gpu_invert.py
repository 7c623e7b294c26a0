"""GPU parity of the iterative inverse (drt3d_planes_invert) against the fp64
oracle iteration (oracle/inverse.py, readings R15-R18): the multigrid
iteration (press_multigrid) and its single-grid special case n_min = N (press_refine).

Tolerance (DESIGN.md §2 T2): the GPU runs the iteration in fp32 (forward, backprojection and
filter fp32; dot products and the step alpha in fp64).  Each fp32 transform carries a relative
error ~ 1e-6 of its terms, and the residual-minimising step is a smooth function of them, so
after k iterations the iterate agrees with the fp64 oracle to ~ k * 1e-6 of its scale: the gate is
max |x_gpu - x_ref| <= 1e-4 * max |x_ref| and residual norms within 1e-4 relative."""
import numpy as np
import pytest

import oracle
from oracle import inverse as inv
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2501_13664_b200 as d3  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d3.lib()
    yield


def _phantom(N):
    x, y, z = np.meshgrid(*[np.arange(N)] * 3, indexing="ij")
    return np.exp(-((x - 0.45 * N) ** 2 / (0.12 * N * N) + (y - 0.55 * N) ** 2 / (0.15 * N * N)
                    + (z - 0.5 * N) ** 2 / (0.18 * N * N)))


@pytest.mark.parametrize("N,mask,iters", [(4, 0xFFF, 3), (16, 0xFFF, 5), (16, 0x0A5, 4), (32, 0xFFF, 3)])
def test_single_grid_matches_oracle(N, mask, iters):
    f = _phantom(N)
    b = oracle.drt_planes(f, mask)                               # fp64 coefficients
    x_ref, rn_ref = inv.press_refine(b, iters, mask)
    x, rn = d3.planes_invert(torch.from_numpy(b.astype(np.float32)).cuda(), iters, mask, n_min=N)
    torch.cuda.synchronize()
    x, rn = x.cpu().numpy().astype(np.float64), rn.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-4 * np.max(np.abs(x_ref))
    assert np.allclose(rn, rn_ref, rtol=1e-4, atol=0)


@pytest.mark.parametrize("N,mask,iters,n_min", [(4, 0xFFF, 2, 2), (16, 0xFFF, 3, 2), (16, 0x0A5, 2, 4),
                                                (32, 0xFFF, 2, 2), (32, 0x801, 2, 8)])
def test_multigrid_matches_oracle(N, mask, iters, n_min):
    f = _phantom(N)
    b = oracle.drt_planes(f, mask)
    x_ref, rn_ref = inv.press_multigrid(b, iters, mask, n_min=n_min)
    x, rn = d3.planes_invert(torch.from_numpy(b.astype(np.float32)).cuda(), iters, mask, n_min=n_min)
    torch.cuda.synchronize()
    x, rn = x.cpu().numpy().astype(np.float64), rn.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-4 * np.max(np.abs(x_ref))
    assert np.allclose(rn, rn_ref, rtol=1e-4, atol=0)


def test_multigrid_n64_residual_in_forward():
    """N = 64 (top level above the on-chip sizes): the residual update r <- r - A e runs inside the
    forward's final pass (TMA reduce-add, invert.cu / api.cu planes_residual); against the fp64
    oracle iteration within T3."""
    N = 64
    f = _phantom(N)
    b = oracle.drt_planes(f, 0xFFF)
    x_ref, rn_ref = inv.press_multigrid(b, 2, 0xFFF, n_min=16)
    x, rn = d3.planes_invert(torch.from_numpy(b.astype(np.float32)).cuda(), 2, 0xFFF, n_min=16)
    torch.cuda.synchronize()
    x, rn = x.cpu().numpy().astype(np.float64), rn.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-4 * np.max(np.abs(x_ref))
    assert np.allclose(rn, rn_ref, rtol=1e-4, atol=0)


def test_invert_random_cube():
    N = 8
    f = synth.normal_cube(N, 77).astype(np.float64)
    b = oracle.drt_planes(f)
    x_ref, rn_ref = inv.press_multigrid(b, 4)
    x, rn = d3.planes_invert(torch.from_numpy(b.astype(np.float32)).cuda(), 4)
    x = x.cpu().numpy()
    assert np.max(np.abs(x - x_ref)) <= 1e-4 * np.max(np.abs(x_ref))
    assert np.allclose(rn.cpu().numpy(), rn_ref, rtol=1e-4)


def test_invert_zero_iters_and_zero_input():
    N = 8
    b = torch.zeros((12, N, N, 3 * N), dtype=torch.float32, device="cuda")
    x, rn = d3.planes_invert(b, 3)
    assert float(x.abs().max()) == 0.0 and float(rn.abs().max()) == 0.0
    f = _phantom(N)
    bb = torch.from_numpy(oracle.drt_planes(f).astype(np.float32)).cuda()
    x, rn = d3.planes_invert(bb, 0)
    assert float(x.abs().max()) == 0.0
    assert abs(float(rn[0]) - float(np.linalg.norm(bb.cpu().numpy().astype(np.float64)))) <= 1e-6 * float(rn[0])


@pytest.mark.parametrize("N", [64, 128])
def test_invert_converges_large(N):
    """At sizes the oracle iteration is slow for (property checks): six multigrid
    iterations through the GPU forward / backward reduce the residual monotonically and bring
    the iterate within 15% (NRMSD) of the cube, as the oracle does at N = 16..64."""
    f = _phantom(N).astype(np.float32)
    ft = torch.from_numpy(f).cuda()
    b = d3.planes(ft[None], 0xFFF)[0]                             # fp32 forward on the GPU
    x, rn = d3.planes_invert(b, 6)
    rn = rn.cpu().numpy()
    assert np.all(np.diff(rn) < 0)
    assert rn[-1] < 0.02 * rn[0]
    err = float(torch.linalg.norm(x - ft) / torch.linalg.norm(ft))
    assert err < 0.15


def test_invert_graph_cache_states():
    """Iterations 2.. replay a captured CUDA graph cached per (device, shapes, buffers): a second call
    on the same buffers (cache hit, new coefficients), a call on other buffers (new graph) and
    iters=1 (no graph) all equal the oracle iteration."""
    N = 16
    f1, f2 = _phantom(N), np.flip(_phantom(N), 0).copy()
    b1, b2 = oracle.drt_planes(f1), oracle.drt_planes(f2)
    ref1, _ = inv.press_multigrid(b1, 3)
    ref2, _ = inv.press_multigrid(b2, 3)
    o = d3.make_opts(batch=1, in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    import ctypes
    wsb = ctypes.c_size_t(0)
    d3.lib().drt3d_planes_invert_workspace_size(N, 2, 0xFFF, ctypes.byref(o), ctypes.byref(wsb))
    ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
    cube = torch.empty((N, N, N), dtype=torch.float32, device="cuda")
    tol = lambda ref: 1e-4 * np.max(np.abs(ref))
    for b, ref in ((b1, ref1), (b2, ref2), (b1, ref1)):                # same buffers: capture, hit, hit
        x, _ = d3.planes_invert(torch.from_numpy(b.astype(np.float32)).cuda(), 3, cube=cube, workspace=ws)
        assert np.max(np.abs(x.cpu().numpy() - ref)) <= tol(ref)
    x, _ = d3.planes_invert(torch.from_numpy(b2.astype(np.float32)).cuda(), 3)   # fresh buffers: new graph
    assert np.max(np.abs(x.cpu().numpy() - ref2)) <= tol(ref2)
    ref_1, _ = inv.press_multigrid(b1, 1)
    x, _ = d3.planes_invert(torch.from_numpy(b1.astype(np.float32)).cuda(), 1, cube=cube, workspace=ws)
    assert np.max(np.abs(x.cpu().numpy() - ref_1)) <= tol(ref_1)
