"""GPU parity of the applications against oracle/apps.py, bit-exact
(integer decisions, R19-R22): argmax, threshold, plane detection on synthetic rooms, and the
ray-denoising pipeline DJT -> threshold -> DJT backprojection."""
import numpy as np
import pytest

import oracle
from oracle import apps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2501_13664_b200 as d3  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d3.lib()
    yield


def _room(N, seed=0, p=0.02):
    f = np.zeros((N, N, N), np.uint8)
    f[3, :, :] = 1
    f[:, N - 4, :] = 1
    f[:, :, 2] = 1
    f[N // 3:N // 2, N // 3:N // 2, N // 3:N // 2] = 1
    rng = np.random.default_rng(seed)
    return (f + (rng.random((N, N, N)) < p)).astype(np.uint8)


@pytest.mark.parametrize("n", [1, 1000, 4096 * 37 + 5])
def test_argmax_ties_smallest_index(n):
    rng = np.random.default_rng(n)
    c = rng.integers(-5, 5, n).astype(np.int32)
    c[rng.integers(0, n, 3)] = 7                                      # ties at the max
    assert d3.coef_argmax(torch.from_numpy(c).cuda()) == int(np.argmax(c))
    c[:] = np.iinfo(np.int32).min
    assert d3.coef_argmax(torch.from_numpy(c).cuda()) == 0


@pytest.mark.parametrize("num,den", [(0, 1), (1, 3), (9, 10), (1, 1)])
def test_threshold_matches_oracle(num, den):
    rng = np.random.default_rng(num + 7 * den)
    c = rng.integers(-1000, 100000, 123457).astype(np.int32)
    got = d3.coef_threshold(torch.from_numpy(c).cuda(), num, den).cpu().numpy()
    assert np.array_equal(got.astype(np.int64), apps.threshold(c, num, den))


@pytest.mark.parametrize("N,mask,num,den,onum,oden", [(16, 0xFFF, 1, 2, 1, 10), (32, 0xFFF, 1, 3, 1, 10),
                                                      (32, 0x0F3, 1, 4, 1, 5), (64, 0xFFF, 1, 3, 1, 20),
                                                      # 31-bit cosine fraction: the exact test needs 128 bits
                                                      (64, 0xFFF, 1, 3, 99999989, 1999999973)])
def test_detect_planes_matches_oracle(N, mask, num, den, onum, oden):
    f = _room(N, N)
    c = d3.planes(torch.from_numpy(f).cuda(), mask)                   # int32 [K,N,N,3N], GPU forward
    flags, am = d3.detect_planes(c, mask, num, den, onum, oden)
    torch.cuda.synchronize()
    ref_flags, ref_am = apps.detect_planes(c.cpu().numpy(), mask, num, den, onum, oden)
    assert int(am.item()) == ref_am
    assert np.array_equal(flags.cpu().numpy(), ref_flags)


def test_detect_room_walls_large():
    """N = 128 (the paper's scene size): the three walls are found (properties)."""
    N = 128
    f = _room(N, 5, p=0.005)
    c = d3.planes(torch.from_numpy(f).cuda(), 0xFFF)
    flags, am = d3.detect_planes(c, 0xFFF, 1, 3, 1, 10)
    idx = torch.nonzero(flags.reshape(-1)).reshape(-1).cpu().numpy()
    assert int(am.item()) in idx.tolist()
    axes = set()
    for i in idx:
        j, s1, s2, D = np.unravel_index(i, c.shape)
        n = apps.plane_normal(int(j), int(s1), int(s2), N)
        if np.count_nonzero(n) == 1:
            axes.add(int(np.argmax(np.abs(n))))
    assert axes == {0, 1, 2}


def _ray_cube(N, s1, s2, d1, d2, seed):
    n = N.bit_length() - 1
    rng = np.random.default_rng(seed)
    f = rng.integers(0, 201, (N, N, N)).astype(np.int32)
    ray = np.zeros_like(f)
    for u in range(N):
        ray[u, oracle.line(n, s1, u) + d1 - N, oracle.line(n, s2, u) + d2 - N] = 1
    return f + 100 * ray, ray


@pytest.mark.parametrize("N,num,den", [(16, 9, 10), (32, 9, 10), (32, 3, 4)])
def test_denoise_pipeline_matches_oracle(N, num, den):
    f, _ = _ray_cube(N, 5, N // 2 - 1, N + 3, N + 2, N)
    c = d3.lines(torch.from_numpy(f).cuda(), 0x001)                   # [1,N,N,2N,2N] int32
    kept = d3.coef_threshold(c, num, den)
    back = d3.lines_adjoint(kept, 0x001)
    torch.cuda.synchronize()
    ref_kept, ref_back = apps.denoise_rays(f, 0x001, num, den)
    assert np.array_equal(kept.cpu().numpy().astype(np.int64), ref_kept)
    assert np.array_equal(back.cpu().numpy().astype(np.int64), ref_back)


def test_denoise_recovers_ray_large():
    N = 64
    s1, s2, d1, d2 = 21, 40, N + 7, N + 11
    f, ray = _ray_cube(N, s1, s2, d1, d2, 9)
    c = d3.lines(torch.from_numpy(f).cuda(), 0x001)
    kept = d3.coef_threshold(c, 95, 100)
    back = d3.lines_adjoint(kept, 0x001).cpu().numpy()                # [N,N,N] (unbatched input)
    assert d3.coef_argmax(c) == np.ravel_multi_index((0, s1, s2, d1, d2), c.shape)
    top = np.argsort(back.reshape(-1))[::-1][:N]
    assert set(top.tolist()) == set(np.flatnonzero(ray).tolist())


def test_select_and_backproject_walls():
    """"When those planes are backprojected, they correspond to the walls": select the
    detected coefficients and back-project them (bit-exact against the oracle's adjoint of the
    same selection); every wall voxel lies on its detected wall plane, whose coefficient is >= N^2."""
    N = 32
    f = _room(N, 1)
    c = d3.planes(torch.from_numpy(f).cuda(), 0xFFF)
    flags, _ = d3.detect_planes(c, 0xFFF, 1, 3, 1, 10)
    sel = d3.coef_select(c, flags)
    back = d3.planes_adjoint(sel, 0xFFF)
    torch.cuda.synchronize()
    cn, fn = c.cpu().numpy().astype(np.int64), flags.cpu().numpy()
    assert np.array_equal(sel.cpu().numpy().astype(np.int64), np.where(fn != 0, cn, 0))
    ref = oracle.drt_planes_adjoint(np.where(fn != 0, cn, 0), 0xFFF)
    b = back.cpu().numpy().astype(np.int64)
    assert np.array_equal(b, ref)
    wall = np.zeros((N, N, N), bool)
    wall[3] = True
    wall[:, N - 4] = True
    wall[:, :, 2] = True
    assert b[wall].min() >= N * N
