"""GPU parity of the backprojection kernels against the
oracle's adjoints (eq:invmap3Dsummation / eq:invmap3DJsummation),
bit-exact for int32 coefficients (sums mod 2^32), plus the adjoint identity
<A f, c> = <f, A^T c> through the GPU forward and backward at larger N."""
import numpy as np
import pytest

import oracle
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


def _wrap32(x):
    return ((np.asarray(x).astype(np.int64) + 2 ** 31) % 2 ** 32) - 2 ** 31


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("mask", [0x001, 0xFFF, 0x5A3])
def test_drt_adjoint_int32(N, mask):
    K = bin(mask).count("1")
    c = synth.uniform_cube(N, 700 + N + mask, np.int32, -100, 100, batch=3 * K * 2).reshape(2, K, N, N, 3 * N)
    got = d3.planes_adjoint(torch.from_numpy(c).cuda(), mask)
    torch.cuda.synchronize()
    ref = np.stack([oracle.drt_planes_adjoint(c[b], mask) for b in range(2)])
    assert got.shape == (2, N, N, N)
    assert np.array_equal(got.cpu().numpy().astype(np.int64), _wrap32(np.round(ref)))


@pytest.mark.parametrize("N", [2, 4, 8, 16])
@pytest.mark.parametrize("mask", [0x001, 0xFFF])
def test_djt_adjoint_int32(N, mask):
    K = bin(mask).count("1")
    c = synth.uniform_cube(N, 800 + N + mask, np.int32, -100, 100, batch=4 * N * K).reshape(1, K, N, N, 2 * N, 2 * N)
    got = d3.lines_adjoint(torch.from_numpy(c).cuda(), mask)
    torch.cuda.synchronize()
    ref = oracle.djt_lines_adjoint(c[0], mask)
    assert np.array_equal(got.cpu().numpy()[0].astype(np.int64), _wrap32(np.round(ref)))


def test_drt_adjoint_float():
    N = 16
    c = synth.normal_cube(N, 901, batch=36).reshape(12, N, N, 3 * N)
    got = d3.planes_adjoint(torch.from_numpy(c).cuda(), 0xFFF).cpu().numpy()
    ref = oracle.drt_planes_adjoint(c.astype(np.float64), 0xFFF)
    scale = oracle.drt_planes_adjoint(np.abs(c).astype(np.float64), 0xFFF)
    assert np.all(np.abs(got - ref) <= 1e-5 * scale)


@pytest.mark.parametrize("N", [64, 256])
def test_drt_adjoint_identity_gpu(N):
    """<A f, c> = <f, A^T c> with the GPU forward and backward (int32, mod 2^32)."""
    f = torch.from_numpy(synth.uniform_cube(N, 950 + N, np.uint8)).cuda()
    mask = 0xFFF if N == 64 else 0x021
    K = bin(mask).count("1")
    g = torch.Generator(device="cuda").manual_seed(N)
    c = torch.randint(-3, 4, (K, N, N, 3 * N), dtype=torch.int32, device="cuda", generator=g)
    af = d3.planes(f, mask)                              # [K, N, N, 3N] int32
    atc = d3.planes_adjoint(c, mask)                     # [N, N, N] int32
    lhs = int((af.to(torch.int64) * c.to(torch.int64)).sum())
    rhs = int((f.to(torch.int64) * atc.to(torch.int64)).sum())
    # no int32 wrap here: |A f| <= 255 N^2 and |A^T c| <= 3 K N^2 * 3 < 2^31, so both sides are exact
    assert lhs == rhs


@pytest.mark.parametrize("N", [16, 32, 64, 128])
def test_djt_adjoint_single_line_closed_form(N):
    """A^T of one unit coefficient (s1, s2, D1, D2) is the indicator of that digital line
    (eq:3DfDJT): voxels (u, l_s1(u) + D1 - N, l_s2(u) + D2 - N) inside the cube."""
    n = N.bit_length() - 1
    cases = [(0, 0, N, N), (N - 1, N - 1, N, N), (N // 3, 2 * N // 3, N + 5, N + 1), (1, N - 2, 3, 2 * N - 2)]
    for (s1, s2, D1, D2) in cases:
        c = torch.zeros((1, 1, N, N, 2 * N, 2 * N), dtype=torch.int32, device="cuda")
        c[0, 0, s1, s2, D1, D2] = 1
        got = d3.lines_adjoint(c, 0x001)[0].cpu().numpy()
        ref = np.zeros((N, N, N), np.int64)
        for u in range(N):
            y, z = oracle.line(n, s1, u) + D1 - N, oracle.line(n, s2, u) + D2 - N
            if 0 <= y < N and 0 <= z < N:
                ref[u, y, z] = 1
        assert np.array_equal(got.astype(np.int64), ref), (s1, s2, D1, D2)


@pytest.mark.parametrize("N", [32, 64, 128])
def test_drt_adjoint_single_plane_closed_form(N):
    """A^T of one unit coefficient (s1, s2, D) of dodecant 0 is the indicator of that digital
    plane (eq:3DfDRT): voxels (x, y, l_s1(x) + l_s2(y) + D - 2N) inside."""
    n = N.bit_length() - 1
    for (s1, s2, D) in [(0, 0, 2 * N + 3), (N - 1, 1, 2 * N - 5), (N // 3, 2 * N // 3, N + 7)]:
        c = torch.zeros((1, 1, N, N, 3 * N), dtype=torch.int32, device="cuda")
        c[0, 0, s1, s2, D] = 1
        got = d3.planes_adjoint(c, 0x001)[0].cpu().numpy()
        ref = np.zeros((N, N, N), np.int64)
        for x in range(N):
            for y in range(N):
                z = oracle.line(n, s1, x) + oracle.line(n, s2, y) + D - 2 * N
                if 0 <= z < N:
                    ref[x, y, z] = 1
        assert np.array_equal(got.astype(np.int64), ref), (s1, s2, D)


@pytest.mark.parametrize("N", [512, 1024])
def test_drt_adjoint_single_plane_max_sizes(N):
    """Three-pass backprojection plans at the largest sizes: one unit coefficient of dodecant 0
    back-projects to exactly its digital plane (eq:3DfDRT)."""
    n = N.bit_length() - 1
    s1, s2, D = N // 3, 2 * N // 3 + 1, N + 11
    c = torch.zeros((1, N, N, 3 * N), dtype=torch.int32, device="cuda")
    c[0, s1, s2, D] = 1
    got = d3.planes_adjoint(c, 0x001)
    del c
    nzg = torch.nonzero(got).cpu().numpy()
    ref = []
    l1 = [oracle.line(n, s1, u) for u in range(N)]
    l2 = [oracle.line(n, s2, u) for u in range(N)]
    for x in range(N):
        for y in range(N):
            z = l1[x] + l2[y] + D - 2 * N
            if 0 <= z < N:
                ref.append((x, y, z))
    assert int(got.sum()) == len(ref)
    assert sorted(map(tuple, nzg.tolist())) == ref
