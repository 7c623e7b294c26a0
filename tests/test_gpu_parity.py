"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer configs must match bit for bit; the float config within the
tolerance DESIGN.md derives (|gpu - ref64| <= 1e-5 * sum|terms|, C-amb-14).
Inputs are the seeded synthetic cubes of synth/ (BASELINE.json configs 1-5).
"""
import numpy as np
import pytest

import oracle
import oracle_pool
import synth
from oracle import tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2501_13664_b200 as d3  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d3.lib()
    yield


def _gpu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _4d(a):
    return a[None] if a.ndim == 3 else a


def _planes(cube, mask, **kw):
    """[B][N][N][N] -> [B][K]...; a 3D cube -> [K]... (the oracle's convention)."""
    out = d3.planes(_gpu(_4d(cube)), mask, **kw)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    return res[0] if cube.ndim == 3 else res


def _lines(cube, mask, **kw):
    out = d3.lines(_gpu(_4d(cube)), mask, **kw)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    return res[0] if cube.ndim == 3 else res


# ------------------------------------------------------------ 3D DRT

def test_cfg1_n16_i32_dodecant0():
    cube = synth.config_input(1)                       # [1][16][16][16] int32
    got = _planes(cube, 0x001)
    ref = oracle.drt_planes(cube, 0x001)
    assert got.dtype == np.int32 and got.shape == (1, 1, 16, 16, 48)
    assert np.array_equal(got.astype(np.int64), ref)


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("dtype", [np.uint8, np.int32])
def test_drt_random_all_dodecants(N, dtype):
    lo, hi = (0, 255) if dtype == np.uint8 else (-1000, 1000)
    cube = synth.uniform_cube(N, 100 + N, dtype, lo, hi, batch=2 if N <= 32 else 1)
    got = _planes(cube, 0xFFF)
    ref = oracle.drt_planes(cube, 0xFFF)
    assert np.array_equal(got.astype(np.int64), ref)


def _full_parity(tmp_path, cube, mask=0xFFF, transform="drt", per_task=1, **kw):
    """GPU call on [B][N][N][N] cubes, then every element of every (cube, dodecant) against the
    oracle recursion in parallel processes (tests/oracle_pool.py)."""
    cube = _4d(cube)
    if transform == "drt":
        got = d3.planes(_gpu(cube), mask, **kw)
    else:
        got = d3.lines(_gpu(cube), mask, **kw)
    torch.cuda.synchronize()
    host = got.cpu().numpy()
    del got
    bad = oracle_pool.compare_all(tmp_path, cube, host, mask, transform, kw.get("table", 0), per_task=per_task)
    assert not bad, bad[:8]
    return host


@pytest.mark.parametrize("N", [128, 256])
@pytest.mark.parametrize("kind", ["u8", "i32", "f32"])
def test_drt_large_all_dodecants_full(N, kind, tmp_path):
    """N = 128 and 256, all 12 dodecants, every element: the K = 4 first passes (SWAR u8, 32-bit
    i32 / f32) and the K = 3 / K = 4 final passes, including the 32-bit TMA-store tile."""
    if kind == "u8":
        cube = synth.uniform_cube(N, 700 + N, np.uint8)
    elif kind == "i32":
        cube = synth.uniform_cube(N, 710 + N, np.int32, -1000, 1000)
    else:
        cube = synth.normal_cube(N, 720 + N)
    _full_parity(tmp_path, cube)


def test_drt_saturated_n256_full(tmp_path):
    """All voxels 255 at N = 256, all 12 dodecants, every element: the tightest case of the u16
    SWAR lanes (stage-4 sums up to 255 * 256 = 65280 of 65535) and of the u16 stage buffer."""
    cube = np.full((256, 256, 256), 255, np.uint8)
    host = _full_parity(tmp_path, cube)
    assert int(host.max()) == 255 * 256 * 256


@pytest.mark.parametrize("table", [d3.DRT3D_TABLE_PRINTED, d3.DRT3D_TABLE_SHARED])
@pytest.mark.parametrize("N", [8, 64])
def test_drt_other_tables(N, table):
    cube = synth.uniform_cube(N, 200 + N, np.uint8)
    got = _planes(cube, 0xFFF, table=table)
    ref = oracle.drt_planes(cube, 0xFFF, table)
    assert np.array_equal(got.astype(np.int64), ref)


@pytest.mark.parametrize("table", [d3.DRT3D_TABLE_PRINTED, d3.DRT3D_TABLE_SHARED])
def test_drt_other_tables_n128_batched_full(table, tmp_path):
    """N = 128 u8, two cubes, the PRINTED and SHARED tables, every element: the first pass's TMA
    brick staging (DESIGN.md §5 item 9) over orientations the default table does not have (z' along
    +x / +y, i.e. an unreversed long brick side off the contiguous axis) and over the batch
    coordinate of its tensor maps."""
    cube = synth.uniform_cube(128, 1280 + table, np.uint8, batch=2).reshape(2, 128, 128, 128)
    _full_parity(tmp_path, cube, table=table, per_task=2)


@pytest.mark.parametrize("mask", [0x001, 0x020, 0x210, 0x801, 0xAAA])
def test_drt_masks(mask):
    cube = synth.uniform_cube(32, 300 + mask, np.uint8)
    got = _planes(cube, mask)
    ref = oracle.drt_planes(cube, mask)
    assert np.array_equal(got.astype(np.int64), ref)


def test_cfg2_n64_sheets_full():
    cube = synth.config_input(2)
    got = _planes(cube, 0xFFF)
    ref = oracle.drt_planes(cube, 0xFFF)
    assert np.array_equal(got.astype(np.int64), ref)


def test_cfg3_n256_full_size(tmp_path):
    """BASELINE config 3 at full size, same launch as bench.py: every element of all 12
    dodecants against the oracle recursion (12 processes), plus the mass and support
    invariants checked on the device."""
    cube = synth.config_input(3)
    N = 256
    gpu = d3.planes(_gpu(cube), 0xFFF)[0]             # cube is [1][N][N][N] -> [12][N][N][3N] int32 on device
    torch.cuda.synchronize()
    f = cube[0]
    # mass: each (s1, s2) column sums to the cube total
    tot = int(f.astype(np.int64).sum())
    sums = gpu.to(torch.int64).sum(dim=3)
    assert bool((sums == tot).all())
    # support: zero below D = 2N - s1 - s2
    s = torch.arange(N, device="cuda")
    lim = 2 * N - s[:, None] - s[None, :]
    D = torch.arange(3 * N, device="cuda")
    below = D[None, None, :] < lim[:, :, None]
    assert int(gpu.masked_select(below.unsqueeze(0).expand_as(gpu)).abs().sum()) == 0
    host = gpu.cpu().numpy()[None]
    del gpu
    bad = oracle_pool.compare_all(tmp_path, cube, host, 0xFFF)
    assert not bad, bad[:8]


def test_cfg5_batched_f32(tmp_path):
    """Config 5: 256 cubes N=32 f32, 12 dodecants, every element of every cube.  Tolerance
    (T1): |gpu - ref64| <= 1e-5 * sum|terms| per element, sum|terms| = the fp64
    transform of |f|; empty planes must be exactly 0."""
    cube = synth.config_input(5)                       # [256][32][32][32] f32
    got = _planes(cube, 0xFFF)                         # [256][12][32][32][96]
    assert got.dtype == np.float32 and np.isfinite(got).all()
    bad = oracle_pool.compare_all(tmp_path, cube, got, 0xFFF, per_task=48)
    assert not bad, bad[:8]


def test_drt_float_small_all_tables():
    cube = synth.normal_cube(16, 9, batch=3)
    got = _planes(cube, 0xFFF)
    for b in range(3):
        ref = oracle.drt_planes(cube[b].astype(np.float64), 0xFFF)
        refabs = oracle.drt_planes(np.abs(cube[b]).astype(np.float64), 0xFFF)
        assert np.all(np.abs(got[b] - ref) <= 1e-5 * refabs)


def test_drt_n16_one_cta_batched():
    """N = 16 runs every stage of an instance in one CTA (k_sep16.cu): one cube x 12 dodecants and
    16 cubes x 12 (more instances than SMs); int32 bit-exact, fp32 within the T1 gate."""
    for batch in (1, 16):
        cube = synth.uniform_cube(16, 70 + batch, np.int32, -1000, 1000, batch=batch)
        got = _planes(cube, 0xFFF)
        for b in range(batch):
            assert np.array_equal(got[b].astype(np.int64), oracle.drt_planes(cube[b], 0xFFF))
        cubef = synth.normal_cube(16, 80 + batch, batch=batch)
        gotf = _planes(cubef, 0xFFF)
        for b in range(batch):
            ref = oracle.drt_planes(cubef[b].astype(np.float64), 0xFFF)
            refabs = oracle.drt_planes(np.abs(cubef[b]).astype(np.float64), 0xFFF)
            assert np.all(np.abs(gotf[b] - ref) <= 1e-5 * refabs)


def test_drt_mosaic_layout():
    # N = 128: the u16 SWAR first pass and the K = 3 final pass's mosaic stores
    for N in (4, 32, 128):
        cube = synth.uniform_cube(N, 400 + N, np.uint8)
        got = _planes(cube, 0xFFF, layout=d3.DRT3D_LAYOUT_MOSAIC)
        assert got.shape == (4 * N, 4 * N, 3 * N - 2)
        ref = oracle.mosaic(oracle.drt_planes(cube, 0xFFF))
        assert np.array_equal(got.astype(np.int64), ref)


def test_drt_edge_cases():
    # zero cube -> zeros; delta at origin -> 1 at D = 2N for all slopes
    N = 64
    z = np.zeros((N, N, N), np.uint8)
    assert not _planes(z, 0xFFF).any()
    z[0, 0, 0] = 1
    got = _planes(z, 0x001)[0]
    exp = np.zeros_like(got)
    exp[:, :, 2 * N] = 1
    assert np.array_equal(got, exp)
    # maximum voxels: 255 everywhere at N=256 reaches 255 N^2 = 16.7M (fits int32)
    full = np.full((1, 256, 256, 256), 255, np.uint8)
    g = d3.planes(_gpu(full), 0x001)
    torch.cuda.synchronize()
    assert int(g[0, 0, 0, 0, 2 * 256]) == 255 * 256 * 256
    assert int(g.max()) == 255 * 256 * 256


def test_drt_deterministic():
    cube = synth.uniform_cube(64, 7, np.uint8)
    a = _planes(cube, 0xFFF)
    b = _planes(cube, 0xFFF)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("N", [8, 16, 32, 64])
def test_drt_int32_wraps_mod_2_32(N):
    # int32 output = exact sum mod 2^32 (include/drt3d.h); N = 16 / 32 run the on-chip kernels
    # (k_sep16 / k_sep32, whose partial sums P, Q, U wrap too), 8 and 64 the pass kernels
    cube = np.full((N, N, N), 2 ** 30, np.int32)
    cube[::3, 1::2, ::5] = -(2 ** 31) + 7
    got = _planes(cube, 0xFFF)
    ref = oracle.drt_planes(cube.astype(np.int64), 0xFFF)
    assert np.array_equal(got.astype(np.int64), ((ref + 2 ** 31) % 2 ** 32) - 2 ** 31)


@pytest.mark.parametrize("N", [16, 32])
def test_drt_saturated_u8_on_chip(N):
    # all-255 u8 cubes through the on-chip kernels: the largest sums (255 N^2), all 12 dodecants
    cube = np.full((2, N, N, N), 255, np.uint8)
    got = _planes(cube, 0xFFF)
    ref = oracle.drt_planes(cube[0], 0xFFF)
    assert np.array_equal(got[0].astype(np.int64), ref) and np.array_equal(got[1], got[0])


# ------------------------------------------------------------ 3D DJT

def test_cfg4_djt_n64_full():
    cube = synth.config_input(4)
    got = _lines(cube, 0x001)
    ref = oracle.djt_lines(cube, 0x001)
    assert got.shape == (1, 1, 64, 64, 128, 128)
    assert np.array_equal(got.astype(np.int64), ref)


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("dtype", [np.uint8, np.int32, np.float32])
def test_djt_random_all_dodecants(N, dtype):
    if dtype == np.float32:
        cube = synth.normal_cube(N, 500 + N, batch=2)
    else:
        cube = synth.uniform_cube(N, 500 + N, dtype, 0, 255, batch=2)
    got = _lines(cube, 0xFFF)
    if dtype == np.float32:
        for b in range(2):
            ref = oracle.djt_lines(cube[b].astype(np.float64), 0xFFF)
            refabs = oracle.djt_lines(np.abs(cube[b]).astype(np.float64), 0xFFF)
            assert np.all(np.abs(got[b] - ref) <= 1e-5 * refabs)
    else:
        ref = oracle.djt_lines(cube, 0xFFF)
        assert np.array_equal(got.astype(np.int64), ref)


@pytest.mark.parametrize("kind", ["i32", "f32"])
def test_djt_n64_all_dodecants_full(kind, tmp_path):
    """DJT N = 64 on all 12 dodecants with 32-bit voxels, every element (K = 3 passes over
    32-bit stage buffers)."""
    if kind == "i32":
        cube = synth.uniform_cube(64, 800, np.int32, -1000, 1000)
    else:
        cube = synth.normal_cube(64, 801)
    _full_parity(tmp_path, cube, transform="djt")


def test_djt_n128_sampled():
    N = 128
    cube = synth.uniform_cube(N, 600, np.uint8)
    gpu = d3.lines(_gpu(cube[None]), 0x001)[0, 0]
    torch.cuda.synchronize()
    assert bool((gpu.to(torch.int64).sum(dim=(2, 3)) == int(cube.astype(np.int64).sum())).all())
    host = gpu.cpu().numpy()
    rng = np.random.default_rng(6)
    for _ in range(300):
        s1, s2, D1, D2 = (int(t) for t in rng.integers(0, [N, N, 2 * N, 2 * N]))
        assert host[s1, s2, D1, D2] == oracle.djt_point(cube, s1, s2, D1, D2)


# ------------------------------------------------------------ maximum sizes (three-pass plans)

def test_drt_n512_sampled():
    """N = 512 (three radix passes): two dodecants, mass and support on every column, sampled
    outputs against eq:3DfDRT by direct summation (oracle.drt_point)."""
    N, mask = 512, 0x801
    f = synth.uniform_cube(N, 512, np.uint8)
    gpu = d3.planes(_gpu(f[None]), mask)[0]                          # [2][N][N][3N] int32, on the device
    torch.cuda.synchronize()
    tot = int(f.astype(np.int64).sum())
    assert bool((gpu.to(torch.int64).sum(dim=3) == tot).all())
    s = torch.arange(N, device="cuda")
    lim = 2 * N - s[:, None] - s[None, :]
    below = torch.arange(3 * N, device="cuda")[None, None, :] < lim[:, :, None]
    for j in range(2):
        assert int(gpu[j].masked_select(below).abs().sum()) == 0
    rows = tables.DRT_HEMISPHERE
    rng = np.random.default_rng(5)
    for j, k in enumerate((0, 11)):
        g = np.ascontiguousarray(oracle.orient(f, rows[k]), dtype=np.float64)   # orient once (1 GB)
        for _ in range(25):
            s1, s2 = int(rng.integers(0, N)), int(rng.integers(0, N))
            Dd = int(rng.integers(2 * N - s1 - s2, 3 * N))
            assert int(gpu[j, s1, s2, Dd]) == oracle.drt_point(g, s1, s2, Dd)


def test_drt_n1024_sparse_sampled():
    """N = 1024, the largest size the boundary accepts (12.9 GB output for one dodecant): a sparse
    cube, mass and support on every column, sampled outputs by direct summation over its
    non-zero voxels with the oracle's digital line (eq:3DfDRT, eq:digitalLine)."""
    N, n = 1024, 10
    rng = np.random.default_rng(1024)
    nz = 3000
    xs, ys, zs = (rng.integers(0, N, nz) for _ in range(3))
    vs = rng.integers(1, 256, nz)
    f = np.zeros((N, N, N), np.uint8)
    f[xs, ys, zs] = vs
    xs, ys, zs = np.nonzero(f)
    vs = f[xs, ys, zs].astype(np.int64)
    gpu = d3.planes(_gpu(f[None]), 0x001)[0, 0]                      # [N][N][3N] int32 (dodecant 0: identity)
    torch.cuda.synchronize()
    assert bool((gpu.to(torch.int64).sum(dim=2) == int(vs.sum())).all())
    lut = {}

    def line(s, u):
        key = (s, u)
        if key not in lut:
            lut[key] = oracle.line(n, s, u)
        return lut[key]
    for _ in range(12):
        s1, s2 = int(rng.integers(0, N)), int(rng.integers(0, N))
        ls1 = np.array([line(s1, int(x)) for x in xs])
        ls2 = np.array([line(s2, int(y)) for y in ys])
        # every D with a voxel on it, plus random D: the plane through voxel i has D = z - l1 - l2 + 2N
        Ds = set((zs - ls1 - ls2 + 2 * N).tolist()[:20]) | {int(d) for d in rng.integers(0, 3 * N, 5)}
        for Dd in Ds:
            ref = int(vs[zs == ls1 + ls2 + Dd - 2 * N].sum())
            assert int(gpu[s1, s2, Dd]) == ref


def test_djt_n256_sampled():
    """N = 256, the largest DJT whose output fits one B200 (4 N^4 int32 = 68.7 GB per dodecant):
    mass per (s1, s2) plane and sampled outputs against eq:3DfDJT by direct summation."""
    N = 256
    cube = synth.uniform_cube(N, 256, np.uint8)
    gpu = d3.lines(_gpu(cube[None]), 0x001)[0, 0]                    # [N][N][2N][2N] int32 on the device
    torch.cuda.synchronize()
    tot = int(cube.astype(np.int64).sum())
    for s1 in range(0, N, 1):
        assert bool((gpu[s1].to(torch.int64).sum(dim=(1, 2)) == tot).all()), s1
    g = np.ascontiguousarray(cube, dtype=np.float64)
    rng = np.random.default_rng(7)
    for _ in range(200):
        s1, s2, D1, D2 = (int(t) for t in rng.integers(0, [N, N, 2 * N, 2 * N]))
        assert int(gpu[s1, s2, D1, D2]) == oracle.djt_point(g, s1, s2, D1, D2)


def test_drt_batched_multichunk_overlap():
    """9 cubes x 12 dodecants at N=128 (108 instances of 5.2 MB stage buffers: more than one
    512 MB chunk), so the call runs several chunks with the cross-stream overlap and alternating
    buffer sets: every cube's result equals its single-cube call, and
    sampled outputs equal the oracle's direct sums."""
    N, B = 128, 9
    cubes = synth.uniform_cube(N, 900, np.uint8, batch=B).reshape(B, N, N, N)
    o = d3.make_opts(batch=B, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)
    ws = d3.drt3d_planes_workspace_size(N, 0xFFF, o)
    o1 = d3.make_opts(batch=1, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)
    assert ws > d3.drt3d_planes_workspace_size(N, 0xFFF, o1)          # several chunks, two buffer sets
    got = d3.planes(_gpu(cubes), 0xFFF)                              # [B][12][N][N][3N]
    for b in (0, 4, 8):
        one = d3.planes(_gpu(cubes[b][None]), 0xFFF)[0]
        assert bool(torch.equal(got[b], one)), b
    torch.cuda.synchronize()
    rng = np.random.default_rng(9)
    rows = tables.DRT_HEMISPHERE
    for b in (0, 8):
        for k in (0, 7):
            g = np.ascontiguousarray(oracle.orient(cubes[b], rows[k]), dtype=np.float64)
            for _ in range(10):
                s1, s2 = int(rng.integers(0, N)), int(rng.integers(0, N))
                Dd = int(rng.integers(2 * N - s1 - s2, 3 * N))
                assert int(got[b, k, s1, s2, Dd]) == oracle.drt_point(g, s1, s2, Dd)


# ------------------------------------------------------------ host-buffer entry points (e2e path)

def _host_call(kind, cube_np, mask, batch):
    """drt3d_planes_host / djt3d_lines_host: pinned host cube in, pinned host output out."""
    N = cube_np.shape[-1]
    K = bin(mask).count("1")
    o = d3.make_opts(batch=batch, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)
    hcube = torch.from_numpy(np.ascontiguousarray(cube_np)).pin_memory()
    shape = (batch, K, N, N, 3 * N) if kind == "drt" else (batch, K, N, N, 2 * N, 2 * N)
    hout = torch.empty(shape, dtype=torch.int32).pin_memory()
    dcube = torch.empty(hcube.shape, dtype=torch.uint8, device="cuda")
    dout = torch.empty(shape, dtype=torch.int32, device="cuda")
    wsb = (d3.drt3d_planes_workspace_size if kind == "drt" else d3.djt3d_lines_workspace_size)(N, mask, o)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    fn = d3.drt3d_planes_host if kind == "drt" else d3.djt3d_lines_host
    st = torch.cuda.current_stream().cuda_stream
    assert fn(hcube.data_ptr(), N, mask, hout.data_ptr(), o, dcube.data_ptr(), dout.data_ptr(), ws.data_ptr(), wsb,
              st) == d3.DRT3D_OK
    torch.cuda.current_stream().synchronize()
    return hout.numpy()


@pytest.mark.parametrize("N,mask,batch", [(64, 0xFFF, 1), (64, 0x5A3, 1), (32, 0x001, 1), (32, 0xFFF, 2),
                                          (256, 0xFFF, 1)])
def test_drt_host_entry(N, mask, batch):
    """The host-buffer call (dodecant groups copied out while the next group computes, batch 1)
    returns exactly the device-buffer result; small sizes also against the oracle."""
    cubes = synth.uniform_cube(N, 31 + N, np.uint8, batch=batch).reshape(batch, N, N, N)
    got = _host_call("drt", cubes, mask, batch)
    dev = d3.planes(_gpu(cubes), mask).cpu().numpy()
    assert np.array_equal(got, dev)
    if N <= 64:
        assert np.array_equal(got[0].astype(np.int64), oracle.drt_planes(cubes[0], mask))


def test_djt_host_entry():
    N, mask = 16, 0x0F1
    cube = synth.uniform_cube(N, 77, np.uint8)
    got = _host_call("djt", cube[None], mask, 1)
    assert np.array_equal(got[0].astype(np.int64), oracle.djt_lines(cube, mask))


def test_entry_points_on_a_side_stream():
    """Every call enqueues on the caller's stream (internal streams fork from and join it): run the
    forward (multi-chunk batch), backprojection, inverse and detection on a non-default stream,
    synchronise only that stream, and compare with default-stream results."""
    N, B = 128, 9
    cubes = synth.uniform_cube(N, 901, np.uint8, batch=B).reshape(B, N, N, N)
    ref = d3.planes(_gpu(cubes), 0xFFF)
    small = _gpu(synth.uniform_cube(16, 5, np.uint8))
    ref_adj = d3.planes_adjoint(d3.planes(small, 0xFFF), 0xFFF)
    ref_inv, _ = d3.planes_invert(d3.planes(small.float(), 0xFFF), 3)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        got = d3.planes(_gpu(cubes), 0xFFF)
        adj = d3.planes_adjoint(d3.planes(small, 0xFFF), 0xFFF)
        xin, _ = d3.planes_invert(d3.planes(small.float(), 0xFFF), 3)
        flags, _ = d3.detect_planes(got[0], 0xFFF, 1, 3, 1, 10)
    s.synchronize()
    assert bool(torch.equal(got, ref))
    assert bool(torch.equal(adj, ref_adj))
    assert bool(torch.equal(xin, ref_inv))                             # deterministic kernels
    ref_flags, _ = d3.detect_planes(ref[0], 0xFFF, 1, 3, 1, 10)
    torch.cuda.synchronize()
    assert bool(torch.equal(flags, ref_flags))


def test_concurrent_host_threads():
    """Three host threads, each on its own stream, call the forward (multi-chunk batch),
    backprojection and inverse concurrently (ctypes releases the GIL): results equal the serial
    ones (per-thread auxiliary streams, the graph cache's lock, per-device attribute flags)."""
    import threading
    N, B = 128, 9
    cubes = [synth.uniform_cube(N, 950 + t, np.uint8, batch=B).reshape(B, N, N, N) for t in range(3)]
    small = [_gpu(synth.uniform_cube(16, 960 + t, np.uint8)) for t in range(3)]
    ref = [d3.planes(_gpu(c), 0xFFF) for c in cubes]
    ref_adj = [d3.planes_adjoint(d3.planes(s, 0xFFF), 0xFFF) for s in small]
    ref_inv = [d3.planes_invert(d3.planes(s.float(), 0xFFF), 3)[0] for s in small]
    torch.cuda.synchronize()
    out, errors = [None] * 3, []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    a = d3.planes(_gpu(cubes[t]), 0xFFF)
                    b = d3.planes_adjoint(d3.planes(small[t], 0xFFF), 0xFFF)
                    c, _ = d3.planes_invert(d3.planes(small[t].float(), 0xFFF), 3)
            s.synchronize()
            out[t] = (a, b, c)
        except Exception as e:                                         # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(3)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(3):
        assert bool(torch.equal(out[t][0], ref[t]))
        assert bool(torch.equal(out[t][1], ref_adj[t]))
        assert bool(torch.equal(out[t][2], ref_inv[t]))


def test_binding_validates_user_buffers():
    """The binding checks caller-supplied buffers and tells the C ABI their real sizes (no
    writes past a short workspace, no coefficient reads past a buffer with fewer dodecants)."""
    cube = _gpu(synth.uniform_cube(32, 61, np.uint8))
    big = _gpu(synth.uniform_cube(64, 61, np.uint8))                   # N = 64 has a workspace
    need = d3.drt3d_planes_workspace_size(64, 0xFFF, d3.make_opts())
    assert need > 0
    with pytest.raises(d3.Drt3dError):
        d3.planes(big, 0xFFF, workspace=torch.empty(need // 2, dtype=torch.uint8, device="cuda"))
    with pytest.raises(d3.Drt3dError):
        d3.planes(cube, 0xFFF, out=torch.empty((12, 32, 32, 95), dtype=torch.int32, device="cuda"))
    with pytest.raises(d3.Drt3dError):
        d3.planes(cube, 0xFFF, out=torch.empty((12, 32, 32, 96), dtype=torch.float32, device="cuda"))
    one = d3.planes(cube, 0x001)                            # [1, N, N, 3N]
    with pytest.raises(d3.Drt3dError):
        d3.planes_adjoint(one, 0xFFF)                       # 12 dodecants' worth from a 1-dodecant buffer
    with pytest.raises(d3.Drt3dError):
        d3.planes_invert(one.float(), 2, mask=0x003)
    with pytest.raises(d3.Drt3dError):
        d3.planes_adjoint(one, 0x001, cube=torch.empty((32, 32, 31), dtype=torch.int32, device="cuda"))
    # a correctly shaped user buffer is used in place
    out = torch.empty((1, 32, 32, 96), dtype=torch.int32, device="cuda")
    assert d3.planes(cube, 0x001, out=out).data_ptr() == out.data_ptr()
    torch.cuda.synchronize()
    assert torch.equal(out, one)


def test_explicit_stream_argument():
    """stream= as a torch stream or a raw handle that is not the current stream: temporaries are
    allocated on that stream, results equal the current-stream call."""
    cube = synth.uniform_cube(64, 62, np.int32, -100, 100)
    ref = _planes(cube, 0xFFF)
    s = torch.cuda.Stream()
    g = _gpu(cube)
    torch.cuda.synchronize()
    a = d3.planes(g, 0xFFF, stream=s)
    b = d3.planes(g, 0xFFF, stream=s.cuda_stream)
    adj = d3.planes_adjoint(a, 0xFFF, stream=s)
    s.synchronize()
    assert np.array_equal(a.cpu().numpy(), ref) and np.array_equal(b.cpu().numpy(), ref)
    assert torch.equal(adj, d3.planes_adjoint(a, 0xFFF))
