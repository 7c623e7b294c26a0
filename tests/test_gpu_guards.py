"""Out-of-bounds and uninitialised-memory checks without compute-sanitizer (closed on this GPU
pool): every buffer a call touches sits between guard bands, and every buffer it
writes starts out poisoned.

- guard bands (4 KiB each side, a fixed non-zero byte pattern) around the cube / coefficients,
  the output and the workspace: a write past either end changes a guard (checked byte for
  byte); a read past the end of an input adds the non-zero pattern into a sum, which the
  comparison with the oracle catches;
- poison: output and workspace are filled with 0xFF bytes (int32 -1, fp32 NaN) before the
  call, so an output element the kernels never write, or a workspace element read before it
  is written, shows up as a mismatch (or a NaN) against the oracle.

Covers every entry point (forward DRT / DJT over the pass plans, the on-chip N = 32 kernel,
the mosaic, both adjoints, the inverse, the applications) at small N, every input dtype.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import apps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2501_13664_b200 as d3  # noqa: E402

G = 4096            # guard bytes per side (keeps 256-byte alignment of the payload)
PAT = 0xA5


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d3.lib()
    yield


class Guarded:
    """A device tensor of `shape`/`dtype` between two guard bands of one allocation."""

    def __init__(self, shape, dtype, fill=None, poison=True):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.nbytes = n
        self.raw = torch.full((G + ((n + 255) // 256) * 256 + G,), PAT, dtype=torch.uint8, device="cuda")
        body = self.raw[G:G + n]
        if fill is not None:
            body.copy_(torch.as_tensor(np.ascontiguousarray(fill)).reshape(-1).view(torch.uint8).cuda())
        elif poison:
            body.fill_(0xFF)
        self.t = body.view(dtype).view(shape)

    def intact(self):
        torch.cuda.synchronize()
        lo, hi = self.raw[:G], self.raw[G + self.nbytes:]
        return bool((lo == PAT).all()) and bool((hi == PAT).all())


def _wrap32(x):
    return ((np.asarray(x).astype(np.int64) + 2 ** 31) % 2 ** 32) - 2 ** 31


def _cube(N, dt, seed, batch=1):
    if dt == np.float32:
        return synth.normal_cube(N, seed, batch=batch)
    lo, hi = (0, 255) if dt == np.uint8 else (-100, 100)
    return synth.uniform_cube(N, seed, dt, lo, hi, batch=batch)


def _tdt(dt):
    return {np.uint8: torch.uint8, np.int32: torch.int32, np.float32: torch.float32}[dt]


def _close(got, ref, refabs=None):
    if got.dtype == np.float32:
        return bool(np.all(np.abs(got.astype(np.float64) - ref) <= 1e-5 * refabs))
    return np.array_equal(got.astype(np.int64), _wrap32(ref))


def _run_transform(kind, N, dt, mask, layout=d3.DRT3D_LAYOUT_STACKED, batch=1):
    f = _cube(N, dt, 40 + N + mask, batch=batch)
    cube = Guarded(f.shape, _tdt(dt), fill=f)
    odt = torch.float32 if dt == np.float32 else torch.int32
    K = bin(mask).count("1")
    o = d3.make_opts(batch=batch, in_dtype=d3._dtype_code(cube.t), out_dtype=d3.DRT3D_F32 if dt == np.float32
                     else d3.DRT3D_I32, layout=layout)
    if kind == "drt":
        shape = (batch, K, N, N, 3 * N) if layout == d3.DRT3D_LAYOUT_STACKED else (batch, 4 * N, 4 * N, 3 * N - 2)
        wsb = d3.drt3d_planes_workspace_size(N, mask, o)
    else:
        shape = (batch, K, N, N, 2 * N, 2 * N)
        wsb = d3.djt3d_lines_workspace_size(N, mask, o)
    out = Guarded(shape, odt)
    ws = Guarded((max(wsb, 256),), torch.uint8)
    fn = d3.planes if kind == "drt" else d3.lines
    kw = {"layout": layout} if kind == "drt" else {}
    fn(cube.t, mask, out=out.t, workspace=ws.t, **kw)
    assert cube.intact() and out.intact() and ws.intact(), (kind, N, dt, mask)
    got = out.t.cpu().numpy()
    for b in range(batch):
        x = f[b].astype(np.float64) if dt == np.float32 else f[b]
        if kind == "drt":
            ref = oracle.drt_planes(x, mask)
            refabs = oracle.drt_planes(np.abs(x), mask) if dt == np.float32 else None
            if layout == d3.DRT3D_LAYOUT_MOSAIC:
                ref = oracle.mosaic(ref)
                refabs = oracle.mosaic(refabs) if refabs is not None else None
        else:
            ref = oracle.djt_lines(x, mask)
            refabs = oracle.djt_lines(np.abs(x), mask) if dt == np.float32 else None
        assert _close(got[b], ref, refabs), (kind, N, dt, mask, b)


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("dt", [np.uint8, np.int32, np.float32])
def test_drt_guards(N, dt):
    _run_transform("drt", N, dt, 0xFFF if N <= 32 else 0x861, batch=2 if N <= 16 else 1)


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("dt", [np.uint8, np.int32, np.float32])
def test_djt_guards(N, dt):
    _run_transform("djt", N, dt, 0xFFF if N <= 16 else 0x011)


@pytest.mark.parametrize("N", [4, 32])
def test_mosaic_guards(N):
    _run_transform("drt", N, np.uint8, 0xFFF, layout=d3.DRT3D_LAYOUT_MOSAIC)


@pytest.mark.parametrize("kind,N", [("drt", 4), ("drt", 16), ("drt", 32), ("drt", 64), ("djt", 4), ("djt", 16)])
@pytest.mark.parametrize("dt", [np.int32, np.float32])
def test_adjoint_guards(kind, N, dt):
    mask = 0xFFF if N <= 16 else 0x0C1
    K = bin(mask).count("1")
    shape = (1, K, N, N, 3 * N) if kind == "drt" else (1, K, N, N, 2 * N, 2 * N)
    n = int(np.prod(shape))
    rng = np.random.default_rng(N + K)
    c = (rng.standard_normal(n).astype(np.float32) if dt == np.float32 else
         rng.integers(-100, 100, n).astype(np.int32)).reshape(shape)
    coef = Guarded(shape, _tdt(dt), fill=c)
    cube = Guarded((1, N, N, N), _tdt(dt))
    wsb = ctypes_ws(kind, N, mask)
    ws = Guarded((max(wsb, 256),), torch.uint8)
    fn = d3.planes_adjoint if kind == "drt" else d3.lines_adjoint
    fn(coef.t, mask, cube=cube.t, workspace=ws.t)
    assert coef.intact() and cube.intact() and ws.intact()
    refn = oracle.drt_planes_adjoint if kind == "drt" else oracle.djt_lines_adjoint
    ref = refn(c[0].astype(np.float64), mask)
    got = cube.t.cpu().numpy()[0]
    if dt == np.float32:
        scale = refn(np.abs(c[0]).astype(np.float64), mask)
        assert np.all(np.abs(got - ref) <= 1e-5 * scale)
    else:
        assert np.array_equal(got.astype(np.int64), _wrap32(np.round(ref)))


def ctypes_ws(kind, N, mask):
    import ctypes
    b = ctypes.c_size_t(0)
    o = d3.make_opts()
    fn = d3.lib().drt3d_planes_adjoint_workspace_size if kind == "drt" else d3.lib().djt3d_lines_adjoint_workspace_size
    assert fn(N, mask, ctypes.byref(o), ctypes.byref(b)) == d3.DRT3D_OK
    return b.value


def test_invert_and_apps_guards():
    import ctypes
    N = 16
    f = synth.normal_cube(N, 9)
    b = oracle.drt_planes(f.astype(np.float64)).astype(np.float32)
    coef = Guarded(b.shape, torch.float32, fill=b)
    x = Guarded((N, N, N), torch.float32)
    o = d3.make_opts(in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    sz = ctypes.c_size_t(0)
    assert d3.lib().drt3d_planes_invert_workspace_size(N, 2, 0xFFF, ctypes.byref(o), ctypes.byref(sz)) == 0
    ws = Guarded((sz.value,), torch.uint8)
    xs, rn = d3.planes_invert(coef.t, 3, cube=x.t, workspace=ws.t)
    assert coef.intact() and x.intact() and ws.intact()
    assert bool(torch.isfinite(xs).all()) and bool(torch.isfinite(rn).all())
    # applications on int32 coefficients
    ci = oracle.drt_planes(synth.uniform_cube(N, 10, np.uint8), 0xFFF).astype(np.int32)
    c = Guarded(ci.shape, torch.int32, fill=ci)
    aw = Guarded((max(d3.lib().drt3d_apps_workspace_size(), 256),), torch.uint8)
    kept = Guarded(ci.shape, torch.int32)
    d3.coef_threshold(c.t, 1, 2, out=kept.t, workspace=aw.t)
    assert c.intact() and kept.intact() and aw.intact()
    assert np.array_equal(kept.t.cpu().numpy().astype(np.int64), apps.threshold(ci, 1, 2))
    flags, am = d3.detect_planes(c.t, 0xFFF, 1, 3, 1, 10, workspace=aw.t)
    assert c.intact() and aw.intact()
    rf, ra = apps.detect_planes(ci, 0xFFF, 1, 3, 1, 10)
    assert int(am.item()) == ra and np.array_equal(flags.cpu().numpy(), rf)
    sel = Guarded(ci.shape, torch.int32)
    d3.coef_select(c.t, flags, out=sel.t)
    assert sel.intact()
    assert np.array_equal(sel.t.cpu().numpy(), np.where(rf == 1, ci, 0))
