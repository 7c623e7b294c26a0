"""B200 (sm_100a) hot path of arXiv 2501.13664: 3D DRT of planes and 3D DJT of lines.

Thin Python binding over the C ABI in include/drt3d.h (libdrt3d.so, built in
tree by `python -m paper_2501_13664_b200.build`).  This module only marshals
arguments: every step of the transform runs in the CUDA kernels.  There is no
CPU fallback -- if the library is missing, every call raises.

Raw C-ABI mirrors keep the C names (drt3d_planes, djt3d_lines, ...); the
torch helpers `planes()` / `lines()` allocate outputs and workspace with
PyTorch (device memory and the current stream only) and call the C ABI.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("D3_LIB") or os.path.join(_HERE, "libdrt3d.so")

DRT3D_OK, DRT3D_ERR_INVALID_ARG, DRT3D_ERR_UNSUPPORTED, DRT3D_ERR_WORKSPACE, DRT3D_ERR_CUDA = range(5)
DRT3D_U8, DRT3D_I32, DRT3D_F32 = range(3)
DRT3D_LAYOUT_STACKED, DRT3D_LAYOUT_MOSAIC = range(2)
DRT3D_TABLE_HEMISPHERE, DRT3D_TABLE_PRINTED, DRT3D_TABLE_SHARED = range(3)

# names declared in include/drt3d.h
C_FUNCTIONS = ("drt3d_status_string", "drt3d_orientation_table", "drt3d_planes_out_elems",
               "drt3d_planes_workspace_size", "drt3d_planes", "djt3d_lines_out_elems",
               "djt3d_lines_workspace_size", "djt3d_lines", "drt3d_planes_host", "djt3d_lines_host",
               "drt3d_planes_adjoint_workspace_size", "drt3d_planes_adjoint",
               "djt3d_lines_adjoint_workspace_size", "djt3d_lines_adjoint",
               "drt3d_planes_invert_workspace_size", "drt3d_planes_invert",
               "drt3d_apps_workspace_size", "drt3d_coef_argmax", "drt3d_coef_threshold", "drt3d_detect_planes",
               "drt3d_coef_select")


class Drt3dError(RuntimeError):
    pass


class drt3d_opts(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int), ("in_dtype", ctypes.c_int), ("out_dtype", ctypes.c_int),
                ("layout", ctypes.c_int), ("table", ctypes.c_int),
                ("events", ctypes.c_void_p), ("max_events", ctypes.c_int),
                ("launches", ctypes.POINTER(ctypes.c_int)), ("launch_kind", ctypes.POINTER(ctypes.c_int))]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdrt3d.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise Drt3dError(f"{LIB_PATH} not found: build it with `python -m paper_2501_13664_b200.build` "
                         "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32
    po = ctypes.POINTER(drt3d_opts)
    L.drt3d_status_string.restype = ctypes.c_char_p
    L.drt3d_status_string.argtypes = [i32]
    L.drt3d_orientation_table.restype = i32
    L.drt3d_orientation_table.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_int8)]
    for t in ("drt3d_planes", "djt3d_lines"):
        f = getattr(L, t + "_out_elems")
        f.restype = sz
        f.argtypes = [i32, u32, po]
        f = getattr(L, t + "_workspace_size")
        f.restype = i32
        f.argtypes = [i32, u32, po, ctypes.POINTER(sz)]
        f = getattr(L, t)
        f.restype = i32
        f.argtypes = [vp, i32, u32, vp, po, vp, sz, vp]
        f = getattr(L, t + "_host")
        f.restype = i32
        f.argtypes = [vp, i32, u32, vp, po, vp, vp, vp, sz, vp]
        f = getattr(L, t + "_adjoint_workspace_size")
        f.restype = i32
        f.argtypes = [i32, u32, po, ctypes.POINTER(sz)]
        f = getattr(L, t + "_adjoint")
        f.restype = i32
        f.argtypes = [vp, i32, u32, vp, po, vp, sz, vp]
    L.drt3d_planes_invert_workspace_size.restype = i32
    L.drt3d_planes_invert_workspace_size.argtypes = [i32, i32, u32, po, ctypes.POINTER(sz)]
    L.drt3d_planes_invert.restype = i32
    L.drt3d_planes_invert.argtypes = [vp, i32, i32, u32, i32, vp, vp, po, vp, sz, vp]
    L.drt3d_apps_workspace_size.restype = sz
    L.drt3d_apps_workspace_size.argtypes = []
    L.drt3d_coef_argmax.restype = i32
    L.drt3d_coef_argmax.argtypes = [vp, sz, vp, vp, sz, vp]
    L.drt3d_coef_threshold.restype = i32
    L.drt3d_coef_threshold.argtypes = [vp, sz, i32, i32, vp, vp, sz, vp]
    L.drt3d_coef_select.restype = i32
    L.drt3d_coef_select.argtypes = [vp, vp, sz, vp, vp]
    L.drt3d_detect_planes.restype = i32
    L.drt3d_detect_planes.argtypes = [vp, i32, u32, i32, i32, i32, i32, po, vp, vp, vp, sz, vp]
    _lib = L
    return L


def status_string(s: int) -> str:
    return lib().drt3d_status_string(s).decode()


def _check(s: int, what: str):
    if s != DRT3D_OK:
        raise Drt3dError(f"{what}: {status_string(s)}")


def make_opts(batch=1, in_dtype=DRT3D_U8, out_dtype=DRT3D_I32, layout=DRT3D_LAYOUT_STACKED,
              table=DRT3D_TABLE_HEMISPHERE) -> drt3d_opts:
    return drt3d_opts(batch, in_dtype, out_dtype, layout, table, None, 0, None, None)


def orientation_table(table: int = DRT3D_TABLE_HEMISPHERE, transform: int = 0):
    rows = (ctypes.c_int8 * 36)()
    _check(lib().drt3d_orientation_table(table, transform, rows), "drt3d_orientation_table")
    return [tuple(rows[3 * k + j] for j in range(3)) for k in range(12)]


# ------------------------------------------------------------ raw C mirrors

def drt3d_planes_out_elems(N, mask, opts=None):
    return lib().drt3d_planes_out_elems(N, mask, ctypes.byref(opts) if opts else None)


def drt3d_planes_workspace_size(N, mask, opts=None):
    b = ctypes.c_size_t(0)
    _check(lib().drt3d_planes_workspace_size(N, mask, ctypes.byref(opts) if opts else None, ctypes.byref(b)),
           "drt3d_planes_workspace_size")
    return b.value


def drt3d_planes(cube_ptr, N, mask, out_ptr, opts, ws_ptr, ws_bytes, stream) -> int:
    return lib().drt3d_planes(cube_ptr, N, mask, out_ptr, ctypes.byref(opts) if opts else None,
                              ws_ptr, ws_bytes, stream)


def djt3d_lines_out_elems(N, mask, opts=None):
    return lib().djt3d_lines_out_elems(N, mask, ctypes.byref(opts) if opts else None)


def djt3d_lines_workspace_size(N, mask, opts=None):
    b = ctypes.c_size_t(0)
    _check(lib().djt3d_lines_workspace_size(N, mask, ctypes.byref(opts) if opts else None, ctypes.byref(b)),
           "djt3d_lines_workspace_size")
    return b.value


def djt3d_lines(cube_ptr, N, mask, out_ptr, opts, ws_ptr, ws_bytes, stream) -> int:
    return lib().djt3d_lines(cube_ptr, N, mask, out_ptr, ctypes.byref(opts) if opts else None,
                             ws_ptr, ws_bytes, stream)


def drt3d_planes_host(hcube_ptr, N, mask, hout_ptr, opts, dcube_ptr, dout_ptr, ws_ptr, ws_bytes, stream) -> int:
    return lib().drt3d_planes_host(hcube_ptr, N, mask, hout_ptr, ctypes.byref(opts) if opts else None,
                                   dcube_ptr, dout_ptr, ws_ptr, ws_bytes, stream)


def djt3d_lines_host(hcube_ptr, N, mask, hout_ptr, opts, dcube_ptr, dout_ptr, ws_ptr, ws_bytes, stream) -> int:
    return lib().djt3d_lines_host(hcube_ptr, N, mask, hout_ptr, ctypes.byref(opts) if opts else None,
                                  dcube_ptr, dout_ptr, ws_ptr, ws_bytes, stream)


# ------------------------------------------------------------ torch helpers
# Every helper allocates its temporaries (contiguous copies, output, workspace) on the stream the
# call is enqueued on, so the caching allocator never hands them to other work while the kernels
# may still use them; caller-supplied buffers are checked (shape, dtype, contiguity, device) and
# the C ABI is told their real sizes.

def _dtype_code(t):
    import torch
    try:
        return {torch.uint8: DRT3D_U8, torch.int32: DRT3D_I32, torch.float32: DRT3D_F32}[t.dtype]
    except KeyError:
        raise Drt3dError(f"unsupported cube dtype {t.dtype} (uint8, int32 or float32)") from None


def _stream(stream, device):
    """torch.cuda.Stream for `stream`: None = the current stream, a torch stream, or a raw
    cudaStream_t handle (wrapped as an external stream)."""
    import torch
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream), device=device)


def _popcount(mask: int) -> int:
    if not 0 < mask < (1 << 12):
        raise Drt3dError(f"dodecant mask {mask:#x} outside [1, 2^12)")
    return bin(mask).count("1")


def _user_tensor(t, shape, dtype, device, what):
    if (tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or not t.is_cuda
            or t.device != device):
        raise Drt3dError(f"{what} must be a contiguous {dtype} CUDA tensor of shape {tuple(shape)} on {device}, "
                         f"got {t.dtype} {tuple(t.shape)} on {t.device}")
    return t


def _workspace(workspace, need, device):
    """(tensor or None, size in bytes actually available)."""
    import torch
    if workspace is None:
        if not need:
            return None, 0
        workspace = torch.empty(need, dtype=torch.uint8, device=device)
    elif not workspace.is_cuda or workspace.device != device or not workspace.is_contiguous():
        raise Drt3dError("workspace must be a contiguous CUDA tensor on the cube's device")
    return workspace, workspace.numel() * workspace.element_size()


def _opts_from(o, opts):
    if opts is not None:
        o.events, o.max_events, o.launches, o.launch_kind = opts.events, opts.max_events, opts.launches, opts.launch_kind


def _prep(cube, layout, table):
    import torch
    if not isinstance(cube, torch.Tensor) or not cube.is_cuda:
        raise Drt3dError("cube must be a CUDA tensor (use the *_host C entry points for host data)")
    c = cube.contiguous()
    if c.dim() == 3:
        c = c.unsqueeze(0)
    if c.dim() != 4 or not (c.shape[1] == c.shape[2] == c.shape[3]):
        raise Drt3dError("cube must be [N,N,N] or [B,N,N,N]")
    dt = _dtype_code(c)
    odt = DRT3D_F32 if dt == DRT3D_F32 else DRT3D_I32
    o = make_opts(batch=c.shape[0], in_dtype=dt, out_dtype=odt, layout=layout, table=table)
    return c, o, (torch.float32 if odt == DRT3D_F32 else torch.int32)


def _transform(kind, cube, mask, layout, table, out, workspace, stream, opts):
    import torch
    st = _stream(stream, cube.device)
    with torch.cuda.stream(st):
        c, o, odt = _prep(cube, layout, table)
        _opts_from(o, opts)
        B, N = c.shape[0], c.shape[1]
        K = _popcount(mask)
        if kind == "drt":
            shape = (B, K, N, N, 3 * N) if layout == DRT3D_LAYOUT_STACKED else (B, 4 * N, 4 * N, 3 * N - 2)
        else:
            shape = (B, K, N, N, 2 * N, 2 * N)
        if out is None:
            out = torch.empty(shape, dtype=odt, device=c.device)
        else:
            # a 3-D cube may come with an output without the batch dimension
            user_shape = shape[1:] if cube.dim() == 3 and tuple(out.shape) == shape[1:] else shape
            out = _user_tensor(out, user_shape, odt, c.device, "out").view(shape)
        need = (drt3d_planes_workspace_size if kind == "drt" else djt3d_lines_workspace_size)(N, mask, o)
        ws, ws_bytes = _workspace(workspace, need, c.device)
        fn = drt3d_planes if kind == "drt" else djt3d_lines
        s = fn(c.data_ptr(), N, mask, out.data_ptr(), o, ws.data_ptr() if ws is not None else None, ws_bytes,
               st.cuda_stream)
    _check(s, "drt3d_planes" if kind == "drt" else "djt3d_lines")
    return out if cube.dim() == 4 else out[0]


def planes(cube, mask: int = 0xFFF, layout: int = DRT3D_LAYOUT_STACKED, table: int = DRT3D_TABLE_HEMISPHERE,
           out=None, workspace=None, stream=None, opts: drt3d_opts | None = None):
    """3D DRT of planes of a CUDA cube [B,N,N,N] (or [N,N,N]).

    Returns out [B, K, N, N, 3N] (STACKED) or [B, 4N, 4N, 3N-2] (MOSAIC).  `stream`: None (the
    current stream), a torch.cuda.Stream or a raw cudaStream_t handle."""
    return _transform("drt", cube, mask, layout, table, out, workspace, stream, opts)


def lines(cube, mask: int = 0x001, table: int = DRT3D_TABLE_HEMISPHERE, out=None, workspace=None, stream=None,
          opts: drt3d_opts | None = None):
    """3D DJT of lines of a CUDA cube: out [B, K, N, N, 2N, 2N]."""
    return _transform("djt", cube, mask, DRT3D_LAYOUT_STACKED, table, out, workspace, stream, opts)


# ------------------------------------------------------------ adjoints (F-1)

def _adjoint(kind, coef, mask, table, cube, workspace, stream, opts):
    import torch
    if not isinstance(coef, torch.Tensor) or not coef.is_cuda:
        raise Drt3dError("coef must be a CUDA tensor")
    st = _stream(stream, coef.device)
    nd = 5 if kind == "drt" else 6
    with torch.cuda.stream(st):
        c = coef.contiguous()
        if c.dim() == nd - 1:
            c = c.unsqueeze(0)
        if c.dim() != nd:
            raise Drt3dError("coef must be the stacked forward layout")
        B, K, N = c.shape[0], c.shape[1], c.shape[2]
        tail = (N, N, 3 * N) if kind == "drt" else (N, N, 2 * N, 2 * N)
        if K != _popcount(mask) or tuple(c.shape[2:]) != tail:
            raise Drt3dError(f"coef shape {tuple(coef.shape)} does not match mask {mask:#x} "
                             f"(expected [B, {_popcount(mask)}, {', '.join(map(str, tail))}])")
        if c.dtype not in (torch.int32, torch.float32):
            raise Drt3dError("coef must be int32 or float32")
        dt = DRT3D_I32 if c.dtype == torch.int32 else DRT3D_F32
        o = make_opts(batch=B, in_dtype=dt, out_dtype=dt, table=table)
        _opts_from(o, opts)
        if cube is None:
            cube = torch.empty((B, N, N, N), dtype=c.dtype, device=c.device)
            res = cube
        else:
            user_shape = (N, N, N) if coef.dim() == nd - 1 and cube.dim() == 3 else (B, N, N, N)
            res = _user_tensor(cube, user_shape, c.dtype, c.device, "cube")
            cube = res.view(B, N, N, N)
        L = lib()
        b = ctypes.c_size_t(0)
        _check(getattr(L, f"{'drt3d_planes' if kind == 'drt' else 'djt3d_lines'}_adjoint_workspace_size")(
            N, mask, ctypes.byref(o), ctypes.byref(b)), "adjoint_workspace_size")
        ws, ws_bytes = _workspace(workspace, max(b.value, 256), c.device)
        fn = L.drt3d_planes_adjoint if kind == "drt" else L.djt3d_lines_adjoint
        s = fn(c.data_ptr(), N, mask, cube.data_ptr(), ctypes.byref(o), ws.data_ptr(), ws_bytes, st.cuda_stream)
    _check(s, f"{kind} adjoint")
    if res is not cube:
        return res
    return cube if coef.dim() == nd else cube[0]


def planes_adjoint(coef, mask: int = 0xFFF, table: int = DRT3D_TABLE_HEMISPHERE, cube=None, workspace=None,
                   stream=None, opts: drt3d_opts | None = None):
    """Backprojection of stacked DRT coefficients [B,K,N,N,3N] (int32 / float32) -> [B,N,N,N]."""
    return _adjoint("drt", coef, mask, table, cube, workspace, stream, opts)


def lines_adjoint(coef, mask: int = 0x001, table: int = DRT3D_TABLE_HEMISPHERE, cube=None, workspace=None,
                  stream=None, opts: drt3d_opts | None = None):
    """Backprojection of stacked DJT coefficients [B,K,N,N,2N,2N] (int32 / float32) -> [B,N,N,N]."""
    return _adjoint("djt", coef, mask, table, cube, workspace, stream, opts)


# ------------------------------------------------------- iterative inverse (F-3)

def planes_invert(coef, iters: int, mask: int = 0xFFF, n_min: int = 2, table: int = DRT3D_TABLE_HEMISPHERE,
                  cube=None, workspace=None, stream=None, opts: drt3d_opts | None = None):
    """Iterative inverse of stacked fp32 DRT coefficients [K,N,N,3N] -> (x [N,N,N] fp32,
    rnorm [iters+1] fp64 residual norms ||b - A x_k||) by drt3d_planes_invert (F-3);
    n_min = coarsest multigrid size (n_min = N: single-grid iteration)."""
    import torch
    if not isinstance(coef, torch.Tensor) or not coef.is_cuda or coef.dtype != torch.float32 or coef.dim() != 4:
        raise Drt3dError("coef must be a CUDA float32 tensor [K,N,N,3N]")
    N = coef.shape[1]
    if coef.shape[0] != _popcount(mask) or tuple(coef.shape[2:]) != (N, 3 * N):
        raise Drt3dError(f"coef shape {tuple(coef.shape)} does not match mask {mask:#x} "
                         f"(expected [{_popcount(mask)}, {N}, {N}, {3 * N}])")
    st = _stream(stream, coef.device)
    with torch.cuda.stream(st):
        c = coef.contiguous()
        o = make_opts(batch=1, in_dtype=DRT3D_F32, out_dtype=DRT3D_F32, table=table)
        if opts is not None:
            o.launches = opts.launches
        if cube is None:
            cube = torch.empty((N, N, N), dtype=torch.float32, device=c.device)
        else:
            _user_tensor(cube, (N, N, N), torch.float32, c.device, "cube")
        rnorm = torch.empty(iters + 1, dtype=torch.float64, device=c.device)
        L = lib()
        b = ctypes.c_size_t(0)
        _check(L.drt3d_planes_invert_workspace_size(N, n_min, mask, ctypes.byref(o), ctypes.byref(b)),
               "invert_workspace_size")
        ws, ws_bytes = _workspace(workspace, max(b.value, 256), c.device)
        s = L.drt3d_planes_invert(c.data_ptr(), N, n_min, mask, iters, cube.data_ptr(), rnorm.data_ptr(),
                                  ctypes.byref(o), ws.data_ptr(), ws_bytes, st.cuda_stream)
    _check(s, "planes invert")
    return cube, rnorm


# ------------------------------------------------------------ applications (F-4)

def _apps_ws(workspace, device):
    return _workspace(workspace, max(lib().drt3d_apps_workspace_size(), 256), device)


def _int32_coef(coef):
    import torch
    if not isinstance(coef, torch.Tensor) or not coef.is_cuda or coef.dtype != torch.int32:
        raise Drt3dError("coef must be a CUDA int32 tensor")
    return coef.contiguous()


def coef_argmax(coef, workspace=None, stream=None) -> int:
    """Flat index of the largest int32 coefficient (smallest index among ties); synchronises."""
    import torch
    st = _stream(stream, coef.device)
    with torch.cuda.stream(st):
        c = _int32_coef(coef)
        ws, ws_bytes = _apps_ws(workspace, c.device)
        idx = torch.empty(1, dtype=torch.int64, device=c.device)
        s = lib().drt3d_coef_argmax(c.data_ptr(), c.numel(), idx.data_ptr(), ws.data_ptr(), ws_bytes, st.cuda_stream)
        _check(s, "coef_argmax")
        return int(idx.item())


def coef_threshold(coef, num: int, den: int, out=None, workspace=None, stream=None):
    """Keep c where c * den >= num * max(c), else 0 (int32, exact)."""
    import torch
    st = _stream(stream, coef.device)
    with torch.cuda.stream(st):
        c = _int32_coef(coef)
        out = torch.empty_like(c) if out is None else _user_tensor(out, c.shape, torch.int32, c.device, "out")
        ws, ws_bytes = _apps_ws(workspace, c.device)
        s = lib().drt3d_coef_threshold(c.data_ptr(), c.numel(), num, den, out.data_ptr(), ws.data_ptr(), ws_bytes,
                                       st.cuda_stream)
    _check(s, "coef_threshold")
    return out


def detect_planes(coef, mask: int, num: int, den: int, onum: int, oden: int, table: int = DRT3D_TABLE_HEMISPHERE,
                  workspace=None, stream=None):
    """Plane detection on stacked int32 DRT coefficients [K,N,N,3N] -> (flags uint8 [K,N,N,3N],
    argmax flat index tensor [1] int64), F-4."""
    import torch
    c0 = _int32_coef(coef)
    if c0.dim() != 4 or c0.shape[0] != _popcount(mask) or tuple(c0.shape[2:]) != (c0.shape[1], 3 * c0.shape[1]):
        raise Drt3dError(f"coef must be [{_popcount(mask)}, N, N, 3N] for mask {mask:#x}, got {tuple(coef.shape)}")
    st = _stream(stream, coef.device)
    with torch.cuda.stream(st):
        c = coef.contiguous()
        N = c.shape[1]
        flags = torch.empty(c.shape, dtype=torch.uint8, device=c.device)
        am = torch.empty(1, dtype=torch.int64, device=c.device)
        o = make_opts(table=table)
        ws, ws_bytes = _apps_ws(workspace, c.device)
        s = lib().drt3d_detect_planes(c.data_ptr(), N, mask, num, den, onum, oden, ctypes.byref(o), flags.data_ptr(),
                                      am.data_ptr(), ws.data_ptr(), ws_bytes, st.cuda_stream)
    _check(s, "detect_planes")
    return flags, am


def coef_select(coef, flags, out=None, stream=None):
    """Keep the flagged int32 coefficients (flags uint8 of the same shape), zero the rest."""
    import torch
    st = _stream(stream, coef.device)
    with torch.cuda.stream(st):
        c = _int32_coef(coef)
        f = flags.contiguous()
        if not f.is_cuda or f.dtype != torch.uint8 or f.shape != c.shape or f.device != c.device:
            raise Drt3dError("coef: CUDA int32; flags: uint8 of the same shape on the same device")
        out = torch.empty_like(c) if out is None else _user_tensor(out, c.shape, torch.int32, c.device, "out")
        s = lib().drt3d_coef_select(c.data_ptr(), f.data_ptr(), c.numel(), out.data_ptr(), st.cuda_stream)
    _check(s, "coef_select")
    return out
