"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only entry points (tables, sizes, validation)
behave as documented.  No kernel is launched here."""
import ctypes
import os
import re

import pytest

import paper_2501_13664_b200 as d3
from oracle import tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2501_13664_b200 import build
    build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "drt3d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b((?:drt3d|djt3d)_[a-z_]+)\s*\(", src))


def test_exports_every_declared_symbol():
    names = _declared()
    assert names == set(d3.C_FUNCTIONS)
    L = d3.lib()
    for n in names:
        assert hasattr(L, n), n


def test_orientation_tables_match_oracle_copy():
    # the library and the oracle each hold their own copy (R6-R8)
    assert d3.orientation_table(d3.DRT3D_TABLE_HEMISPHERE, 0) == tables.DRT_HEMISPHERE
    assert d3.orientation_table(d3.DRT3D_TABLE_HEMISPHERE, 1) == tables.DJT_HEMISPHERE
    assert d3.orientation_table(d3.DRT3D_TABLE_PRINTED, 0) == tables.DRT_PRINTED
    assert d3.orientation_table(d3.DRT3D_TABLE_PRINTED, 1) == tables.DRT_PRINTED
    assert d3.orientation_table(d3.DRT3D_TABLE_SHARED, 0) == tables.SHARED


def test_out_elems():
    o = d3.make_opts()
    assert d3.drt3d_planes_out_elems(256, 0xFFF, o) == 12 * 256 * 256 * 768
    assert d3.drt3d_planes_out_elems(16, 0x1, o) == 16 * 16 * 48
    o5 = d3.make_opts(batch=256, in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    assert d3.drt3d_planes_out_elems(32, 0xFFF, o5) == 256 * 12 * 32 * 32 * 96
    om = d3.make_opts(layout=d3.DRT3D_LAYOUT_MOSAIC)
    assert d3.drt3d_planes_out_elems(8, 0xFFF, om) == 32 * 32 * 22
    assert d3.djt3d_lines_out_elems(64, 0x1, o) == 64 * 64 * 128 * 128
    assert d3.drt3d_planes_out_elems(12, 0x1, o) == 0        # invalid N


def test_workspace_sizes():
    o = d3.make_opts()
    # N = 16 stacked: every stage of an instance in one CTA (k_sep16.cu), no workspace
    assert d3.drt3d_planes_workspace_size(16, 0x1, o) == 0
    assert d3.drt3d_planes_workspace_size(16, 0xFFF, d3.make_opts(batch=64)) == 0
    # N = 16 mosaic: the pass kernels; 12 instances run two radix-4 passes (DESIGN.md §5 "Pass plan"):
    # stage-2 rows N^2 x pitch round8(3N - base) u16, base = floor16(2N - 2 (2^2 - 1) - 7) = 16 -> 32
    om = d3.make_opts(layout=d3.DRT3D_LAYOUT_MOSAIC)
    assert d3.drt3d_planes_workspace_size(16, 0xFFF, om) == 12 * 16 * 16 * 32 * 2
    assert d3.drt3d_planes_workspace_size(32, 0xFFF, o) == 0                  # u8 N = 32: on-chip kernel
    ws = d3.drt3d_planes_workspace_size(256, 0xFFF, o)
    # N=256, 12 dodecants in one chunk: 12 stage-4 buffers of N^2 rows x u16, pitch
    # round16(3N - base) with base = floor16(2N - 2 (2^4 - 1) - 7) = 464 -> 304
    assert ws == 12 * 256 * 256 * 304 * 2
    assert ws <= 512 << 20
    assert d3.djt3d_lines_workspace_size(64, 0x1, o) > 0


@pytest.mark.parametrize("N,mask,kw,err", [
    (12, 0x1, {}, d3.DRT3D_ERR_INVALID_ARG),
    (1, 0x1, {}, d3.DRT3D_ERR_INVALID_ARG),
    (2048, 0x1, {}, d3.DRT3D_ERR_INVALID_ARG),
    (16, 0x0, {}, d3.DRT3D_ERR_INVALID_ARG),
    (16, 0x1000, {}, d3.DRT3D_ERR_INVALID_ARG),
    (16, 0x1, dict(in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_F32), d3.DRT3D_ERR_INVALID_ARG),
    (16, 0x1, dict(batch=0), d3.DRT3D_ERR_INVALID_ARG),
    (16, 0x1, dict(layout=d3.DRT3D_LAYOUT_MOSAIC), d3.DRT3D_ERR_INVALID_ARG),   # mosaic needs 0xFFF
    (16, 0x1, dict(table=7), d3.DRT3D_ERR_INVALID_ARG),
])
def test_validation_rejects_before_launch(N, mask, kw, err):
    o = d3.make_opts(**kw)
    # bogus device pointers: validation must fail before anything touches them
    assert d3.drt3d_planes(16, N, mask, 1 << 40, o, None, 0, None) == err


def test_null_and_workspace_errors():
    o = d3.make_opts()
    assert d3.drt3d_planes(None, 16, 1, 1 << 40, o, None, 0, None) == d3.DRT3D_ERR_INVALID_ARG
    assert d3.drt3d_planes(16, 16, 1, None, o, None, 0, None) == d3.DRT3D_ERR_INVALID_ARG
    assert d3.drt3d_planes(16, 256, 1, 1 << 40, o, None, 0, None) == d3.DRT3D_ERR_WORKSPACE
    assert d3.djt3d_lines(16, 64, 1, 1 << 40, o, None, 0, None) == d3.DRT3D_ERR_WORKSPACE
    assert d3.djt3d_lines(16, 64, 1, (1 << 40) + 4, o, None, 0, None) == d3.DRT3D_ERR_INVALID_ARG  # misaligned out
    assert d3.status_string(d3.DRT3D_ERR_CUDA) == "DRT3D_ERR_CUDA"


def _size(fn, *args):
    b = ctypes.c_size_t(0)
    s = fn(*args, ctypes.byref(b))
    return s, b.value


def test_adjoint_invert_apps_sizes():
    L = d3.lib()
    o32 = d3.make_opts(in_dtype=d3.DRT3D_I32, out_dtype=d3.DRT3D_I32)
    s, a256 = _size(L.drt3d_planes_adjoint_workspace_size, 256, 0xFFF, ctypes.byref(o32))
    assert s == d3.DRT3D_OK and 1 << 30 < a256 < 4 << 30               # 12 dodecants per chunk at N = 256
    s, a1 = _size(L.drt3d_planes_adjoint_workspace_size, 256, 0x001, ctypes.byref(o32))
    assert s == d3.DRT3D_OK and a1 < a256
    s, j64 = _size(L.djt3d_lines_adjoint_workspace_size, 64, 0x001, ctypes.byref(o32))
    assert s == d3.DRT3D_OK and j64 >= 2 * 64 * 64 * 128 * 128 * 4
    of = d3.make_opts(in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    s, i2 = _size(L.drt3d_planes_invert_workspace_size, 64, 2, 0xFFF, ctypes.byref(of))
    s2, i64 = _size(L.drt3d_planes_invert_workspace_size, 64, 64, 0xFFF, ctypes.byref(of))
    assert s == s2 == d3.DRT3D_OK and i64 < i2                         # single grid needs fewer levels
    assert L.drt3d_apps_workspace_size() >= 256


def test_adjoint_invert_apps_validation():
    """Every rejection happens on the host before any launch (bogus device pointers)."""
    L = d3.lib()
    bogus, mis = 1 << 40, (1 << 40) + 4
    o32 = d3.make_opts(in_dtype=d3.DRT3D_I32, out_dtype=d3.DRT3D_I32)
    po = ctypes.byref(o32)
    E, W = d3.DRT3D_ERR_INVALID_ARG, d3.DRT3D_ERR_WORKSPACE
    assert L.drt3d_planes_adjoint(bogus, 12, 0xFFF, bogus, po, bogus, 1 << 40, None) == E     # N not 2^k
    assert L.drt3d_planes_adjoint(bogus, 16, 0x0, bogus, po, bogus, 1 << 40, None) == E       # empty mask
    assert L.drt3d_planes_adjoint(None, 16, 0x1, bogus, po, bogus, 1 << 40, None) == E
    assert L.drt3d_planes_adjoint(mis, 16, 0x1, bogus, po, bogus, 1 << 40, None) == E         # misaligned coef
    assert L.drt3d_planes_adjoint(bogus, 16, 0x1, mis, po, bogus, 1 << 40, None) == E         # misaligned cube
    assert L.drt3d_planes_adjoint(bogus, 16, 0x1, bogus << 2, po, None, 0, None) == W
    assert L.drt3d_planes_adjoint(bogus, 16, 0x1, bogus << 2, po, bogus + 16, 1 << 40, None) == W   # ws alignment
    assert L.djt3d_lines_adjoint(bogus, 16, 0x1, bogus << 2, po, None, 0, None) == W
    u8 = d3.make_opts(in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_U8)
    assert L.drt3d_planes_adjoint(bogus, 16, 0x1, bogus << 2, ctypes.byref(u8), bogus, 1 << 40, None) == E
    of = d3.make_opts(in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    pf = ctypes.byref(of)
    assert L.drt3d_planes_invert(bogus, 16, 3, 0xFFF, 2, bogus, None, pf, bogus, 1 << 40, None) == E   # n_min not 2^k
    assert L.drt3d_planes_invert(bogus, 16, 32, 0xFFF, 2, bogus, None, pf, bogus, 1 << 40, None) == E  # n_min > N
    assert L.drt3d_planes_invert(bogus, 16, 2, 0xFFF, -1, bogus, None, pf, bogus, 1 << 40, None) == E  # iters < 0
    assert L.drt3d_planes_invert(mis, 16, 2, 0xFFF, 2, bogus, None, pf, bogus, 1 << 40, None) == E
    assert L.drt3d_planes_invert(bogus, 16, 2, 0xFFF, 2, bogus, None, ctypes.byref(o32), bogus, 1 << 40, None) == E
    assert L.drt3d_planes_invert(bogus, 16, 2, 0xFFF, 2, bogus, None, pf, None, 0, None) == W
    ob = d3.make_opts(in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32, batch=2)
    assert L.drt3d_planes_invert(bogus, 16, 2, 0xFFF, 2, bogus, None, ctypes.byref(ob), bogus, 1 << 40, None) == E
    ws = L.drt3d_apps_workspace_size()
    assert L.drt3d_coef_argmax(bogus, 0, bogus, bogus, ws, None) == E                         # empty array
    assert L.drt3d_coef_argmax(bogus, 10, bogus, bogus, ws - 1, None) == W
    assert L.drt3d_coef_threshold(bogus, 10, 1, 0, bogus, bogus, ws, None) == E                # den = 0
    assert L.drt3d_coef_threshold(bogus, 10, -1, 2, bogus, bogus, ws, None) == E               # num < 0
    assert L.drt3d_detect_planes(bogus, 12, 0xFFF, 1, 3, 1, 10, None, bogus, None, bogus, ws, None) == E
    assert L.drt3d_detect_planes(bogus, 16, 0xFFF, 1, 3, 1, 0, None, bogus, None, bogus, ws, None) == E
    assert L.drt3d_coef_select(bogus, None, 10, bogus, None) == E
