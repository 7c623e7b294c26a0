"""Oracle pins for the multi-dodecant adjoints: the
orientation transpose is the inverse permutation, and the full 12-dodecant
operators satisfy <A f, c> = <f, A^T c> exactly (F8)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import tables


@pytest.mark.parametrize("row", tables.DRT_HEMISPHERE + tables.DJT_HEMISPHERE)
def test_unorient_inverts_orient(row):
    f = synth.uniform_cube(8, 71, np.int32, -50, 50)
    assert np.array_equal(oracle.unorient(oracle.orient(f, row), row), f)
    # and it is the transpose: <orient(f), h> = <f, unorient(h)>
    h = synth.uniform_cube(8, 72, np.int32, -50, 50)
    assert int((oracle.orient(f, row).astype(np.int64) * h).sum()) == int((f.astype(np.int64) * oracle.unorient(h, row)).sum())


@pytest.mark.parametrize("N", [4, 8])
def test_drt_planes_adjoint_identity(N):
    f = synth.uniform_cube(N, 80 + N, np.int32, -20, 20)
    c = synth.uniform_cube(N, 81 + N, np.int32, -20, 20, batch=36).reshape(12, N, N, 3 * N)
    lhs = int((oracle.drt_planes(f, 0xFFF).astype(np.int64) * c).sum())
    rhs = oracle.drt_planes_adjoint(c, 0xFFF)
    assert np.all(rhs == np.round(rhs))
    assert lhs == int((f.astype(np.int64) * rhs.astype(np.int64)).sum())


@pytest.mark.parametrize("N", [4, 8])
def test_djt_lines_adjoint_identity(N):
    f = synth.uniform_cube(N, 90 + N, np.int32, -20, 20)
    c = synth.uniform_cube(N, 91 + N, np.int32, -20, 20, batch=12 * 4 * N).reshape(12, N, N, 2 * N, 2 * N)
    lhs = int((oracle.djt_lines(f, 0xFFF).astype(np.int64) * c).sum())
    rhs = oracle.djt_lines_adjoint(c, 0xFFF)
    assert lhs == int((f.astype(np.int64) * rhs.astype(np.int64)).sum())
