"""The parallel full-size comparison helper (tests/oracle_pool.py) catches single-element
errors, both for integers (exact) and for floats (T1 gate)."""
import numpy as np

import oracle
import oracle_pool
import synth


def test_pool_integer_exact_and_detects_one_error(tmp_path):
    cubes = synth.uniform_cube(8, 31, np.uint8, batch=2)
    ref = np.stack([oracle.drt_planes(c, 0x0F3) for c in cubes]).astype(np.int32)
    assert oracle_pool.compare_all(tmp_path, cubes, ref, 0x0F3, procs=2) == []
    ref[1, 3, 2, 5, 17] += 1
    assert oracle_pool.compare_all(tmp_path, cubes, ref, 0x0F3, procs=2) == [(1, 3, 5, 1)]


def test_pool_int32_wrap_and_djt(tmp_path):
    cubes = np.full((1, 4, 4, 4), 2 ** 30, np.int32)
    ref = oracle.djt_lines(cubes[0].astype(np.int64), 0x003)[None]
    wrapped = (((ref + 2 ** 31) % 2 ** 32) - 2 ** 31).astype(np.int32)
    assert oracle_pool.compare_all(tmp_path, cubes, wrapped, 0x003, "djt", procs=1) == []


def test_pool_float_gate(tmp_path):
    cubes = synth.normal_cube(8, 32, batch=1)
    ref = oracle.drt_planes(cubes[0].astype(np.float64), 0x001)[None].astype(np.float32)
    assert oracle_pool.compare_all(tmp_path, cubes, ref, 0x001, procs=1) == []
    ref[0, 0, 3, 3, 20] *= 1.001
    assert len(oracle_pool.compare_all(tmp_path, cubes, ref, 0x001, procs=1)) == 1
