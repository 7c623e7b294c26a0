"""Full-size element-wise parity against the oracle in parallel processes (test infrastructure).

The GPU result and the input cubes are saved to .npy files; spawned workers (numpy + oracle
only, no CUDA) each recompute the oracle for some (cube, dodecant) instances and compare every
element with the GPU slice, read through a memory map.  Integer results must match exactly
(int32 output = the int64 oracle sum mod 2^32); float results pass the T1 gate of DESIGN.md:
|gpu - ref64| <= 1e-5 * sum|terms| per element (sum|terms| = the fp64 transform of |f|) and
elements with empty support exactly 0.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np


def _check(args):
    cube_path, out_path, transform, table, items = args
    import oracle  # noqa: WPS433 (worker-side import: spawned processes start clean)
    from oracle import tables

    cubes = np.load(cube_path, mmap_mode="r")
    out = np.load(out_path, mmap_mode="r")
    rows = tables.table(table, transform)
    fn = oracle.drt_alg1 if transform == "drt" else oracle.djt_alg3
    bad = []
    for b, j, k in items:
        f = np.asarray(cubes[b])
        g = np.asarray(out[b, j])
        if f.dtype.kind == "f":
            ref = fn(oracle.orient(f.astype(np.float64), rows[k]))
            refabs = fn(oracle.orient(np.abs(f).astype(np.float64), rows[k]))
            err = np.abs(g.astype(np.float64) - ref)
            nbad = int(np.count_nonzero(err > 1e-5 * refabs)) + int(np.count_nonzero(g[refabs == 0]))
        else:
            ref = fn(oracle.orient(f, rows[k]))
            ref32 = ((ref + 2 ** 31) % 2 ** 32) - 2 ** 31
            nbad = int(np.count_nonzero(g.astype(np.int64) != ref32))
        if nbad:
            bad.append((b, j, k, nbad))
    return bad


def compare_all(tmpdir, cubes: np.ndarray, gpu_out: np.ndarray, mask: int, transform: str = "drt",
                table: int = 0, procs: int | None = None, per_task: int = 1):
    """cubes [B][N][N][N]; gpu_out [B][K][...] (stacked).  Returns the list of failing
    (cube, slot, dodecant, mismatches); empty means every element passed."""
    cubes = np.ascontiguousarray(cubes)
    cp = os.path.join(str(tmpdir), "cubes.npy")
    op = os.path.join(str(tmpdir), "gpu_out.npy")
    np.save(cp, cubes)
    np.save(op, np.ascontiguousarray(gpu_out))
    ks = [k for k in range(12) if (mask >> k) & 1]
    items = [(b, j, k) for b in range(cubes.shape[0]) for j, k in enumerate(ks)]
    chunks = [items[i:i + per_task] for i in range(0, len(items), per_task)]
    procs = procs or min(len(chunks), os.cpu_count() or 1, 16)
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_check, [(cp, op, transform, table, c) for c in chunks])
    os.remove(op)
    return [x for r in res for x in r]
