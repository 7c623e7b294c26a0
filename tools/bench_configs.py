"""Secondary measurement: every BASELINE.json config through the C ABI on one B200.

Inputs are the seeded synthetic cubes of synth/ (DESIGN.md §4), resident in HBM; each call is
timed with CUDA events on the launching stream after 3 warm-ups, median of 10 (a 512 MB L2 flush
between calls).  Prints one JSON object per config; the headline line is bench.py's (config 3).
"""
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2501_13664_b200 as d3  # noqa: E402

CFG = {
    1: ("drt", 0x001), 2: ("drt", 0xFFF), 3: ("drt", 0xFFF), 4: ("djt", 0x001), 5: ("drt", 0xFFF),
}


def run(cfg, iters=10):
    kind, mask = CFG[cfg]
    cube = torch.from_numpy(synth.config_input(cfg)).cuda()
    B, N = cube.shape[0], cube.shape[1]
    K = bin(mask).count("1")
    fn = (lambda: d3.planes(cube, mask, out=out, workspace=ws)) if kind == "drt" else \
        (lambda: d3.lines(cube, mask, out=out, workspace=ws))
    o = d3.make_opts(batch=B, in_dtype=d3._dtype_code(cube), out_dtype=d3.DRT3D_F32 if cube.dtype == torch.float32
                     else d3.DRT3D_I32)
    if kind == "drt":
        out = torch.empty((B, K, N, N, 3 * N), dtype=torch.float32 if cube.dtype == torch.float32 else torch.int32,
                          device="cuda")
        wsb = d3.drt3d_planes_workspace_size(N, mask, o)
    else:
        out = torch.empty((B, K, N, N, 2 * N, 2 * N), dtype=torch.float32 if cube.dtype == torch.float32 else torch.int32,
                          device="cuda")
        wsb = d3.djt3d_lines_workspace_size(N, mask, o)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    vox = B * N ** 3
    cells = out.numel()
    res = {"config": cfg, "transform": kind, "N": N, "batch": B, "dodecants": K, "dtype": str(cube.dtype),
           "ms_median": ms, "ms_best": min(ts), "gvoxel_per_s": vox / (ms * 1e-3) / 1e9,
           "out_cells_per_s": cells / (ms * 1e-3), "out_bytes": out.numel() * out.element_size(),
           "out_write_gbs": out.numel() * out.element_size() / (ms * 1e-3) / 1e9}
    if kind == "drt":
        res["gplanes_per_s"] = B * K * N * N * (2 * N - 1) / (ms * 1e-3) / 1e9
    return res


def run_adjoint(cfg, iters=5):
    """Backprojection (F-1) on the coefficient shape of config cfg (3: DRT N=256 x12, 4: DJT N=64)."""
    kind, mask = CFG[cfg]
    N = {3: 256, 4: 64}[cfg]
    K = bin(mask).count("1")
    shape = (1, K, N, N, 3 * N) if kind == "drt" else (1, K, N, N, 2 * N, 2 * N)
    g = torch.Generator(device="cuda").manual_seed(cfg)
    coef = torch.randint(0, 1000, shape, dtype=torch.int32, device="cuda", generator=g)
    cube = torch.empty((1, N, N, N), dtype=torch.int32, device="cuda")
    fn = (lambda: d3.planes_adjoint(coef, mask, cube=cube)) if kind == "drt" else \
        (lambda: d3.lines_adjoint(coef, mask, cube=cube))
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    return {"config": f"adjoint-{cfg}", "transform": kind + "_adjoint", "N": N, "batch": 1, "dodecants": K,
            "ms_median": ms, "gvoxel_per_s": N ** 3 / (ms * 1e-3) / 1e9,
            "coef_read_gbs": coef.numel() * 4 / (ms * 1e-3) / 1e9}


def run_invert(N, iters=6):
    """Iterative inverse (F-3): `iters` multigrid iterations (n_min = 2) over all 12 dodecants,
    fp32, on a smooth synthetic phantom."""
    x, y, z = torch.meshgrid(*[torch.arange(N, dtype=torch.float32, device="cuda")] * 3, indexing="ij")
    f = torch.exp(-((x - 0.45 * N) ** 2 / (0.12 * N * N) + (y - 0.55 * N) ** 2 / (0.15 * N * N)
                    + (z - 0.5 * N) ** 2 / (0.18 * N * N)))
    b = d3.planes(f[None].contiguous(), 0xFFF)[0]
    o = d3.make_opts(batch=1, in_dtype=d3.DRT3D_F32, out_dtype=d3.DRT3D_F32)
    wsb = ctypes.c_size_t(0)
    d3.lib().drt3d_planes_invert_workspace_size(N, 2, 0xFFF, ctypes.byref(o), ctypes.byref(wsb))
    ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
    cube = torch.empty((N, N, N), dtype=torch.float32, device="cuda")
    d3.planes_invert(b, 1, cube=cube, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, rn = d3.planes_invert(b, iters, cube=cube, workspace=ws)
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    ms = statistics.median(ts)
    err = float(torch.linalg.norm(cube - f) / torch.linalg.norm(f))
    return {"config": f"invert-N{N}", "transform": "drt_invert", "N": N, "iters": iters, "dodecants": 12,
            "ms_median": ms, "ms_per_iter": ms / iters, "nrmsd": err,
            "rnorm_ratio": float(rn[-1] / rn[0]), "workspace_mb": wsb.value / 2 ** 20}


def _time(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    return statistics.median(ts)


def run_apps():
    """F-4: plane detection on a synthetic 128^3 room (PAPER.md:679's scene size: three walls, a box,
    0.5% clutter), and ray denoising (DJT dodecant 0 -> threshold 0.95 max -> backprojection) at N=64."""
    import numpy as np
    N = 128
    rng = np.random.default_rng(5)
    f = np.zeros((N, N, N), np.uint8)
    f[3, :, :] = 1
    f[:, N - 4, :] = 1
    f[:, :, 2] = 1
    f[N // 3:N // 2, N // 3:N // 2, N // 3:N // 2] = 1
    f = (f + (rng.random((N, N, N)) < 0.005)).astype(np.uint8)
    cube = torch.from_numpy(f).cuda()
    c = d3.planes(cube, 0xFFF)
    ws = d3._apps_ws(None, c.device)[0]
    t_fwd = _time(lambda: d3.planes(cube, 0xFFF, out=c))
    t_det = _time(lambda: d3.detect_planes(c, 0xFFF, 1, 3, 1, 10, workspace=ws))
    flags, _ = d3.detect_planes(c, 0xFFF, 1, 3, 1, 10, workspace=ws)
    yield {"config": "detect-N128", "transform": "drt+detect_planes", "N": N, "dodecants": 12,
           "forward_ms": t_fwd, "detect_ms": t_det, "coef_gbs_detect": c.numel() * 4 / (t_det * 1e-3) / 1e9,
           "planes_found": int(flags.sum())}
    N = 64
    g = torch.from_numpy(rng.integers(0, 201, (N, N, N)).astype(np.int32)).cuda()
    lc = d3.lines(g, 0x001)
    kept = torch.empty_like(lc)

    def pipe():
        d3.lines(g, 0x001, out=lc)
        d3.coef_threshold(lc, 95, 100, out=kept, workspace=ws)
        d3.lines_adjoint(kept, 0x001)
    t_pipe = _time(pipe)
    t_thr = _time(lambda: d3.coef_threshold(lc, 95, 100, out=kept, workspace=ws))
    yield {"config": "denoise-N64", "transform": "djt+threshold+djt_adjoint", "N": N, "dodecants": 1,
           "pipeline_ms": t_pipe, "threshold_ms": t_thr, "coef_gbs_threshold": 2 * lc.numel() * 4 / (t_thr * 1e-3) / 1e9}


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for c in cfgs:
        print(json.dumps(run(c, iters=10 if len(sys.argv) == 1 else 2)), flush=True)
    if len(sys.argv) == 1:
        for c in (3, 4):
            print(json.dumps(run_adjoint(c)), flush=True)
        for n in (64, 128, 256):
            print(json.dumps(run_invert(n)), flush=True)
        for r in run_apps():
            print(json.dumps(r), flush=True)
