"""Small invocations of every C-ABI entry point, for compute-sanitizer (memcheck,
racecheck, initcheck, synccheck on every kernel at small N).

usage: compute-sanitizer --tool <tool> python tools/sanitize_cases.py [quick]
Each case's result is checked against the device result of the same call at a smaller size or
with an invariant (mass per column), so a sanitizer-clean run is also a correct one.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2501_13664_b200 as d3  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
Ns = (4, 8, 16, 32) if quick else (4, 8, 16, 32, 64)


def cube(N, dt, seed, batch=None):
    if dt == np.float32:
        return torch.from_numpy(synth.normal_cube(N, seed, batch=batch)).cuda()
    lo, hi = (0, 255) if dt == np.uint8 else (-100, 100)
    return torch.from_numpy(synth.uniform_cube(N, seed, dt, lo, hi, batch=batch)).cuda()


n_cases = 0
for N in Ns:
    for dt in (np.uint8, np.int32, np.float32):
        c = cube(N, dt, 10 + N, batch=2 if N <= 16 else None)
        out = d3.planes(c, 0xFFF)
        tot = c.to(torch.float64).sum(dim=(-3, -2, -1))
        col = out.to(torch.float64).sum(dim=-1)                # mass per (s1, s2) column
        assert torch.allclose(col, tot.reshape(tot.shape + (1, 1, 1)).expand_as(col), rtol=1e-4, atol=1e-2), (N, dt)
        d3.planes(c, 0x421)
        lines = d3.lines(c, 0xFFF if N <= 16 else 0x003)
        if dt != np.uint8:
            d3.planes_adjoint(out, 0xFFF)
            d3.lines_adjoint(lines, 0xFFF if N <= 16 else 0x003)
        n_cases += 5
    if N in (8, 32):
        d3.planes(cube(N, np.uint8, 3), 0xFFF, layout=d3.DRT3D_LAYOUT_MOSAIC)
        d3.planes(cube(N, np.int32, 4), 0xFFF, table=d3.DRT3D_TABLE_PRINTED)
        n_cases += 2
# iterative inverse (F-3) and applications (F-4)
f = cube(16, np.float32, 5)
b = d3.planes(f, 0xFFF)
d3.planes_invert(b, 2)
c = d3.planes(cube(32, np.uint8, 6), 0xFFF)
d3.coef_argmax(c)
d3.coef_threshold(c, 1, 2)
flags, _ = d3.detect_planes(c, 0xFFF, 1, 3, 1, 10)
d3.planes_adjoint(d3.coef_select(c, flags), 0xFFF)
n_cases += 6
# host-buffer entry (pinned host memory, copy stream)
hc = torch.from_numpy(synth.uniform_cube(32, 7, np.uint8)).pin_memory()
ho = torch.empty((12, 32, 32, 96), dtype=torch.int32).pin_memory()
dc = torch.empty((32, 32, 32), dtype=torch.uint8, device="cuda")
do = torch.empty((12, 32, 32, 96), dtype=torch.int32, device="cuda")
o = d3.make_opts()
wsb = d3.drt3d_planes_workspace_size(32, 0xFFF, o)
ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
assert d3.drt3d_planes_host(hc.data_ptr(), 32, 0xFFF, ho.data_ptr(), o, dc.data_ptr(), do.data_ptr(),
                            ws.data_ptr(), wsb, st) == d3.DRT3D_OK
n_cases += 1
torch.cuda.synchronize()
print(f"sanitize_cases: {n_cases} calls OK")
