"""Per-phase clock accounting of the SWAR first pass (debug build libdrt3d_swprof.so)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["D3_LIB"] = os.path.join(ROOT, "paper_2501_13664_b200", "libdrt3d_swprof.so")
import numpy as np, torch
import paper_2501_13664_b200 as d3, synth
L = d3.lib()
cube = torch.from_numpy(synth.config_input(3)).cuda()
for _ in range(3):
    out = d3.planes(cube, 0xFFF)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
for mask, name in ((0xFFF, "all 12 dodecants (one launch)"), (0x001, "dodecant 0 (z-fast)"), (0x010, "dodecant 4 (y-fast)"), (0x100, "dodecant 8 (x-fast)")):
    L.d3_swar_prof_read(buf)
    out = d3.planes(cube, mask)
    torch.cuda.synchronize()
    L.d3_swar_prof_read(buf)
    v = list(buf)
    n = max(v[7], 1)
    tot = sum(v[:6])
    print(name, "tiles", v[7])
    for i, nm in enumerate(["staging", "x-step", "swap write + bar", "y-step", "unpack write + bar", "copy-out"]):
        print(f"  {nm:20s} {v[i] / n:8.0f} cycles/tile ({100 * v[i] / tot:4.1f}%)")
