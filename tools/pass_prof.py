"""Per-phase clock accounting of the u16 final pass (debug build libdrt3d_ppprof.so)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["D3_LIB"] = os.path.join(ROOT, "paper_2501_13664_b200", "libdrt3d_ppprof.so")
import numpy as np, torch
import paper_2501_13664_b200 as d3, synth
L = d3.lib()
cube = torch.from_numpy(synth.config_input(3)).cuda()
for _ in range(3):
    out = d3.planes(cube, 0xFFF)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
L.d3_pass_prof_read(buf)
out = d3.planes(cube, 0xFFF)
torch.cuda.synchronize()
L.d3_pass_prof_read(buf)
v = list(buf)
n = max(v[7], 1)
names = ["staging issue", "staging wait+bar", "x-step", "bar after x", "write X + bar", "y-step", "stores"]
tot = sum(v[:7])
for i, nm in enumerate(names):
    print(f"{nm:18s} {v[i] / n:9.0f} cycles per tile  ({100 * v[i] / tot:4.1f}%)")
print("tiles", v[7], "total cycles per tile", tot / n)
