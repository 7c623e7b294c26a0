"""Per-phase clock accounting of the separable on-chip N = 32 kernel (debug build libdrt3d_sepprof.so,
bash tools/build_variant.sh sepprof -DD3_PROF_SEP32): lane 0 of warps 0 (X1 / Y1 side) and 7
(zero writer / Y2 side), cycles per CTA."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["D3_LIB"] = os.path.join(ROOT, "paper_2501_13664_b200", "libdrt3d_sepprof.so")
import torch
import paper_2501_13664_b200 as d3, synth
L = d3.lib()
cube = torch.from_numpy(synth.config_input(5)).cuda()
for _ in range(3):
    out = d3.planes(cube, 0xFFF)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
L.d3_sep_prof_read(buf)
out = d3.planes(cube, 0xFFF, out=out)
torch.cuda.synchronize()
L.d3_sep_prof_read(buf)
v = list(buf)
names = ["staging", "X1 / zeros", "cluster barrier", "X2", "Y batch 0", "Y batch 1", "(end)"]
for b, who in ((0, "warp 0"), (16, "warp 7")):
    n = max(v[b + 15], 1)
    tot = sum(v[b:b + 6])
    print(who, "CTAs", n, "cycles/CTA", tot / n)
    for i, nm in enumerate(names[:6]):
        print(f"  {nm:18s} {v[b + i] / n:8.0f} ({100 * v[b + i] / tot:4.1f}%)")
