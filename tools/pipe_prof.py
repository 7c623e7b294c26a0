"""Per-role clock accounting of the pipelined final pass (debug build libdrt3d_prof.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["D3_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "paper_2501_13664_b200", "libdrt3d_prof.so")
import numpy as np, torch
import paper_2501_13664_b200 as d3, synth
L = d3.lib()
cube = torch.from_numpy(synth.config_input(3)).cuda()
for _ in range(3):
    out = d3.planes(cube, 0xFFF)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
L.d3_pipe_prof_read(buf)
out = d3.planes(cube, 0x001)
torch.cuda.synchronize()
L.d3_pipe_prof_read(buf)
v = list(buf)
names = {0: "P wait empty", 1: "P issue", 4: "X wait raw", 5: "X accumulate", 6: "X wait Xempty", 7: "X write X",
         8: "Y wait Xfull", 9: "Y accumulate", 10: "Y store", 12: "X total", 13: "Y total", 14: "P total"}
# role order in the kernel: prof_base 0 = X (tid 0), 4 = Y, 8 = P
remap = {0: "X wait raw", 1: "X accumulate", 2: "X wait Xempty", 3: "X write X",
         4: "Y wait Xfull", 5: "Y accumulate", 6: "Y store", 7: "-",
         8: "P wait empty", 9: "P issue", 10: "-", 11: "-", 12: "X total", 13: "Y total", 14: "P total", 15: "-"}
for i in range(16):
    if remap[i] != "-":
        print(f"{remap[i]:16s} {v[i] / 148 / 1e3:10.1f} kcycles per CTA")
