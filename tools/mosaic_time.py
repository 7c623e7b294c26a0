"""Stacked vs mosaic layout of the 12-dodecant DRT (u8 -> i32), CUDA events, median of 10."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2501_13664_b200 as d3
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for N in (64, 128, 256):
    cube = torch.from_numpy(synth.uniform_cube(N, 5, __import__("numpy").uint8)).cuda()
    for lay, name in ((d3.DRT3D_LAYOUT_STACKED, "stacked"), (d3.DRT3D_LAYOUT_MOSAIC, "mosaic")):
        out = d3.planes(cube, 0xFFF, layout=lay)
        ts = []
        for i in range(13):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); d3.planes(cube, 0xFFF, layout=lay, out=out); b.record(); torch.cuda.synchronize()
            if i >= 3: ts.append(a.elapsed_time(b))
        print(N, name, "ms", round(statistics.median(ts), 4), "out GB", out.numel() * 4 / 1e9)
