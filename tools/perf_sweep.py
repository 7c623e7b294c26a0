"""Forward transforms over sizes, dtypes and dodecant counts (CUDA events, median of 5 after 2
warm-ups, 512 MB L2 flush between calls): output GB/s, to spot slow paths."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2501_13664_b200 as d3
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def cube_of(N, dt, B=1):
    if dt == "f32":
        return torch.from_numpy(synth.normal_cube(N, 1, batch=B)).cuda()
    return torch.from_numpy(synth.uniform_cube(N, 1, np.uint8 if dt == "u8" else np.int32, 0, 255, batch=B)).cuda()
def timeit(fn):
    ts = []
    for i in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b))
    return statistics.median(ts)
cases = []
for N, masks in ((64, (0x1, 0xFFF)), (128, (0x1, 0xFFF)), (256, (0x1, 0xFFF)), (512, (0x1,))):
    for dt in ("u8", "i32", "f32"):
        for m in masks:
            cases.append(("drt", N, dt, m))
for N, masks in ((32, (0x1, 0xFFF)), (64, (0x1, 0xFFF)), (128, (0x1,))):
    for dt in ("u8", "f32"):
        for m in masks:
            cases.append(("djt", N, dt, m))
for kind, N, dt, m in cases:
    c = cube_of(N, dt)
    fn = d3.planes if kind == "drt" else d3.lines
    out = fn(c, m)
    ms = timeit(lambda: fn(c, m, out=out))
    gb = out.numel() * 4 / 1e9
    print(json.dumps({"kind": kind, "N": N, "dtype": dt, "dodecants": bin(m).count("1"), "ms": round(ms, 4),
                      "out_GB": round(gb, 3), "out_GBps": round(gb / ms * 1e3, 1)}), flush=True)
    del out
    torch.cuda.empty_cache()
