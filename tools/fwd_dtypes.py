"""Forward DRT N=256 x12 for each input dtype (u8 -> i32, i32 -> i32, f32 -> f32), CUDA events."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_13664_b200 as d3

N = 256
g = torch.Generator(device="cuda").manual_seed(0)
base = torch.randint(0, 256, (1, N, N, N), dtype=torch.int32, device="cuda", generator=g)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, cube in (("u8", base.to(torch.uint8)), ("i32", base), ("f32", base.to(torch.float32))):
    out = d3.planes(cube, 0xFFF)
    ts = []
    for _ in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); d3.planes(cube, 0xFFF, out=out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"in": name, "N": N, "dodecants": 12, "ms_median": statistics.median(ts[2:])}))
