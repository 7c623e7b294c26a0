"""N = 32, 256 cubes x 12 dodecants, per input dtype (u8 / i32 / f32): one C-ABI call timed with CUDA
events (median of 10 after 3 warm-ups, 512 MB L2 flush between calls).  D3_LIB selects the library."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2501_13664_b200 as d3

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name in ("u8", "i32", "f32"):
    if name == "f32":
        cube = synth.config_input(5)
    else:
        cube = synth.uniform_cube(32, 5, np.uint8 if name == "u8" else np.int32, 0, 255, batch=256)
    c = torch.from_numpy(cube).cuda()
    out = d3.planes(c, 0xFFF)
    ts = []
    for i in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); d3.planes(c, 0xFFF, out=out); b.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    print(json.dumps({"lib": os.path.basename(d3.LIB_PATH), "in": name, "N": 32, "batch": 256, "dodecants": 12,
                      "ms_median": statistics.median(ts)}))
