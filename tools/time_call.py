"""Time one C-ABI transform call (CUDA events, median of 10 after 3 warm-ups, L2 flushed between
calls).  usage: python tools/time_call.py drt|djt N u8|i32|f32 batch mask"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2501_13664_b200 as d3  # noqa: E402

kind, N, dt, B, mask = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5], 0)
npdt = {"u8": np.uint8, "i32": np.int32, "f32": np.float32}[dt]
cube = synth.normal_cube(N, 1, batch=B) if dt == "f32" else synth.uniform_cube(N, 1, npdt, 0, 255, batch=B)
c = torch.from_numpy(cube).cuda()
fn = d3.planes if kind == "drt" else d3.lines
out = fn(c, mask)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(13):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn(c, mask, out=out)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
print(f"{kind} N={N} {dt} batch={B} mask={mask:#x} lib={os.path.basename(d3.LIB_PATH)} ms_median {statistics.median(ts):.4f} "
      f"best {min(ts):.4f} out_GB/s {out.numel() * 4 / min(ts) / 1e6:.0f}")
