import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_13664_b200 as d3
N = 512
def col0(f):
    out = d3.planes(torch.from_numpy(f).cuda()[None], 0x001)[0, 0]
    return int(out[0, 0].to(torch.int64).sum()), int(out[N//2, 7].to(torch.int64).sum())
for axis in (0, 1, 2):
    lost = []
    for v in range(0, N, 8):
        f = np.zeros((N, N, N), np.uint8)
        idx = [slice(None)] * 3; idx[axis] = v
        f[tuple(idx)] = 1
        a, b = col0(f)
        if a != N * N or b != N * N: lost.append((v, a, b))
    print('axis', axis, 'planes with lost mass (every 8th):', lost[:12], len(lost))
