import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_13664_b200 as d3
N = 512
rng = np.random.default_rng(0)
f = rng.integers(0, 4, (N, N, N)).astype(np.uint8)
tot = int(f.astype(np.int64).sum())
for dt in (torch.uint8, torch.int32, torch.float32):
    cube = torch.from_numpy(f).cuda().to(dt)
    out = d3.planes(cube[None], 0x001)[0, 0].to(torch.float64)
    torch.cuda.synchronize()
    sums = out.sum(dim=2)
    bad = (sums != tot)
    print(dt, 'bad columns', int(bad.sum()), 'of', N * N)
    if int(bad.sum()):
        idx = torch.nonzero(bad)[:8].cpu().numpy().tolist()
        print('  first bad (s1,s2):', idx, 'sums', [float(sums[a, b]) for a, b in idx[:4]], 'tot', tot)
        b1 = bad.any(dim=1).nonzero().reshape(-1)[:20].cpu().numpy().tolist()
        b2 = bad.any(dim=0).nonzero().reshape(-1)[:20].cpu().numpy().tolist()
        print('  bad s1 values', b1, '\n  bad s2 values', b2)
        print('  bad count per s1 mod 8', [int(bad[i::8].sum()) for i in range(8)], 'per s2 mod 8', [int(bad[:, i::8].sum()) for i in range(8)])
