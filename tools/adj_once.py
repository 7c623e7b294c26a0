"""Run the DRT N=256 x12 backprojection once (after one warm-up) -- target for ncu."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2501_13664_b200 as d3  # noqa: E402

N, mask = 256, 0xFFF
g = torch.Generator(device="cuda").manual_seed(3)
coef = torch.randint(0, 1000, (1, 12, N, N, 3 * N), dtype=torch.int32, device="cuda", generator=g)
cube = torch.empty((1, N, N, N), dtype=torch.int32, device="cuda")
for _ in range(2):
    d3.planes_adjoint(coef, mask, cube=cube)
torch.cuda.synchronize()
