"""Runs the DESIGN.md quick-start snippet end to end (from the repo root)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2501_13664_b200 as d3
cube = torch.randint(0, 256, (256, 256, 256), dtype=torch.uint8, device="cuda")
coef = d3.planes(cube, 0xFFF)
rays = d3.lines(cube, 0x001)
back = d3.planes_adjoint(coef, 0xFFF)
x, rnorm = d3.planes_invert(coef.float(), iters=6)
flags, am = d3.detect_planes(coef, 0xFFF, 1, 3, 1, 10)
walls = d3.planes_adjoint(d3.coef_select(coef, flags), 0xFFF)
torch.cuda.synchronize()
print(coef.shape, rays.shape, back.shape, x.shape, rnorm[-1].item() / rnorm[0].item(), int(flags.sum()), walls.shape)
