"""One multigrid inverse call (2 iterations) at N (argv[1], default 256), 12 dodecants -- target for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2501_13664_b200 as d3
N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cube = torch.from_numpy(synth.normal_cube(N, 3)).cuda()
b = d3.planes(cube, 0xFFF)
x, rn = d3.planes_invert(b, 2)
torch.cuda.synchronize()
print("rnorm", rn.cpu().numpy())
