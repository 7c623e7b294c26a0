"""cfg4 (DJT N=64, dodecant 0) a few times -- target for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2501_13664_b200 as d3
cube = torch.from_numpy(synth.config_input(4)).cuda()
out = d3.lines(cube, 0x001)
for _ in range(3):
    d3.lines(cube, 0x001, out=out)
torch.cuda.synchronize()
