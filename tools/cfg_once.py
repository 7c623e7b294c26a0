"""One BASELINE config (argv[1]) called twice through the C ABI (the second call is the one ncu summarises)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2501_13664_b200 as d3
cfg = int(sys.argv[1])
kind, mask = {1: ("drt", 0x001), 2: ("drt", 0xFFF), 3: ("drt", 0xFFF), 4: ("djt", 0x001), 5: ("drt", 0xFFF)}[cfg]
cube = torch.from_numpy(synth.config_input(cfg)).cuda()
fn = d3.planes if kind == "drt" else d3.lines
out = fn(cube, mask)
fn(cube, mask, out=out)
torch.cuda.synchronize()
