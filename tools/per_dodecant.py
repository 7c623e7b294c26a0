"""First-pass / final-pass time per dodecant (one-dodecant calls, per-launch CUDA events through
opts.events) on the cfg3 cube: exposes orientation-dependent staging costs."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2501_13664_b200 as d3
N = 256
cube = torch.from_numpy(synth.config_input(3)).cuda()
out = torch.empty((1, 1, N, N, 3 * N), dtype=torch.int32, device="cuda")
o = d3.make_opts(batch=1, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
for e in evs: e.record()
torch.cuda.synchronize()
arr = (ctypes.c_void_p * 8)(*[e.cuda_event for e in evs])
o.events = ctypes.cast(arr, ctypes.c_void_p); o.max_events = 4
ws_b = d3.drt3d_planes_workspace_size(N, 0x001, o)
ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
rows = d3.orientation_table()
for k in range(12):
    t0, t1 = [], []
    for _ in range(6):
        assert d3.drt3d_planes(cube.data_ptr(), N, 1 << k, out.data_ptr(), o, ws.data_ptr(), ws_b, st) == 0
        torch.cuda.synchronize()
        t0.append(evs[0].elapsed_time(evs[1])); t1.append(evs[2].elapsed_time(evs[3]))
    print(k, rows[k], 'first %.1f us' % (1e3 * statistics.median(t0[2:])), 'final %.1f us' % (1e3 * statistics.median(t1[2:])))
