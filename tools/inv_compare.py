"""The multigrid inverse through two libraries (D3_LIB_A, D3_LIB_B): results and timing per iteration."""
import ctypes, os, sys, json, statistics, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, json, statistics
sys.path.insert(0, %r)
import numpy as np, torch, synth, paper_2501_13664_b200 as d3
res = {}
for N in (64, 128, 256):
    cube = torch.from_numpy(synth.normal_cube(N, 3)).cuda()
    b = d3.planes(cube, 0xFFF)
    x, rn = d3.planes_invert(b, 3)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(); d3.planes_invert(b, 3); a1.record(); torch.cuda.synchronize(); ts.append(a0.elapsed_time(a1) / 3)
    np.save("/tmp/inv_x_%%d_%%s.npy" %% (N, os.environ["TAG"]), x.cpu().numpy())
    res[N] = {"rnorm": [float(v) for v in rn.cpu().numpy()], "ms_per_iter": min(ts)}
print(json.dumps(res))
''' % ROOT
out = {}
for tag, lib in (("A", os.environ["D3_LIB_A"]), ("B", os.environ["D3_LIB_B"])):
    env = dict(os.environ, D3_LIB=lib, TAG=tag)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    out[tag] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
import numpy as np
for N in ("64", "128", "256"):
    same = bool(np.array_equal(np.load("/tmp/inv_x_%s_A.npy" % N), np.load("/tmp/inv_x_%s_B.npy" % N)))
    print(N, "A", out["A"][N], "B", out["B"][N], "x identical:", same)
