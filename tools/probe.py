"""Run one transform configuration in a fresh process and report errors (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_13664_b200 as d3, synth, oracle

def main(kind, N, mask, dtype):
    dt = {"u8": np.uint8, "i32": np.int32, "f32": np.float32}[dtype]
    cube = synth.normal_cube(N, 1, batch=1) if dt == np.float32 else synth.uniform_cube(N, 1, dt, 0, 255, batch=1)
    g = torch.from_numpy(cube).cuda()
    out = d3.planes(g, mask) if kind == "drt" else d3.lines(g, mask)
    torch.cuda.synchronize()
    ref = oracle.drt_planes(cube, mask) if kind == "drt" else oracle.djt_lines(cube, mask)
    got = out.cpu().numpy()
    ok = np.allclose(got, ref, rtol=1e-4, atol=1e-3) if dt == np.float32 else np.array_equal(got.astype(np.int64), ref)
    print(kind, N, hex(mask), dtype, "OK" if ok else "MISMATCH", flush=True)

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3], 0), sys.argv[4])
