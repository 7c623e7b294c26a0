"""Bit-exact check of a side-library variant against the product library on the cfg3 workload
(and a saturated cube): both libraries run the same cube into outputs pre-filled with -1, the
outputs must be identical and contain no -1 left over.  usage: python tools/variant_check.py TAG
(runs the variant in a subprocess with D3_LIB set; measurement tooling, GPU only)."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(kind):
    import torch
    import paper_2501_13664_b200 as d3
    from synth import sparse_cube
    N = 256
    if kind == "sparse":
        cube = torch.from_numpy(sparse_cube(N, 3)).cuda()
    else:
        cube = torch.full((N, N, N), 255, dtype=torch.uint8, device="cuda")
    out = torch.full((12, N, N, 3 * N), -1, dtype=torch.int32, device="cuda")
    d3.planes(cube, 0xFFF, out=out)
    torch.cuda.synchronize()
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
    print(kind, h, int((out == -1).sum()))


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        run(sys.argv[2])
        sys.exit(0)
    tag = sys.argv[1]
    ok = True
    for kind in ("sparse", "saturated"):
        res = []
        for lib in (None, os.path.join(ROOT, "paper_2501_13664_b200", f"libdrt3d_{tag}.so")):
            env = dict(os.environ)
            env.pop("D3_LIB", None)
            if lib:
                env["D3_LIB"] = lib
            r = subprocess.run([sys.executable, __file__, "--run", kind], env=env, capture_output=True, text=True)
            res.append(r.stdout.strip() or r.stderr[-500:])
        same = res[0] == res[1] and res[0].endswith(" 0")
        ok &= same
        print(kind, "base:", res[0], "| variant:", res[1], "->", "OK" if same else "MISMATCH")
    sys.exit(0 if ok else 1)
