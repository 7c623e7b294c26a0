"""Aggregate an ncu SASS source page (csv) by opcode: executed instructions,
stall samples, shared-memory wavefronts (ideal / excessive)."""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    agg = defaultdict(lambda: [0, 0, 0, 0, 0])
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        op = r[ix["Source"]].strip().split(" ")[0]
        if op.startswith("@"):
            op = r[ix["Source"]].strip().split(" ")[1]
        op = op.split(".")[0]
        def f(k):
            try:
                return float(r[ix[k]].replace(",", "") or 0)
            except (ValueError, KeyError):
                return 0.0
        a = agg[op]
        a[0] += f("Instructions Executed")
        a[1] += f("Warp Stall Sampling (All Samples)")
        a[2] += f("L1 Wavefronts Shared")
        a[3] += f("L1 Wavefronts Shared Excessive")
        a[4] += f("Warp Stall Sampling (Not-issued Samples)")
    ti = sum(a[0] for a in agg.values()) or 1
    ts = sum(a[1] for a in agg.values()) or 1
    print(f"total warp-instr {ti:.0f}  stall samples {ts:.0f}")
    for op, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(top)]:
        print(f"{op:10s} inst {100*a[0]/ti:5.1f}%  samples {100*a[1]/ts:5.1f}%  smem_wf {a[2]:10.0f}  excess {a[3]:9.0f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
