"""Condense an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list
into ID, kernel, block, grid, duration (ns) and print per-kernel shares."""
import csv
import sys
from collections import defaultdict


def main(src, dst):
    lines = [l for l in open(src) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(dst, "w") as out:
        w = csv.writer(out)
        w.writerow(["ID", "Kernel", "Block", "Grid", "gpu__time_duration.sum_ns"])
        for r in rows[1:]:
            d = dict(zip(h, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"][:110]
            ns = float(d["Metric Value"].replace(",", ""))
            w.writerow([d["ID"], name, d["Block Size"], d["Grid Size"], ns])
            tot[name] += ns
            cnt[name] += 1
    s = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / s:5.1f}%  n={cnt[k]:4d}  mean={v / cnt[k] / 1e3:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
