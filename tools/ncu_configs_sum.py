"""Summarise gpurun_out/ncu_cfg<k>.csv: the launches of the second call of each config ->
total duration, DRAM read+write bytes, GB/s and % of the measured 6540 GB/s copy peak."""
import csv, json
PEAK = 6540.2
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
for c in (1, 2, 3, 4, 5):
    rows = [r for r in csv.reader(l for l in open(f"gpurun_out/ncu_cfg{c}.csv") if not l.startswith("=="))]
    h = rows[0]
    ids = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
        ids.setdefault(int(d["ID"]), {})[d["Metric Name"]] = v
    launches = [ids[k] for k in sorted(ids)]
    second = launches[len(launches) // 2:]
    t = sum(x["gpu__time_duration.sum"] for x in second)
    b = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in second)
    print(json.dumps({"config": c, "launches": len(second), "kernel_ms": t * 1e3, "dram_bytes": b,
                      "dram_gbs": b / t / 1e9, "pct_of_measured_peak": 100 * b / t / 1e9 / PEAK}))
