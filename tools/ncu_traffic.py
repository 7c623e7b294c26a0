"""Write profiles/ncu_traffic.json from an ncu --set full report: mean dram read+write bytes per
launch of each kernel (the bench's roofline `traffic` uses the final pass)."""
import csv, json, subprocess, sys
from collections import defaultdict


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    acc = defaultdict(list)
    units = rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ui = h.index("dram__bytes_read.sum")
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(units[ui], 1)
        wi = h.index("dram__bytes_write.sum")
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(units[wi], 1)
        acc[d["Kernel Name"]].append(rd + wr)
    res = {k: sum(v) / len(v) for k, v in acc.items()}
    fin = [v for k, v in res.items() if "drt_pass_kernel" in k and ", 0, 1>" in k]
    j = {"source": rep.split("/")[-1] + " (ncu --set full --cache-control none --clock-control none)",
         "per_kernel_dram_bytes_per_launch": res,
         "final_pass_dram_bytes_per_launch": fin[0] if fin else None}
    json.dump(j, open(out, "w"), indent=1)
    print(json.dumps(j, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
