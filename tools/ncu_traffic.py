"""DRAM traffic per launch of the dominant kernel (3x3 FP4 conv_tc launches) from
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv
written to profiles/ncu_conv_tc_summary.json (read by bench.py as roofline.traffic)."""
import csv
import io
import json
import sys
from collections import defaultdict

src = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_conv_tc_summary.json"
txt = open(src).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
per = defaultdict(dict)
names = {}
for r in rows:
    per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    per[r["ID"]]["unit_" + r["Metric Name"]] = r["Metric Unit"]
    names[r["ID"]] = r["Kernel Name"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
launches = []
for i, m in per.items():
    nm = names[i]
    if "conv_tc_kernel<9" not in nm:
        continue
    targs = [a.strip() for a in nm.split("conv_tc_kernel<", 1)[1].split(">", 1)[0].split(",")]
    if len(targs) < 5 or targs[4] not in ("1", "true"):  # template arg FP4 (any CPS / commit variant)
        continue
    rd = m["dram__bytes_read.sum"] * scale[m["unit_dram__bytes_read.sum"]]
    wr = m["dram__bytes_write.sum"] * scale[m["unit_dram__bytes_write.sum"]]
    t = m["gpu__time_duration.sum"] * scale[m["unit_gpu__time_duration.sum"]]
    launches.append({"id": int(i), "dram_read": rd, "dram_write": wr, "seconds": t})
launches.sort(key=lambda d: d["id"])
launches = launches[:17]  # one forward: the 17 3x3 convs
n = len(launches)
summary = {
    "source": src, "kernel": "conv_tc_kernel<9, false, 8, CPS, true, *> (3x3, kind::mxf4, every variant)",
    "launches": n,
    "dram_bytes_per_launch_avg": sum(d["dram_read"] + d["dram_write"] for d in launches) / max(n, 1),
    "dram_read_per_launch_avg": sum(d["dram_read"] for d in launches) / max(n, 1),
    "dram_write_per_launch_avg": sum(d["dram_write"] for d in launches) / max(n, 1),
    "per_launch": launches,
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "per_launch"}))
