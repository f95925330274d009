#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/x_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [names...] > profiles/x_full.md
    python tools/ncu_summary.py multi name1=a.ncu-rep name2=b.ncu-rep ... > profiles/x_full.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (realtime)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem LSU wavefronts %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def table(path):
    txt = open(path).read()
    return list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))


def launches(path):
    rows = table(path)
    tot = sum(float(r["Metric Value"]) for r in rows)
    print(f"# ncu launch list (`gpu__time_duration.sum`, --clock-control none)\n\nsource: `{path}`; "
          f"{len(rows)} launches, {tot/1e3:.1f} us total (cold-cache, serialised)\n")
    print("| id | kernel | grid | block | us | share |\n|---|---|---|---|---|---|")
    for r in rows:
        t = float(r["Metric Value"])
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        print(f"| {r['ID']} | `{name}` | {r['Grid Size']} | {r['Block Size']} | {t/1e3:.1f} | "
              f"{100*t/tot:.1f}% |")


def full(path, names):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary\n\nsource: `{path}`\n")
    cols = names or [f"launch {i}" for i in range(len(data))]
    print("| metric | unit | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    kn = idx.get("Kernel Name")
    if kn is not None:
        print("| kernel | | " + " | ".join(f"`{d[kn].split('(')[0]}`" for d in data) + " |")
    for key, label in KEYS:
        if key in idx:
            i = idx[key]
            print(f"| {label} (`{key}`) | {units[i]} | " + " | ".join(d[i] for d in data) + " |")


def multi(pairs):
    """One column per report (first launch of each): name=path arguments."""
    cols, datas, units, idx = [], [], None, None
    for pr in pairs:
        name, path = pr.split("=", 1)
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, u, data = rows[0], rows[1], rows[2:]
        i = {h: k for k, h in enumerate(hdr)}
        cols.append(name)
        datas.append({h: data[0][k] for h, k in i.items()})
        units = units or {h: u[k] for h, k in i.items()}
    print("# ncu --set full summary (first captured launch of each report)\n")
    print("| metric | unit | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    print("| kernel | | " + " | ".join(f"`{d.get('Kernel Name', '').split('(')[0]}`" for d in datas) + " |")
    for key, label in KEYS:
        if key in units:
            print(f"| {label} (`{key}`) | {units[key]} | " + " | ".join(d.get(key, "") for d in datas) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "multi":
        multi(sys.argv[2:])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3:])
