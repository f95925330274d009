"""Per-region stall breakdown of an ncu source page (SASS), with role markers."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
step = int(sys.argv[2]) if len(sys.argv) > 2 else 250
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(raw.splitlines()[1:]))))
hdr, data = rows[0], rows[1:]
isrc = hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iall] or 0) for r in data)
MARK = {"LDGSTS": "cp.async", "UTCIMMA": "mma", "UBLKCP": "bulk", "LDTM": "ldtm", "STTM": "sttm",
        "STG": "stg", "SYNCS.PHASECHK": "wait", "LDG": "ldg", "FFMA": "ffma", "DFMA": "dfma"}
for s in range(0, len(data), step):
    seg = data[s:s + step]
    smp = sum(int(r[iall] or 0) for r in seg)
    if smp == 0:
        continue
    ex = sum(int(r[iex] or 0) for r in seg)
    marks = sorted({v for r in seg for k, v in MARK.items() if k in r[isrc] and int(r[iex] or 0) > 0})
    st = sorted(((sum(int(r[i] or 0) for r in seg), hdr[i][6:]) for i in stalls), reverse=True)[:4]
    print(f"{s:5d} {100*smp/tot:5.1f}% ex={ex:11d} [{','.join(marks)}] " +
          " ".join(f"{n}={100*v/tot:.1f}" for v, n in st))
