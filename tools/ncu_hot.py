"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, isrc, iall, inot, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                     "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"))
data = rows[1:]
tot = sum(int(r[iall]) for r in data)
print(f"total samples {tot}, {len(data)} SASS lines")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iall]))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {int(r[iall]):7d} {100*int(r[iall])/tot:5.1f}% ex={r[iex]:>9} {r[isrc].strip()[:90]}")

if len(sys.argv) > 3:
    step = int(sys.argv[3])
    print("\nregion  samples  warp-instr")
    for s in range(0, len(data), step):
        seg = data[s:s + step]
        smp = sum(int(r[iall]) for r in seg)
        ex = sum(int(r[iex] or 0) for r in seg)
        print(f"{s:5d}-{s+step:5d} {100*smp/tot:5.1f}% {ex:12d}  {seg[0][isrc].strip()[:50]}")
