"""Build libmbunet.so with extra nvcc flags for some sources into build/ab/<name>.so
(e.g. -DMBU_TIMELINE for conv_tc.cu), leaving the in-tree library alone.
usage: python tools/build_variant.py <name> <src.cu>[,<src.cu>] <flag> [<flag> ...]"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import __graft_entry__ as G  # noqa: E402

name, srcs, flags = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
out = G.ROOT / "build" / "ab"
out.mkdir(parents=True, exist_ok=True)
objs = []
for src in sorted(G.CSRC.glob("*.cu")):
    obj = out / f"{name}.{src.stem}.o"
    fl = G.NVCC_FLAGS + (flags if src.name in srcs else [])
    subprocess.run([G._nvcc(), *fl, "-c", "-o", str(obj), str(src)], check=True, capture_output=True)
    objs.append(str(obj))
subprocess.run([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                str(out / f"{name}.so"), *objs], check=True)
print(out / f"{name}.so")
