"""Build libmbunet.so variants that differ only in conv_tc.cu's flags, reusing the cached
objects of the other sources (build/obj). Variants compile in parallel.
usage: python tools/build_conv_variant.py name1="-DFLAG1 -DFLAG2" name2="-DFLAG3" ...
Outputs build/ab/<name>.so (use with MBU_LIB=... / tools/ab_bench.sh)."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import __graft_entry__ as G  # noqa: E402

G.build_lib()  # refresh build/obj for the current sources
out = G.ROOT / "build" / "ab"
out.mkdir(parents=True, exist_ok=True)
objdir = G.ROOT / "build" / "obj"
others = []
for src in sorted(G.CSRC.glob("*.cu")):
    if src.name == "conv_tc.cu":
        continue
    cands = sorted(objdir.glob(f"{src.stem}.*.o"), key=lambda p: p.stat().st_mtime)
    others.append(str(cands[-1]))


def one(spec):
    name, flags = spec.split("=", 1)
    obj = out / f"{name}.conv_tc.o"
    subprocess.run([G._nvcc(), *G.NVCC_FLAGS, *flags.split(), "-c", "-o", str(obj),
                    str(G.CSRC / "conv_tc.cu")], check=True, capture_output=True)
    subprocess.run([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                    str(out / f"{name}.so"), str(obj), *others], check=True)
    return str(out / f"{name}.so")


with ThreadPoolExecutor(len(sys.argv) - 1) as ex:
    for p in ex.map(one, sys.argv[1:]):
        print(p)
