"""Fast A/B builds: recompile ONE strip translation unit with extra flags / defines and link
it with the in-tree objects of the others (build/libtfn_*.o from the last full build).
   python tools/build_variant_tu.py name sobel "-Xptxas -O2" [-DFOO=1 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2005_08165_b200 import build as b  # noqa: E402

name, tu, extra = sys.argv[1], sys.argv[2], sys.argv[3].split()
defs = sys.argv[4:]
bdir = os.path.join(b.HERE, "build")
src = f"tfn_strip_{tu}.cu"
obj = os.path.join(bdir, f"var_{name}_{tu}.o")
cmd = ["nvcc", *b.ARCH, *b.NVCC_FLAGS, *extra, *defs, "-I", os.path.join(b.ROOT, "include"), "-c",
       os.path.join(b.CSRC, src), "-o", obj]
out = subprocess.run(cmd, capture_output=True, text=True)
if out.returncode:
    sys.exit(out.stdout + out.stderr)
objs = [os.path.join(bdir, f"libtfn_{s.replace('.cu', '.o')}") for s in b.SOURCES if s != src] + [obj]
so = os.path.join(b.ROOT, "abl", f"lib_{name}.so")
os.makedirs(os.path.dirname(so), exist_ok=True)
subprocess.check_call(["nvcc", *b.ARCH, "-shared", "-o", so, *objs, "-lcudart"])
print(so)
