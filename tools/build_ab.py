"""Build A/B variants of libtfn.so into abl/ (git-ignored, travels to the GPU box):
   python tools/build_ab.py name:DEF=1,DEF2=3 name2: ..."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2005_08165_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(b.ROOT, "abl"), exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    t = time.time()
    out = os.path.join(b.ROOT, "abl", f"lib_{name}.so")
    b.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    for f in os.listdir(os.path.join(b.HERE, "build")):       # keep the gpurun snapshot small
        if f.startswith(f"lib_{name}_"):
            os.remove(os.path.join(b.HERE, "build", f))
    print(f"{out} ({time.time() - t:.0f} s)", flush=True)
