"""Build libtfn.so (the C ABI + sm_100a kernels) in-tree with nvcc.

`python -m paper_2005_08165_b200.build` or __graft_entry__.build().  The .so is
git-ignored but travels to the GPU box with the gpurun snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libtfn.so")
SOURCES = ["tfn_abi.cu", "tfn_kernels.cu", "tfn_stats.cu", "tfn_strip_fd.cu", "tfn_strip_sobel.cu",
           "tfn_strip_scharr.cu", "tfn_strip_prewitt.cu", "tfn_strip_custom.cu",
           "tfn_planefit.cu", "tfn_f32_fd.cu", "tfn_f32_sobel.cu", "tfn_f32_scharr.cu", "tfn_f32_prewitt.cu",
           "tfn_f32_custom.cu"]
HEADERS = ["tfn_device.cuh", "tfn_kernels.h", "tfn_strip.cuh", "tfn_strip_inst.cuh", "tfn_f32.cuh", "tfn_f32_inst.cuh", "tfn_tma.cuh",
           os.path.join("..", "..", "include", "tfn.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    SO_ = out or SO
    if not force and out is None and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for src in SOURCES:
        tag = os.path.basename(SO_).replace(".so", "")
        obj = os.path.join(HERE, "build", f"{tag}_{src.replace('.cu', '.o')}")
        extra = os.environ.get("TFN_NVCC_EXTRA", "").split()      # A/B of compiler knobs (tools/build_ab.py)
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    log = []
    for src, cmd, p in procs:
        out = p.communicate()[0].decode()
        log.append(f"== {src}\n{out}")
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed for {src}")
    with open(os.path.join(HERE, "build", "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    cmd = [nvcc, *ARCH, "-shared", "-o", SO_ + ".tmp", *objs, "-lcudart"]   # driver API via cudaGetDriverEntryPoint
    subprocess.check_call(cmd)
    os.replace(SO_ + ".tmp", SO_)
    if verbose:
        print("\n".join(log))
    return SO_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
