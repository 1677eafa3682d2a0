"""A/B of the warp-specialised prototype against the production strip kernel:
bitwise comparison + CUDA-event timing on config-2 frames.  python tools/ws/ws_ab.py lib.so [...]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2005_08165_b200 as tfn  # noqa: E402
import tfn_scenes as ts  # noqa: E402

B, H, W = 1024, 480, 640
K = ts.K_VGA
sc = ts.random_scenes(B, K, H, W, seed=0)
z = ts.render(sc, K, H, W, device="cuda").depth.contiguous()
est = tfn.Estimator(K, filter="sobel", nz_mode="median", kernel="strip")
ref = torch.empty((B, 3, H, W), device="cuda")
work = torch.zeros(4, dtype=torch.int32, device="cuda")


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


t_ref = timeit(lambda: est.estimate(z, out=ref))
print(f"strip: {B*H*W/t_ref/1e6:.1f} Gpx/s ({t_ref:.3f} ms)", flush=True)
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    lib.ws_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_float,
                           ctypes.c_float, ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_int, ctypes.c_void_p]
    out = torch.full((B, 3, H, W), 7.0, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for sh in (48,):
        run = lambda: lib.ws_run(z.data_ptr(), B, H, W, K.fx, K.fy, K.u0, K.v0, out.data_ptr(), sh,  # noqa: E731
                                 work.data_ptr(), 0, st)
        rc = run()
        torch.cuda.synchronize()
        same = torch.equal(out.view(torch.int32), ref.view(torch.int32))
        t = timeit(run)
        print(f"{os.path.basename(path)} sh={sh} occ={lib.ws_occupancy()} rc={rc}: {B*H*W/t/1e6:.1f} Gpx/s "
              f"({t:.3f} ms) bitwise={same}", flush=True)
