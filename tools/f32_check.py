"""Quick GPU check of the fp32 unit-step kernel: parity vs the oracle on the standard scenes
and timing against the round-1 strip kernel on configs[1] (diagnostic, not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import tfn_scenes as ts
import paper_2005_08165_b200 as tfn
from tests.parity import compare


def run(sample, K, f, m, kernel, disp=False):
    est = tfn.Estimator(K, filter=f, nz_mode=m, kernel=kernel)
    x = torch.as_tensor(np.ascontiguousarray(sample, dtype=np.float32)).cuda()
    out = est.estimate_disparity(x, 60.0) if disp else est.estimate(x)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def check(name, s, K, f, m, kernels=("f32", "f32masked"), disp=False):
    s = np.ascontiguousarray(s, dtype=np.float32)
    if s.ndim == 2:
        s = s[None]
    r = oracle.estimate(s, K, f, m, disparity=disp, f_tc=60.0, threads=8)
    for k in kernels:
        g = run(s, K, f, m, k, disp)
        res = compare(g, r, s, K)
        ok = res["mask_equal"] and res["n_bad"] == 0
        print(f"{'OK ' if ok else 'BAD'} {name:22s} {f:7s} {m:6s} {k:10s} max={res['max_deg']:.2e} "
              f"maskdiff={res['mask_diff']} bad={res['n_bad']} tie={res['n_tie']} {res.get('worst', '')}", flush=True)


def timeit(K, f, m, kernel, x, reps=10):
    est = tfn.Estimator(K, filter=f, nz_mode=m, kernel=kernel)
    out = torch.empty((x.shape[0], 3, x.shape[1], x.shape[2]), device="cuda")
    if kernel.startswith("f32"):
        tfn.tfn.tfn_set_option(est.h, tfn.tfn.OPT_COUNT_SPECIAL, 1)
        est.estimate(x, out=out)
        n = tfn.tfn.tfn_debug_special_count(est.h)
        print(f"special pixels {kernel} {f}/{m}: {n} of {x.numel()} ({n / x.numel():.5f})", flush=True)
        tfn.tfn.tfn_set_option(est.h, tfn.tfn.OPT_COUNT_SPECIAL, 0)
    for _ in range(3):
        est.estimate(x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        est.estimate(x, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gpx = x.numel() / ms / 1e6
    print(f"time {kernel:10s} {f}/{m}: {ms:.3f} ms  {gpx:.1f} Gpx/s  {gpx * 16 / 6548.5:.3f} of HBM", flush=True)
    return out


if __name__ == "__main__":
    K = ts.K_VGA
    what = sys.argv[1:] or ["parity", "time"]
    if "time" in what:
        sc = ts.random_scenes(1024, K, 480, 640, seed=0)
        x = ts.render(sc, K, 480, 640, device="cuda").depth
        ks = ("strip", "f32", "f32masked")
        for w in what:
            if w.startswith("kernels="):
                ks = tuple(w.split("=")[1].split(","))
        for k in ks:
            timeit(K, "sobel", "median", k, x)
        for k in ks:
            timeit(K, "sobel", "mean", k, x)
        del x
    if "parity" in what:
        c1 = ts.render(ts.config1_scene(), K, 480, 640).depth.numpy()
        for f in ("fd", "sobel", "scharr", "prewitt"):
            for m in ("mean", "median"):
                check("cfg1", c1, K, f, m)
        r8 = ts.render(ts.random_scenes(8, K, 480, 640, seed=0), K, 480, 640, keep_depth64=True)
        for f in ("sobel", "fd"):
            for m in ("mean", "median"):
                check("random8", r8.depth.numpy(), K, f, m)
        check("random8-disp", ts.depth_to_disparity(r8.depth64, 500.0, 0.12).numpy(), K, "scharr", "median", disp=True)
        for n in [(0.4, -0.4 * (1 + 3e-4), -1.0), (1e-3, 5e-4, -1.0), (0.0, -0.3, -1.0), (0.3, 0.3, -1.0)]:
            z = ts.render(ts.plane_scene(n, (0, 0, 3.0)), K, 480, 640).depth.numpy()
            check(f"plane{n[:2]}", z, K, "sobel", "median")
        zh = ts.render(ts.random_scenes(2, ts.K_1080, 1080, 1920, seed=3, holes=True, salt=0.01), ts.K_1080, 1080,
                       1920).depth.numpy()
        check("holes1080", zh, ts.K_1080, "prewitt", "median")
        zn = ts.add_gaussian_noise(r8.depth[:2], ts.NOISE_PRESETS["high"], seed=5).numpy()
        check("noise-high", zn, K, "sobel", "median")
        z = r8.depth.numpy()[:2].copy()
        rng = np.random.default_rng(5)
        bad = np.array([0.0, -1.0, np.nan, np.inf, -np.inf, 1e-45, -0.0], np.float32)
        sel = rng.random(z.shape) < 0.15
        z[sel] = bad[rng.integers(0, len(bad), sel.sum())]
        check("invalid15%", z, K, "sobel", "median")
    if "prof" in what:
        kern = "f32"
        for w in what:
            if w.startswith("kernel="):
                kern = w.split("=")[1]
        sc = ts.random_scenes(256, K, 480, 640, seed=0)
        x = ts.render(sc, K, 480, 640, device="cuda").depth
        timeit(K, "sobel", "median", kern, x, reps=3)
