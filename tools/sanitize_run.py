"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck; one tool per run):
every kernel variant the library launches, on ragged frame sizes and odd strip heights —
strip kernel fast (register prefetch), masked and general (TMA ring), per-pixel, uint16 codes
(cp.async ring), fused point cloud, fp32 unit-step kernels (TMA ring + special-pixel queue),
stats and plane fit.  Prints one line per case; exits non-zero on a CUDA error."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import tfn_scenes as ts
import paper_2005_08165_b200 as tfn


def frames(n, H, W, holes=False, seed=1):
    K = ts.Intrinsics(200.0, 210.0, W / 2 - 0.3, H / 2 + 0.7)
    sc = ts.random_scenes(n, K, H, W, seed=seed, holes=holes, salt=0.02 if holes else 0.0)
    return K, ts.render(sc, K, H, W, device="cuda")


def main():
    cases = [(2, 33, 132), (1, 70, 260), (1, 31, 1024), (2, 48, 640), (1, 5, 8)]
    for (n, H, W) in cases:
        K, r = frames(n, H, W, holes=True)
        x = r.depth
        for kern in ("strip", "masked", "general", "pixel", "f32", "f32masked"):
            for mode in ("median", "mean"):
                for sh in (0, 5, 13):
                    est = tfn.Estimator(K, "sobel", mode, kernel=kern, strip_h=sh)
                    out = est.estimate(x)
                    torch.cuda.synchronize()
        est = tfn.Estimator(K, "fd", "median", kernel="strip", layout="packed")
        est.estimate(x)
        d = ts.depth_to_disparity(x.double(), 200.0, 0.1).float()
        tfn.Estimator(ts.Intrinsics(200.0, 200.0, K.u0, K.v0), "scharr", "median", kernel="f32").estimate_disparity(d, 20.0)
        codes = torch.round(x * 1000.0).clamp(0, 65535).to(torch.int32).to(torch.uint16)
        tfn.Estimator(K, "sobel", "median", out_dtype="f16").estimate(codes)
        tfn.Estimator(K, "prewitt", "median").estimate_points(x)
        out = tfn.Estimator(K, "sobel", "median").estimate(x)
        tfn.stats(out, r.gt)
        tfn.Estimator(K, "sobel", "median").plane_fit(x[:1], method="pca") if hasattr(tfn.Estimator, "plane_fit") else None
        torch.cuda.synchronize()
        print(f"ok {n}x{H}x{W}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
