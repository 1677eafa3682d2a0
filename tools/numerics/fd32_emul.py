"""Emulate (numpy, IEEE fp32) an fp32 evaluation of the FD gradients for the strip kernel:
g_u = (z_W - z_E) w_W w_E, g_v = (z_N - z_S) w_N w_S (one difference each: relative error a few
ulp, no cancellation), s = g_u + g_v and t = g_v - g_u re-paired along the diagonals,
s = (z_N - z_E) w_N w_E + (z_W - z_S) w_W w_S, t = (z_E - z_S) w_E w_S + (z_N - z_W) w_N w_W,
with a same-sign guard on each pair (mixed signs -> fp64 fallback for that pixel's s, t).
Measures the angle vs the exact fp64 gradients (fp64 finish) and the guard's firing rate per
pixel and per 128-pixel warp row.  Exploration tool."""
import sys
import warnings

import numpy as np

warnings.filterwarnings("ignore")
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import df_emul as de  # noqa: E402
import tfn_scenes as ts  # noqa: E402

fl = de.fl


def fd32(z, perturb=0, amp=None):
    z = z.astype(np.float32)
    w = fl(1.0 / z.astype(np.float64))
    if perturb:
        rng = np.random.default_rng(perturb)
        w = np.nextafter(w, np.where(rng.random(w.shape) < 0.5, np.float32(0), np.float32(np.inf)))
    C = (slice(1, -1), slice(1, -1))
    zE, zW, zN, zS = z[1:-1, 2:], z[1:-1, :-2], z[:-2, 1:-1], z[2:, 1:-1]
    wE, wW, wN, wS = w[1:-1, 2:], w[1:-1, :-2], w[:-2, 1:-1], w[2:, 1:-1]
    gu = fl(fl(zW - zE) * fl(wW * wE))
    gv = fl(fl(zN - zS) * fl(wN * wS))
    D1 = fl(fl(zN - zE) * fl(wN * wE)); D2 = fl(fl(zW - zS) * fl(wW * wS))
    D3 = fl(fl(zE - zS) * fl(wE * wS)); D4 = fl(fl(zN - zW) * fl(wN * wW))
    s = fl(D1 + D2); t = fl(D3 + D4)
    if amp is None:   # same-sign guard
        bad = (np.signbit(D1) != np.signbit(D2)) & (D1 != 0) & (D2 != 0)
        bad |= (np.signbit(D3) != np.signbit(D4)) & (D3 != 0) & (D4 != 0)
    else:             # amplification guard |D1| + |D2| <= amp |s|
        bad = (np.abs(D1) + np.abs(D2) > amp * np.abs(s)) | (np.abs(D3) + np.abs(D4) > amp * np.abs(t))
    return gu, gv, s, t, bad


def fd64(z):
    w = 1.0 / z.astype(np.float64)
    gu = w[1:-1, 2:] - w[1:-1, :-2]
    gv = w[2:, 1:-1] - w[:-2, 1:-1]
    return gu, gv, gu + gv, gv - gu


def run(name, z, K, perturb=0, amp=None):
    z = np.asarray(z)
    if z.ndim == 3:
        z = z[0]
    E = fd64(z)
    gu, gv, s, t, bad = fd32(z, perturb, amp)
    s6, t6 = E[2], E[3]
    # fallback: fp64 s, t (rounded to fp32) where the guard fires
    s = np.where(bad, fl(s6), s); t = np.where(bad, fl(t6), t)
    nE, ok = de.finish(z, K, *E)
    nB, _ = de.finish(z, K, gu, gv, s, t)
    m = ok & np.isfinite(nE).all(axis=0)
    err = np.where(m, de.angle(nB, nE), 0)
    H, W = bad.shape
    rows = np.pad(bad, ((0, 0), (0, (-W) % 128))).reshape(H, -1, 128).any(axis=2)
    print(f"{name:30s} max {err.max():.2e} deg  >1e-4: {(err > 1e-4).sum():4d}  guard px {bad[m].mean():.4f}  "
          f"warp-rows {rows.mean():.3f}")


if __name__ == "__main__":
    K = ts.K_VGA
    amp = float(sys.argv[1]) if len(sys.argv) > 1 else None
    r = ts.render(ts.random_scenes(8, K, 480, 640, seed=0), K, 480, 640)
    for b in range(4):
        run(f"random scene {b}", r.depth[b].numpy(), K, amp=amp)
    run("random scene 0 +-1ulp w", r.depth[0].numpy(), K, perturb=3, amp=amp)
    for n in [(0.4, -0.4 * (1 + 3e-4), -1.0), (1e-3, 5e-4, -1.0), (0.3, 0.3, -1.0)]:
        run(f"plane {n}", ts.render(ts.plane_scene(n, (0, 0, 3.0)), K, 480, 640).depth.numpy(), K, amp=amp)
    c1 = ts.render(ts.config1_scene(), K, 480, 640).depth.numpy()
    run("config1 scene", c1, K, amp=amp)
    zn = ts.add_gaussian_noise(r.depth[:1], ts.NOISE_PRESETS["high"], seed=5).numpy()
    run("noise high", zn, K, amp=amp)
