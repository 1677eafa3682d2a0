"""Emulate (numpy, IEEE fp32 ops) a double-float (hi + lo fp32) evaluation of the Sobel
gradients g_u, g_v and the multipliers s = g_u + g_v, t = g_v - g_u, against the fp64 path the
strip kernel uses (w = 1/z in fp64, fp64 sums, rounded once to fp32), and measure the angle
difference each makes in the final normal (finish in fp64).  Exploration tool."""
import sys
import warnings
import numpy as np
warnings.filterwarnings('ignore')

sys.path.insert(0, '/root/repo')
import tfn_scenes as ts

f32 = np.float32


def fl(x):
    return x.astype(np.float32)


def fma32(a, b, c):      # exact fp32 fma: a*b exact in fp64, one rounding of a*b + c (c = +-1 here)
    return (a.astype(np.float64) * b.astype(np.float64) + c).astype(np.float32)


def grads_df(z, perturb=0):
    z = z.astype(np.float32)
    whi = fl(1.0 / z.astype(np.float64))
    if perturb:
        rng = np.random.default_rng(perturb)
        whi = np.nextafter(whi, np.where(rng.random(whi.shape) < 0.5, f32(0), f32(np.inf)))
    e = fma32(-z, whi, 1.0)
    wlo = fl(whi * e)

    def sob(a):   # a: (hi or lo) field -> (gu, gv) parts with the kernel's order
        dh = fl(a[:, 2:] - a[:, :-2])           # D_h(row, u) for u = 1..W-2
        gu = fl(fl(dh[:-2] + fl(f32(2) * dh[1:-1])) + dh[2:])
        dv = fl(a[2:] - a[:-2])                  # D_v(v, col)
        gv = fl(fl(dv[:, :-2] + fl(f32(2) * dv[:, 1:-1])) + dv[:, 2:])
        return gu, gv

    guh, gvh = sob(whi)
    gul, gvl = sob(wlo)
    gu = fl(guh + gul)
    gv = fl(gvh + gvl)
    s = fl(fl(guh + gvh) + fl(gul + gvl))
    t = fl(fl(gvh - guh) + fl(gvl - gul))
    return gu, gv, s, t


def grads_64(z):
    w = 1.0 / z.astype(np.float64)
    dh = w[:, 2:] - w[:, :-2]
    gu = (dh[:-2] + 2 * dh[1:-1]) + dh[2:]
    dv = w[2:] - w[:-2]
    gv = (dv[:, :-2] + 2 * dv[:, 1:-1]) + dv[:, 2:]
    return gu, gv, gu + gv, gv - gu


def finish(z, K, gu, gv, s, t):
    """fp64 finish (median of the 8 candidates, orientation, normalisation) on interior pixels"""
    z = z.astype(np.float64)
    H, W = z.shape
    zc = z[1:-1, 1:-1]
    gu, gv, s, t = [np.asarray(x, np.float64) for x in (gu, gv, s, t)]
    # neighbour offsets (du, dv) and their m = du*gu + dv*gv
    nb = [(1, 0, gu), (-1, 0, -gu), (0, 1, gv), (0, -1, -gv), (1, 1, s), (-1, -1, -s), (-1, 1, t), (1, -1, -t)]
    cands = []
    for du, dv, m in nb:
        zj = z[1 + dv:H - 1 + dv, 1 + du:W - 1 + du]
        with np.errstate(all='ignore'):
            cands.append(m * zj / (zj - zc))
    c = np.stack(cands)
    phi = np.median(c, axis=0)
    u = np.arange(1, W - 1)[None, :] - K.u0
    v = np.arange(1, H - 1)[:, None] - K.v0
    n = np.stack([K.fx * gu, K.fy * gv, -(u * gu + v * gv + phi)])
    n = n / np.linalg.norm(n, axis=0)
    n = np.where(phi < 0, -n, n)
    return n, np.isfinite(c).all(axis=0)


def angle(a, b):
    d = np.clip((a * b).sum(axis=0), -1, 1)
    return np.degrees(np.arccos(d))


def run(name, z, K, perturb=0, show=0):
    z = np.asarray(z)
    if z.ndim == 3:
        z = z[0]
    gu6, gv6, s6, t6 = grads_64(z)
    A = [fl(x) for x in (gu6, gv6, s6, t6)]
    B = grads_df(z, perturb)
    nE, ok = finish(z, K, gu6, gv6, s6, t6)
    nA, _ = finish(z, K, *A)
    nB, _ = finish(z, K, *B)
    m = ok & np.isfinite(nE).all(axis=0)
    eA, eB = angle(nA, nE)[m], angle(nB, nE)[m]
    rel = lambda x, y: np.abs(np.asarray(x, np.float64) - y) / np.maximum(np.abs(y), 1e-300)
    print(f"{name:28s} px {m.sum():8d}  fp64-path max {eA.max():.2e} deg  double-float max {eB.max():.2e} deg "
          f"(>1e-4: {(eB > 1e-4).sum()}, >1e-3: {(eB > 1e-3).sum()})  max rel err s {np.nanmax(rel(B[2], s6)[m]):.1e} "
          f"t {np.nanmax(rel(B[3], t6)[m]):.1e}")
    if show:
        eBf = np.where(m, angle(nB, nE), 0)
        for (v, u) in np.argwhere(eBf > 1e-4)[:show]:
            win = z[v:v + 3, u:u + 3]
            print("   px", v + 1, u + 1, "err %.2e" % eBf[v, u], "zmax/zmin %.3f" % (win.max() / win.min()),
                  "gu %.3e gv %.3e s %.3e t %.3e" % (gu6[v, u], gv6[v, u], s6[v, u], t6[v, u]),
                  "rel s %.1e t %.1e" % (rel(B[2], s6)[v, u], rel(B[3], t6)[v, u]))


def main():
    K = ts.K_VGA
    r = ts.render(ts.random_scenes(8, K, 480, 640, seed=0), K, 480, 640)
    for b in range(4):
        run(f"random scene {b}", r.depth[b].numpy(), K, show=8)
        run(f"random scene {b} (w_hi +-1ulp)", r.depth[b].numpy(), K, perturb=b + 1)
    for n in [(0.4, -0.4 * (1 + 3e-4), -1.0), (1e-3, 5e-4, -1.0), (0.0, -0.3, -1.0), (0.3, 0.3, -1.0)]:
        z = ts.render(ts.plane_scene(n, (0, 0, 3.0)), K, 480, 640).depth.numpy()
        run(f"plane {n}", z, K)
    c1 = ts.render(ts.config1_scene(), K, 480, 640).depth.numpy()
    run("config1 scene", c1 if c1.ndim == 2 else c1[0], K)
    for level in ("low", "high"):
        zn = ts.add_gaussian_noise(r.depth[:2], ts.NOISE_PRESETS[level], seed=5).numpy()
        run(f"noise {level}", zn[0], K)
    q = np.round(r.depth[0].numpy() * 1000) / 1000
    run("mm-quantized", q.astype(np.float32), K)


def occlusions():
    K = ts.K_VGA
    r = ts.render(ts.random_scenes(8, K, 480, 640, seed=0), K, 480, 640)
    for scale in (1e-3, 1.0, 3e3):
        z = r.depth.numpy()[:2].astype(np.float64) * scale
        rng = np.random.default_rng(int(scale * 1000) % 2**31)
        for _ in range(40):
            b, v, u = rng.integers(0, 2), rng.integers(0, 440), rng.integers(0, 600)
            h, w = rng.integers(3, 40), rng.integers(3, 40)
            z[b, v:v + h, u:u + w] *= rng.choice([0.01, 100.0])
        z = z.astype(np.float32)
        for b in range(2):
            run(f"occlusions x{scale} frame {b}", z[b], K, show=4)

if __name__ == "__main__":
    occlusions() if "occ" in sys.argv else main()
