"""Adversarial check of the double-float (fp32 hi + lo) gradient idea (tools/numerics/df_emul.py): random 3x3
windows split by a line into two planes with a 1.1-3x depth ratio; angle of the normal from
double-float gradients vs exact fp64 gradients at the window centre.  DESIGN §12."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
import df_emul as de
f32 = np.float32
fl = de.fl
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
N = 400000
fx = 500.0
worst = 0
for rep in range(10):
    # window pixel coords relative to a random centre (u, v) in a VGA image
    uc = rng.uniform(-320, 320, N); vc = rng.uniform(-240, 240, N)
    du = np.array([-1, 0, 1])[None, None, :]; dv = np.array([-1, 0, 1])[None, :, None]
    U = (uc[:, None, None] + du) / fx; V = (vc[:, None, None] + dv) / fx
    def plane_depth():
        n = rng.normal(size=(N, 3)); n[:, 2] = -np.abs(n[:, 2]) - 0.05
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        d = rng.uniform(0.5, 5, N)
        # plane n.p = -d (p = Z (U, V, 1)) -> Z = -d / (n . (U, V, 1))
        den = n[:, 0, None, None] * U + n[:, 1, None, None] * V + n[:, 2, None, None]
        return -d[:, None, None] / den
    Z1 = plane_depth(); Z2 = Z1 * rng.uniform(1.1, 3.0, N)[:, None, None] * rng.choice([1, -1], N)[:, None, None] ** 0
    Z2 = np.where(rng.random(N)[:, None, None] < 0.5, Z1 * rng.uniform(1.1, 3.0, N)[:, None, None], plane_depth())
    # split line through the window: a u + b v > c
    a = rng.normal(size=N); b = rng.normal(size=N); c = rng.normal(scale=0.8, size=N)
    side = (a[:, None, None] * du + b[:, None, None] * dv) > c[:, None, None]
    Z = np.where(side, Z2, Z1)
    ok = (Z > 0.05).all(axis=(1, 2)) & (Z < 100).all(axis=(1, 2))
    Z = Z[ok].astype(np.float32); ucc = uc[ok]; vcc = vc[ok]
    n = Z.shape[0]
    z64 = Z.astype(np.float64)
    w = 1 / z64
    gu = (w[:, 0, 2] - w[:, 0, 0]) + 2 * (w[:, 1, 2] - w[:, 1, 0]) + (w[:, 2, 2] - w[:, 2, 0])
    gv = (w[:, 2, 0] - w[:, 0, 0]) + 2 * (w[:, 2, 1] - w[:, 0, 1]) + (w[:, 2, 2] - w[:, 0, 2])
    whi = fl(w); e = (-z64 * whi.astype(np.float64) + 1.0).astype(np.float32); wlo = fl(whi * e)
    def sob(A):
        dh = [fl(A[:, r, 2] - A[:, r, 0]) for r in range(3)]
        g_u = fl(fl(dh[0] + fl(f32(2) * dh[1])) + dh[2])
        dvv = [fl(A[:, 2, c2] - A[:, 0, c2]) for c2 in range(3)]
        g_v = fl(fl(dvv[0] + fl(f32(2) * dvv[1])) + dvv[2])
        return g_u, g_v
    guh, gvh = sob(whi); gul, gvl = sob(wlo)
    B = (fl(guh + gul), fl(gvh + gvl), fl(fl(guh + gvh) + fl(gul + gvl)), fl(fl(gvh - guh) + fl(gvl - gul)))
    E = (gu, gv, gu + gv, gv - gu)
    def fin(g):
        g_u, g_v, s, t = [np.asarray(x, np.float64) for x in g]
        zc = z64[:, 1, 1]
        nb = [(1, 0, g_u), (-1, 0, -g_u), (0, 1, g_v), (0, -1, -g_v), (1, 1, s), (-1, -1, -s), (-1, 1, t), (1, -1, -t)]
        cs = np.stack([m * z64[:, 1 + dv_, 1 + du_] / (z64[:, 1 + dv_, 1 + du_] - zc) for du_, dv_, m in nb])
        phi = np.median(cs, axis=0)
        nn = np.stack([fx * g_u, fx * g_v, -(ucc * g_u + vcc * g_v + phi)])
        nn /= np.linalg.norm(nn, axis=0)
        return np.where(phi < 0, -nn, nn), np.isfinite(cs).all(axis=0)
    nE, okE = fin(E); nB, _ = fin(B)
    err = np.degrees(np.arccos(np.clip((nE * nB).sum(0), -1, 1)))
    err = np.where(okE, err, 0)
    i = np.argmax(err)
    worst = max(worst, err[i])
    print(rep, n, 'max %.3e deg' % err[i], '>1e-4: %d  >3e-4: %d  >1e-3: %d' % ((err > 1e-4).sum(), (err > 3e-4).sum(), (err > 1e-3).sum()),
          'ratio %.2f' % (Z[i].max() / Z[i].min()))
print('worst', worst)
