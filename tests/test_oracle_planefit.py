"""N4 oracle (oracle.plane_fit / smallest_eigvec_sym): PlanePCA (Eq. 3) and PlaneSVD
(Eq. 2) pinned to SPEC S:251-280's examples, closed forms and a brute-force SVD."""
import math

import numpy as np
import pytest

import oracle
import tfn_scenes as ts

METHODS = ("pca", "svd")


def _ang(a, b):
    a = np.moveaxis(a, 0, -1) if a.ndim == 3 else a
    b = np.moveaxis(b, 0, -1) if b.ndim == 3 else b
    c = np.linalg.norm(np.cross(a, b), axis=-1)
    return np.degrees(np.arctan2(c, np.sum(a * b, axis=-1)))


def test_eigvec_spec_examples():
    """diag(1,2,3) -> [1,0,0]; identity -> [1,0,0] by the tie-break; the null
    vector of a sum of v v^T over 20 random unit vectors orthogonal to n -> +-n (1e-8)"""
    assert np.allclose(oracle.smallest_eigvec_sym(np.diag([1.0, 2.0, 3.0])), [1, 0, 0], atol=1e-15)
    assert np.allclose(oracle.smallest_eigvec_sym(np.diag([3.0, 1.0, 2.0])), [0, 1, 0], atol=1e-15)
    assert np.array_equal(oracle.smallest_eigvec_sym(np.eye(3)), [1.0, 0.0, 0.0])
    rng = np.random.default_rng(0)
    for d in (3, 4):
        for _ in range(20):
            n = rng.normal(size=d); n /= np.linalg.norm(n)
            M = np.zeros((d, d))
            for _ in range(20):
                x = rng.normal(size=d); x -= (x @ n) * n; x /= np.linalg.norm(x)
                M += np.outer(x, x)
            e = oracle.smallest_eigvec_sym(M)
            assert min(np.linalg.norm(e - n), np.linalg.norm(e + n)) < 1e-8
    with pytest.raises(ValueError):
        oracle.smallest_eigvec_sym(np.array([[1.0, 2.0, 0], [0, 1, 0], [0, 0, 1]]))


def test_eigvec_matches_brute_force_eigh():
    """against numpy's LAPACK eigh on random symmetric 3x3 / 4x4 (distinct eigenvalues)"""
    rng = np.random.default_rng(1)
    for d in (3, 4):
        for _ in range(200):
            A = rng.normal(size=(d, d)); M = A @ A.T
            w, V = np.linalg.eigh(M)
            e = oracle.smallest_eigvec_sym(M)
            assert min(np.linalg.norm(e - V[:, 0]), np.linalg.norm(e + V[:, 0])) < 1e-9


@pytest.mark.parametrize("m", METHODS)
def test_spec_shared_examples(m, golden):
    """S:248-250 shared estimator examples: slanted plane fixture -> [-0.7071, 0, -0.7071]
    within 0.01 deg at interior pixels; constant depth -> [0,0,-1] within 1e-6 deg;
    on-axis sphere, principal-point pixel -> [0,0,-1] within 0.1 deg"""
    K = ts.Intrinsics(1.0, 1.0, 0.0, 0.0)
    # the SPEC fixture plane x + z = 2: z = 2 / (1 + u) with K = (1,1,0,0)
    H, W = 6, 6
    u = np.arange(W, dtype=np.float64)[None, :].repeat(H, 0)
    z = 2.0 / (1.0 + u)
    n = oracle.plane_fit(z, K, m)[0]
    inner = n[:, 1:-1, 1:-1].reshape(3, -1).T
    ref = np.array([-1.0, 0.0, -1.0]) / math.sqrt(2.0)
    assert _ang(inner, np.broadcast_to(ref, inner.shape)).max() < 0.01
    zc = np.full((8, 9), 2.5)
    n = oracle.plane_fit(zc, ts.K_VGA, m)[0]
    inner = n[:, 1:-1, 1:-1].reshape(3, -1).T
    assert _ang(inner, np.broadcast_to([0, 0, -1.0], inner.shape)).max() < 1e-6
    Ks = ts.Intrinsics(500.0, 500.0, 320.0, 240.0)
    zs = ts.render(ts.sphere_scene((0, 0, 3), 1.0), Ks, 480, 644, keep_depth64=True).depth64.numpy()
    n = oracle.plane_fit(zs[:, 236:245, 316:325], ts.Intrinsics(500.0, 500.0, 4.0, 4.0), m)[0]
    assert _ang(n[:, 4, 4][None], np.array([[0, 0, -1.0]]))[0] < 0.1


@pytest.mark.parametrize("m", METHODS)
def test_tilted_planes_exact_and_validity(m):
    """Eq. 1: on an exact plane both fits return its camera-facing normal (<= 1e-9 deg);
    border, invalid centres and k < 3 give NaN"""
    K = ts.Intrinsics(60.0, 55.0, 31.5, 23.25)
    rng = np.random.default_rng(7)
    for _ in range(3):
        t, a = rng.uniform(0.1, 1.0), rng.uniform(0, 2 * math.pi)
        n_true = np.array([math.sin(t) * math.cos(a), math.sin(t) * math.sin(a), -math.cos(t)])
        z = ts.render(ts.plane_scene(n_true, (0, 0, rng.uniform(2, 5))), K, 48, 64, keep_depth64=True).depth64.numpy()
        z[0, 10, 10] = 0.0                        # invalid centre
        z[0, 20:23, 30:33] = 0.0; z[0, 21, 31] = 3.0   # isolated: k = 0
        n = oracle.plane_fit(z, K, m)[0]
        ok = np.all(np.isfinite(n), 0)
        assert not ok[0].any() and not ok[:, 0].any() and not ok[10, 10] and not ok[21, 31]
        err = _ang(n, np.broadcast_to(n_true[:, None, None], n.shape))[ok]
        assert err.max() < 1e-9


def test_plane_svd_matches_brute_force_svd():
    """Eq. 2 literally: numpy SVD of [Q+ 1] on random curved neighbourhoods agrees with the
    oracle's PlaneSVD (1e-6 deg); PlanePCA with numpy's SVD of the centred Q+ (Eq. 3, 1e-8)"""
    K = ts.Intrinsics(500.0, 500.0, 320.0, 240.0)
    sc = ts.random_scenes(1, K, 480, 640, seed=5)
    z = ts.render(sc, K, 480, 640, keep_depth64=True).depth64.numpy()[0]
    rng = np.random.default_rng(2)
    for _ in range(150):
        v, u = rng.integers(1, 479), rng.integers(1, 639)
        win = z[v - 1:v + 2, u - 1:u + 2]
        if not np.all(win > 0):
            continue
        Kw = ts.Intrinsics(K.fx, K.fy, K.u0 - (u - 1), K.v0 - (v - 1))
        pts = np.array([[(uu - Kw.u0) * win[vv, uu] / Kw.fx, (vv - Kw.v0) * win[vv, uu] / Kw.fy, win[vv, uu]]
                        for vv in range(3) for uu in range(3)])
        p = pts[4]
        for m in METHODS:
            if m == "svd":
                A = np.hstack([pts, np.ones((9, 1))])
                nn = np.linalg.svd(A)[2][-1][:3]
            else:
                nn = np.linalg.svd(pts - pts.mean(0))[2][-1]
            nn = nn / np.linalg.norm(nn)
            if nn @ p > 0:
                nn = -nn
            got = oracle.plane_fit(win, Kw, m)[0][:, 1, 1]
            # PlaneSVD goes through the 4x4 normal matrix, which squares the
            # condition number of [Q+ 1]: allow 1e-6 deg there, 1e-8 deg for PlanePCA
            assert _ang(got[None], nn[None])[0] < (1e-6 if m == "svd" else 1e-8), (m, v, u)
