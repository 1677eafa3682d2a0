"""Oracle pins, part 1: every component of the oracle against values printed in
the paper or in SPEC (tests/golden/spec_examples.json, each entry cited), plus
closed-form checks of the individual steps.  Pin P7 of SURVEY.md §8(c)."""
import math

import numpy as np
import pytest

import oracle
from oracle import metrics


def test_backproject_examples(golden):
    for ex in golden["backproject"]:
        p = oracle.backproject(ex["K"], *ex["uvz"])
        np.testing.assert_allclose(p, ex["p"], rtol=0, atol=1e-15, err_msg=ex["cite"])


def test_backproject_roundtrip_eq13():
    # Eq. 13: z [u v 1]^T = K p  — projecting the back-projected point recovers (u,v,z)
    rng = np.random.default_rng(0)
    for _ in range(200):
        K = (rng.uniform(50, 2000), rng.uniform(50, 2000), rng.uniform(0, 640), rng.uniform(0, 480))
        u, v, z = rng.uniform(-100, 800), rng.uniform(-100, 600), rng.uniform(0.1, 50)
        p = oracle.backproject(K, u, v, z)
        assert p[2] == z
        assert abs(K[0] * p[0] / p[2] + K[2] - u) <= 1e-9 * max(1, abs(u))
        assert abs(K[1] * p[1] / p[2] + K[3] - v) <= 1e-9 * max(1, abs(v))


def test_inverse_depth_and_validity(golden):
    for ex in golden["inverse_depth"]:
        assert oracle.inverse_depth(ex["z"]) == ex["x"], ex["cite"]
    for z in golden["invalid_samples"]["values"]:
        assert not oracle.valid_sample(float(z)), z
    for z in (1.1754943508222875e-38, 1e-3, 2.0, 3.0e38):
        assert oracle.valid_sample(z)


def test_disparity_to_depth(golden):
    for ex in golden["disparity_to_depth"]:
        assert abs(oracle.disparity_to_depth(ex["f"] * ex["tc"], ex["d"]) - ex["z"]) < 1e-12, ex["cite"]


def test_orientation(golden):
    for ex in golden["orient"]:
        np.testing.assert_allclose(oracle.orient_toward_camera(ex["n"], ex["p"]), ex["out"],
                                   atol=1e-15, err_msg=ex["cite"])
    # idempotent and camera-facing
    rng = np.random.default_rng(1)
    for _ in range(100):
        n, p = rng.normal(size=3), rng.normal(size=3)
        p[2] = abs(p[2]) + 0.1
        a = oracle.orient_toward_camera(n, p)
        b = oracle.orient_toward_camera(a, p)
        np.testing.assert_allclose(a, b, rtol=0, atol=4e-16)   # idempotent up to renormalisation rounding
        assert float(a @ p) <= 0.0


def test_filter_weights_q1():
    assert oracle.weights("fd") == (0.0, 1.0)
    assert oracle.weights("sobel") == (1.0, 2.0)
    assert oracle.weights("scharr") == (3.0, 10.0)
    assert oracle.weights("prewitt") == (1.0, 1.0)


def test_gradient_examples(golden):
    H, W = 5, 6
    u = np.arange(W, dtype=float)[None, :].repeat(H, 0)
    v = np.arange(H, dtype=float)[:, None].repeat(W, 1)
    gu, gv = oracle.gradient_at(u, 2, 2, "sobel")
    assert gu == 8.0 and gv == 0.0
    row = np.array([[0.2, 0.4, 0.7]] * 3)
    gu, _ = oracle.gradient_at(row, 1, 1, "fd")
    assert abs(gu - 0.5) < 1e-15
    aff = 0.1 * u + 0.05 * v + 0.3
    for vv in range(1, H - 1):
        for uu in range(1, W - 1):
            gu, gv = oracle.gradient_at(aff, vv, uu, "fd")
            assert abs(gu - 0.2) < 1e-14 and abs(gv - 0.1) < 1e-14


@pytest.mark.parametrize("filt,scale", [("fd", 2), ("sobel", 8), ("scharr", 32), ("prewitt", 6)])
def test_gradient_kernel_exact_on_affine(filt, scale):
    # each kernel gives s*(alpha,beta) on any affine image; s = 2(2kp+k0)
    rng = np.random.default_rng(2)
    a, b, c = rng.normal(size=3)
    H, W = 7, 9
    img = a * np.arange(W)[None, :] + b * np.arange(H)[:, None] + c
    gu, gv = oracle.gradient_at(img, 3, 4, filt)
    assert abs(gu - scale * a) < 1e-12 and abs(gv - scale * b) < 1e-12


def test_gradient_transpose_symmetry():
    rng = np.random.default_rng(3)
    img = rng.normal(size=(6, 7))
    for f in ("fd", "sobel", "scharr", "prewitt"):
        gu, gv = oracle.gradient_at(img, 2, 3, f)
        tu, tv = oracle.gradient_at(img.T.copy(), 3, 2, f)
        assert gu == tv and gv == tu


def test_aggregate_examples(golden):
    for ex in golden["aggregate"]:
        assert oracle.aggregate(ex["values"], ex["mode"]) == ex["out"], ex["cite"]


def test_median_brute_force():
    # median == middle order statistic(s) of the sorted list, for k = 1..8
    rng = np.random.default_rng(4)
    for _ in range(500):
        k = int(rng.integers(1, 9))
        x = rng.normal(size=k) * 10.0 ** int(rng.integers(-3, 4))
        assert oracle.aggregate(x, "median") == np.median(x)
        assert abs(oracle.aggregate(x, "mean") - x.mean()) <= 1e-12 * np.abs(x).sum()


def test_nz_candidate_examples(golden):
    for ex in golden["nz_candidate"]:
        assert oracle.nz_candidate([0, 0, 0], ex["delta"], ex["nx"], ex["ny"]) == ex["out"], ex["cite"]


def test_metrics_examples(golden):
    for ex in golden["angular_error"]:
        assert abs(metrics.angular_error_deg(ex["a"], ex["b"]) - ex["deg"]) < 1e-12, ex["cite"]
    for ex in golden["aae"]:
        assert metrics.aae(ex["psi"]) == ex["out"]
    for ex in golden["pgp"]:
        assert abs(metrics.pgp(ex["psi"], ex["phi"]) - ex["out"]) < 1e-15, ex["cite"]
    for row in golden["pi_table3"]["rows"]:
        for ea, pi in zip(row["e_A"], row["pi"]):
            assert abs(metrics.pi_score(ea, row["t"]) - pi) <= 0.005 * (row["t"] + ea), row["cite"]


def test_angular_error_small_angles():
    # Q16: atan2 form resolves 1e-3 degree; arccos in fp64 cannot below ~1e-6 deg
    for deg in (1e-3, 1e-5, 0.1, 45.0, 179.9):
        t = math.radians(deg)
        a = [1.0, 0.0, 0.0]
        b = [math.cos(t), math.sin(t), 0.0]
        assert abs(metrics.angular_error_deg(a, b) - deg) < 1e-10 * max(1.0, deg)


def test_pgp_monotone():
    rng = np.random.default_rng(5)
    psi = rng.uniform(0, 180, size=1000)
    vals = [metrics.pgp(psi, phi) for phi in np.linspace(0, 180, 50)]
    assert all(b >= a for a, b in zip(vals, vals[1:])) and vals[-1] == 1.0


def test_backproject_image_pins():
    """N3 oracle: every valid pixel's point satisfies Eq. 13's closed form X/Z = (u-u0)/fx,
    Y/Z = (v-v0)/fy and, for a rendered plane, lies on that plane (n . p = n . q within
    1e-9 m); invalid samples give NaN; the SPEC example point is reproduced."""
    import oracle
    import tfn_scenes as ts
    K = ts.Intrinsics(510.0, 490.0, 31.7, 22.3)
    n, q = np.array([0.3, -0.2, -1.0]), np.array([0.0, 0.0, 3.0])
    r = ts.render(ts.plane_scene(tuple(n), tuple(q)), K, 48, 64, keep_depth64=True)
    z = r.depth64.numpy().copy()
    z[0, 5, 7] = 0.0
    z[0, 9, 9] = np.nan
    p = oracle.backproject_image(z, K)
    assert p.shape == (1, 3, 48, 64)
    assert np.isnan(p[0, :, 5, 7]).all() and np.isnan(p[0, :, 9, 9]).all()
    ok = np.isfinite(z[0]) & (z[0] >= np.finfo(np.float32).tiny)
    assert np.isnan(p[0, 0][~ok]).all()
    vv, uu = np.nonzero(ok)
    X, Y, Z = p[0, 0][ok], p[0, 1][ok], p[0, 2][ok]
    assert np.array_equal(Z, z[0][ok])
    assert np.allclose(X / Z, (uu - K.u0) / K.fx, rtol=0, atol=1e-12)
    assert np.allclose(Y / Z, (vv - K.v0) / K.fy, rtol=0, atol=1e-12)
    nn = n / np.linalg.norm(n)
    assert np.abs(nn[0] * X + nn[1] * Y + nn[2] * Z - nn @ q).max() < 1e-9
def test_backproject_image_spec_examples(golden):
    """the SPEC back-projection examples through the image routine"""
    import oracle
    for ex in golden["backproject"]:
        u, v, zval = ex["uvz"]
        z = np.zeros((1, v + 1, u + 1))
        z[0, v, u] = zval
        p = oracle.backproject_image(z, tuple(ex["K"]))
        assert np.allclose(p[0, :, v, u], ex["p"], rtol=0, atol=1e-12), ex["cite"]
