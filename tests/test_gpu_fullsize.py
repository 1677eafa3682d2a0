"""BASELINE.json configs at full size, in the launch configuration bench.py times (one
launch over the whole batch, default strip geometry, AUTO variant selection after the
bench's warm-up calls), checked against the fp64 oracle on whole frames and on sampled
pixels (the oracle finishes those in seconds).  configs[1] is in test_gpu_parity.py; this
file covers configs[2] (disparity), configs[3] (1080p holes: AUTO -> masked variant), the N1
workload (uint16 codes -> half normals) and the FD launch configurations (16 warps/SM)."""
import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts
from oracle import metrics
from tests.parity import TOL_DEG, assert_parity, compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

F, B_ = 500.0, 0.12
# half normals: each component rounded to nearest half (relative error <= 2^-11), so the
# direction moves by at most ~ sqrt(3) * 2^-11 rad = 0.049 deg on top of the fp32 parity bar
TOL_F16_DEG = TOL_DEG + 0.049


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


def render_gpu(sc, K, H, W, n, chunk=128, disp=False):
    out = []
    for lo in range(0, n, chunk):
        r = ts.render(sc.subset(lo, min(n, lo + chunk)), K, H, W, device="cuda", keep_depth64=disp)
        out.append(ts.depth_to_disparity(r.depth64, F, B_) if disp else r.depth)
    return torch.cat(out)


def sampled(g, frame, K, f, m, rng, n=2000, disp=False, tol=TOL_DEG):
    H, W = frame.shape
    pix = [tuple(p) for p in rng.integers(0, (H, W), size=(n, 2))] + [(0, 0), (H - 1, W - 1), (1, 1)]
    r = oracle.estimate_pixels(frame, K, pix, f, m, disparity=disp, f_tc=F * B_)
    gg = np.stack([g[:, v, u] for v, u in pix]).astype(np.float64)
    okg, okr = np.all(np.isfinite(gg), 1), np.all(np.isfinite(r), 1)
    assert np.array_equal(okg, okr)
    if not okr.any():
        return
    fx, fy, u0, v0 = K.as_tuple()
    p = np.array([[(u - u0) / fx, (v - v0) / fy, 1.0] for v, u in pix])[okr]
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    a = metrics.angular_error_deg(gg[okr], r[okr])
    tie = np.abs(np.sum(r[okr] * p, 1)) < 1e-6
    a = np.where(tie, np.minimum(a, metrics.angular_error_deg(-gg[okr], r[okr])), a)
    assert a.max() <= tol, a.max()


def warm(est, call, n=5):
    """the bench's warm-up calls; synchronised one by one so that AUTO's asynchronous
    special-rate read-back (a pinned word + event) is visible to the next call"""
    for _ in range(n):
        call()
        torch.cuda.synchronize()


def test_full_size_config3_disparity(tfn):
    n, H, W = 1024, 480, 640
    sc = ts.random_scenes(n, ts.K_VGA, H, W, seed=0)
    d = render_gpu(sc, ts.K_VGA, H, W, n, disp=True)
    est = tfn.Estimator(ts.K_VGA, "scharr", "median")
    warm(est, lambda: est.estimate_disparity(d, F * B_))
    out = est.estimate_disparity(d, F * B_).cpu().numpy()
    rng = np.random.default_rng(3)
    for i, fi in enumerate((0, 513, 1023)):
        r = ts.render(sc.subset(fi, fi + 1), ts.K_VGA, H, W, keep_depth64=True)
        frame = ts.depth_to_disparity(r.depth64, F, B_)[0].numpy()
        assert np.array_equal(frame, d[fi].cpu().numpy())
        if i == 0:
            ref = oracle.estimate(frame, ts.K_VGA, "scharr", "median", disparity=True, f_tc=F * B_)
            assert_parity(compare(out[fi][None], ref[None], frame[None], ts.K_VGA), "config 3 frame 0")
        else:
            sampled(out[fi], frame, ts.K_VGA, "scharr", "median", rng, disp=True)


def test_full_size_config4_holes_auto_masked(tfn):
    from paper_2005_08165_b200 import tfn as T
    n, H, W = 128, 1080, 1920
    sc = ts.random_scenes(n, ts.K_1080, H, W, seed=0, holes=True, salt=0.01)
    z = render_gpu(sc, ts.K_1080, H, W, n, chunk=16)
    est = tfn.Estimator(ts.K_1080, "prewitt", "median")
    warm(est, lambda: est.estimate(z), n=8)
    assert T.tfn_auto_variant(est.h) == 4           # the bench launch runs the masked variant
    out = est.estimate(z).cpu().numpy()
    rng = np.random.default_rng(4)
    for i, fi in enumerate((0, 64, 127)):
        frame = ts.render(sc.subset(fi, fi + 1), ts.K_1080, H, W).depth[0].numpy()
        assert np.array_equal(frame, z[fi].cpu().numpy())
        if i == 0:
            ref = oracle.estimate(frame, ts.K_1080, "prewitt", "median", threads=8)
            assert_parity(compare(out[fi][None], ref[None], frame[None], ts.K_1080), "config 4 frame 0")
        else:
            sampled(out[fi], frame, ts.K_1080, "prewitt", "median", rng)


def test_full_size_config6_u16_half(tfn):
    n, H, W = 1024, 480, 640
    sc = ts.random_scenes(n, ts.K_VGA, H, W, seed=0)
    z = render_gpu(sc, ts.K_VGA, H, W, n)
    codes = torch.where(torch.isfinite(z) & (z > 0), torch.round(z * 1000.0), torch.zeros_like(z))
    codes = codes.clamp(0, 65535).to(torch.int32).to(torch.uint16)
    est = tfn.Estimator(ts.K_VGA, "sobel", "median", out_dtype="f16")
    warm(est, lambda: est.estimate(codes, depth_scale=1e-3))
    out = est.estimate(codes, depth_scale=1e-3).cpu().float().numpy()
    for fi in (0, 1023):
        z64 = codes[fi].cpu().to(torch.int32).numpy().astype(np.float64) * 1e-3
        ref = oracle.estimate(z64, ts.K_VGA, "sobel", "median")
        res = compare(out[fi][None], ref[None], z64[None], ts.K_VGA, tol=TOL_F16_DEG)
        assert res["mask_equal"] and res["n_bad"] == 0, res


@pytest.mark.parametrize("m,disp", [("mean", False), ("median", False), ("mean", True)])
def test_full_size_fd_16_warps(tfn, m, disp):
    """FD at full configs[1] / configs[2] size in the launch configuration bench.py times for
    `--filter fd` (round 2: 16 warps/SM; FD + median through the TMA ring; disparity FD + mean
    with fp32 gradients): one whole frame against the oracle, sampled pixels on two
    more"""
    n, H, W = 1024, 480, 640
    sc = ts.random_scenes(n, ts.K_VGA, H, W, seed=0)
    x = render_gpu(sc, ts.K_VGA, H, W, n, disp=disp)
    est = tfn.Estimator(ts.K_VGA, "fd", m)
    call = (lambda: est.estimate_disparity(x, F * B_)) if disp else (lambda: est.estimate(x))
    warm(est, call)
    out = call().cpu().numpy()
    rng = np.random.default_rng(5)
    for i, fi in enumerate((0, 511, 1023)):
        r = ts.render(sc.subset(fi, fi + 1), ts.K_VGA, H, W, keep_depth64=disp)
        frame = (ts.depth_to_disparity(r.depth64, F, B_) if disp else r.depth)[0].numpy()
        assert np.array_equal(frame, x[fi].cpu().numpy())
        if i == 0:
            ref = oracle.estimate(frame, ts.K_VGA, "fd", m, disparity=disp, f_tc=F * B_, threads=8)
            assert_parity(compare(out[fi][None], ref[None], frame[None], ts.K_VGA), f"fd/{m}/disp={disp} frame 0")
        else:
            sampled(out[fi], frame, ts.K_VGA, "fd", m, rng, disp=disp)
