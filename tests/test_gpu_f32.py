"""GPU parity of the fp32 unit-step kernels (TFN_OPT_KERNEL 5 = "f32", 6 = "f32masked",
tfn_f32.cuh) against the fp64 oracle, through the C ABI, on the same hard
cases as the round-1 kernels.  These kernels are NOT bit-identical to the others (their
gradients are fp32 3-term sums under a same-sign guard); each must meet the gate on its
own: identical invalid mask and <= 1e-3 deg per valid pixel.  Also: the
special-pixel count is small on clean scenes and large on noise (the guard works), and the
G = 1/2/4/8 frame shards of a config-5 stream give the same int64 statistics vector through
tfn_stats (SURVEY §4 "Distributed", §8(e))."""
import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts
from tests.parity import assert_parity, compare
from tests.test_gpu_parity import F_TC, FILTERS, MODES, _general_cases, run_gpu

pytestmark = pytest.mark.gpu
KERNELS = ("f32", "f32masked")


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def cfg1():
    return ts.render(ts.config1_scene(), ts.K_VGA, 480, 640, keep_depth64=True)


@pytest.fixture(scope="module")
def random8():
    return ts.render(ts.random_scenes(8, ts.K_VGA, 480, 640, seed=0), ts.K_VGA, 480, 640, keep_depth64=True)


def _check(tfn, s, K, f, m, disp=False, kernels=KERNELS, **kw):
    s = np.ascontiguousarray(s, dtype=np.float32)
    if s.ndim == 2:
        s = s[None]
    r = oracle.estimate(s, K, f, m, disparity=disp, f_tc=F_TC, threads=4)
    for k in kernels:
        g = run_gpu(tfn, s, K, f, m, disp=disp, kernel=k, **kw)
        res = compare(g, r, s, K)
        assert_parity(res, f"{k} {f}/{m}/{'disp' if disp else 'depth'} {kw}")


@pytest.mark.parametrize("f", FILTERS)
@pytest.mark.parametrize("m", MODES)
def test_f32_config1(tfn, cfg1, f, m):
    _check(tfn, cfg1.depth.numpy(), ts.K_VGA, f, m)


@pytest.mark.parametrize("m", MODES)
def test_f32_random_scenes_layouts(tfn, random8, m):
    for f in ("sobel", "fd", "scharr"):
        _check(tfn, random8.depth.numpy(), ts.K_VGA, f, m)
    _check(tfn, random8.depth.numpy()[:2], ts.K_VGA, "prewitt", m, layout="packed")


def test_f32_hard_cases(tfn, cfg1, random8):
    """skips, holes, invalid encodings, millimetre quantization, flat / apex, ragged sizes,
    disparity with holes — every case through both fp32 kernels"""
    for name, z, K, disp in _general_cases(cfg1, random8):
        for f in ("sobel", "fd"):
            for m in MODES:
                _check(tfn, z, K, f, m, disp=disp)


@pytest.mark.parametrize("n", [(0.4, -0.4 * (1 + 3e-4), -1.0), (1e-3, 5e-4, -1.0), (0.0, -0.3, -1.0),
                               (0.7, 0.0, -1.0), (0.3, 0.3, -1.0)])
def test_f32_adversarial_planes(tfn, n):
    """the near-diagonal isoline plane is exactly where round 1 needed fp64 (s = g_u + g_v
    cancels); here s is summed from diagonal differences and stays accurate"""
    z = ts.render(ts.plane_scene(n, (0, 0, 3.0)), ts.K_VGA, 480, 640).depth.numpy()
    for m in MODES:
        _check(tfn, z, ts.K_VGA, "sobel", m)


@pytest.mark.parametrize("scale", [1e-3, 1.0, 3e3])
def test_f32_extreme_scales_and_occlusions(tfn, random8, scale):
    z = random8.depth.numpy()[:2].astype(np.float64) * scale
    rng = np.random.default_rng(int(scale * 1000) % 2**31)
    for _ in range(40):
        b, v, u = rng.integers(0, 2), rng.integers(0, 440), rng.integers(0, 600)
        h, w = rng.integers(3, 40), rng.integers(3, 40)
        z[b, v:v + h, u:u + w] *= rng.choice([0.01, 100.0])
    z = z.astype(np.float32)
    for K in (ts.Intrinsics(500.0, 470.0, 321.3, 238.9), ts.Intrinsics(5.0, 5.0, 320.0, 240.0),
              ts.Intrinsics(5e4, 4.5e4, -100.0, 900.0)):
        for f in ("fd", "sobel"):
            for m in MODES:
                _check(tfn, z, K, f, m)


def test_f32_disparity_and_noise(tfn, random8):
    d = ts.depth_to_disparity(random8.depth64[:3], 500.0, 0.12).numpy()
    for f in ("fd", "scharr"):
        for m in MODES:
            _check(tfn, d, ts.K_VGA, f, m, disp=True)
    for level in ("low", "high"):
        z = ts.add_gaussian_noise(random8.depth[:2], ts.NOISE_PRESETS[level], seed=5).numpy()
        for f in FILTERS:
            _check(tfn, z, ts.K_VGA, f, "median")


def test_f32_special_rate(tfn, random8):
    """the guard sends < 2 % of clean-scene pixels to the exact path, and most pixels of
    noisy depth (where the fp32 multipliers are unreliable)"""
    from paper_2005_08165_b200 import tfn as T
    est = tfn.Estimator(ts.K_VGA, "sobel", "median", kernel="f32")
    T.tfn_set_option(est.h, T.OPT_COUNT_SPECIAL, 1)
    x = random8.depth.cuda()
    est.estimate(x)
    n_clean = T.tfn_debug_special_count(est.h)
    assert 0 <= n_clean < 0.02 * x.numel(), n_clean
    z = ts.add_gaussian_noise(random8.depth, ts.NOISE_PRESETS["high"], seed=5).cuda()
    est.estimate(z)
    n_noise = T.tfn_debug_special_count(est.h)
    assert n_noise > 0.5 * z.numel(), n_noise


def test_stats_identical_for_any_shard_count(tfn):
    """config 5 in miniature: 48 frames streamed in 8-frame chunks through estimate + tfn_stats
    as G = 1, 2, 4, 8 ranks would shard them (each rank's vector summed as the NCCL all-reduce
    does); every G gives the same int64 vector, bit for bit"""
    from paper_2005_08165_b200 import dist as tdist
    n, chunk = 48, 8
    K = ts.K_VGA
    est = tfn.Estimator(K, "sobel", "median")
    vecs = {}
    for G in (1, 2, 4, 8):
        total = torch.zeros(8, dtype=torch.int64)
        for r in range(G):
            lo, hi = tdist.shard(n, r, G)
            acc = torch.zeros(8, dtype=torch.int64, device="cuda")
            for a, b in tdist.chunks(lo, hi, chunk):
                rr = ts.render(ts.random_scenes(b - a, K, 480, 640, seed=0, first_frame=a), K, 480, 640, device="cuda")
                out = est.estimate(rr.depth)
                tfn.stats(out, rr.gt, acc=acc)
            torch.cuda.synchronize()
            total += acc.cpu()
        vecs[G] = total.tolist()
    assert vecs[1][7] == n * 480 * 640
    assert vecs[1] == vecs[2] == vecs[4] == vecs[8], vecs


def test_no_writes_outside_buffers(tfn):
    """every kernel variant writes exactly its output (and point-cloud) buffer: both sit inside
    larger allocations whose margins hold a canary pattern that must survive (ragged widths,
    odd strip heights, holes).  With compute-sanitizer closed on the GPU pool this, the
    bounds-checked build (TFN_BOUNDS_CHECK) and the ring-stress build carry the memory-safety
    evidence."""
    canary = -12345.678
    for (n, H, W) in ((2, 33, 132), (1, 70, 260), (1, 31, 1024), (3, 5, 8)):
        K = ts.Intrinsics(200.0, 210.0, W / 2 - 0.3, H / 2 + 0.7)
        x = ts.render(ts.random_scenes(n, K, H, W, seed=4, holes=True, salt=0.02), K, H, W, device="cuda").depth
        pad = 4096
        for kern in ("strip", "masked", "general", "pixel", "f32", "f32masked"):
            for layout in ("planar", "packed"):
                for sh in (0, 5):
                    est = tfn.Estimator(K, "sobel", "median", kernel=kern, layout=layout, strip_h=sh)
                    buf = torch.full((n * 3 * H * W + 2 * pad,), canary, device="cuda")
                    shape = (n, 3, H, W) if layout == "planar" else (n, H, W, 3)
                    out = buf[pad:pad + n * 3 * H * W].view(shape)
                    est.estimate(x, out=out)
                    torch.cuda.synchronize()
                    assert (buf[:pad] == canary).all() and (buf[-pad:] == canary).all(), (kern, layout, sh, H, W)
                    assert not (out == canary).any(), (kern, layout, sh, H, W)     # every pixel written
        est = tfn.Estimator(K, "prewitt", "median")
        buf = torch.full((2 * n * 3 * H * W + 3 * pad,), canary, device="cuda")
        nrm = buf[pad:pad + n * 3 * H * W].view(n, 3, H, W)
        pts = buf[2 * pad + n * 3 * H * W:2 * pad + 2 * n * 3 * H * W].view(n, 3, H, W)
        est.estimate_points(x, out=nrm, points=pts)
        torch.cuda.synchronize()
        assert (buf[:pad] == canary).all() and (buf[pad + n * 3 * H * W:2 * pad + n * 3 * H * W] == canary).all()
        assert (buf[-pad:] == canary).all()
