"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element, on seeded synthetic inputs (SURVEY.md §8(c) gate: identical invalid mask,
<= 1e-3 deg per valid pixel).  Also: strip kernel == per-pixel kernel bit for bit,
layouts, host-buffer path, edge inputs, the Phi probe (P8), the stats kernel (a8),
and sampled parity at BASELINE.json's full config-2 size in the bench launch config.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts
from oracle import metrics
from tests.parity import TOL_DEG, assert_kernels_agree, assert_parity, compare, fd32_variant, planar

pytestmark = pytest.mark.gpu

FILTERS = ("fd", "sobel", "scharr", "prewitt")
MODES = ("mean", "median")
F_TC = 500.0 * 0.12


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


def run_gpu(tfn, sample, K, f, m, disp=False, layout="planar", kernel="auto", **kw):
    est = tfn.Estimator(K, filter=f, nz_mode=m, layout=layout, kernel=kernel, **kw)
    x = torch.as_tensor(np.ascontiguousarray(sample, dtype=np.float32)).cuda()
    if x.dim() == 2:
        x = x[None]
    out = est.estimate_disparity(x, F_TC) if disp else est.estimate(x)
    torch.cuda.synchronize()
    return planar(out.cpu().numpy(), layout)


def check(tfn, sample, K, f, m, disp=False, **kw):
    s = np.ascontiguousarray(sample, dtype=np.float32)
    if s.ndim == 2:
        s = s[None]
    g = run_gpu(tfn, s, K, f, m, disp=disp, **kw)
    r = oracle.estimate(s, K, f, m, disparity=disp, f_tc=F_TC, threads=4)
    res = compare(g, r, s, K)
    assert_parity(res, f"{f}/{m}/{'disp' if disp else 'depth'} {kw}")
    return g, res


# ------------------------------------------------------------------ config 1 (configs[0])
@pytest.fixture(scope="module")
def cfg1():
    return ts.render(ts.config1_scene(), ts.K_VGA, 480, 640, keep_depth64=True)


@pytest.mark.parametrize("f", FILTERS)
@pytest.mark.parametrize("m", MODES)
def test_config1_parity_and_kernels_bitwise(tfn, cfg1, f, m):
    z = cfg1.depth.numpy()
    g_strip, res = check(tfn, z, ts.K_VGA, f, m, kernel="strip")
    g_pix = run_gpu(tfn, z, ts.K_VGA, f, m, kernel="pixel")
    assert np.array_equal(g_strip.view(np.uint32), g_pix.view(np.uint32)), "strip != pixel kernel"
    assert res["n_valid"] > 290000


def test_layouts_and_strip_heights_bitwise(tfn, cfg1):
    z = cfg1.depth.numpy()
    base = run_gpu(tfn, z, ts.K_VGA, "sobel", "median")
    for layout in ("packed",):
        assert np.array_equal(base.view(np.uint32), run_gpu(tfn, z, ts.K_VGA, "sobel", "median", layout=layout).view(np.uint32))
    for sh in (1, 3, 7, 32, 480, 1000):
        g = run_gpu(tfn, z, ts.K_VGA, "sobel", "median", kernel="strip", strip_h=sh)
        assert np.array_equal(base.view(np.uint32), g.view(np.uint32)), sh
    g = run_gpu(tfn, z, ts.K_VGA, "sobel", "median", kernel="strip", grid=1)
    assert np.array_equal(base.view(np.uint32), g.view(np.uint32))


# ------------------------------------------------------------------ configs 2 / 3 / 4 (small)
@pytest.fixture(scope="module")
def random8():
    sc = ts.random_scenes(8, ts.K_VGA, 480, 640, seed=123)
    return ts.render(sc, ts.K_VGA, 480, 640, keep_depth64=True)


@pytest.mark.parametrize("f", FILTERS)
@pytest.mark.parametrize("m", MODES)
def test_random_scenes_parity(tfn, random8, f, m):
    check(tfn, random8.depth.numpy(), ts.K_VGA, f, m)


@pytest.mark.parametrize("f", ("fd", "scharr"))
@pytest.mark.parametrize("m", MODES)
def test_disparity_parity(tfn, random8, f, m):
    d = ts.depth_to_disparity(random8.depth64, 500.0, 0.12).numpy()
    g, _ = check(tfn, d, ts.K_VGA, f, m, disp=True)
    # depth path and disparity path agree (Eq. 20) on pixels valid in both
    z = random8.depth.numpy()
    gz = run_gpu(tfn, z, ts.K_VGA, f, m)
    ok = np.all(np.isfinite(g), 1) & np.all(np.isfinite(gz), 1)
    a = metrics.angular_error_deg(np.moveaxis(g, 1, -1)[ok], np.moveaxis(gz, 1, -1)[ok])
    assert np.percentile(a, 99) < 0.05


def test_disparity_baseline_cancels(tfn, random8):
    d = ts.depth_to_disparity(random8.depth64[:2], 500.0, 0.12).cuda().contiguous()
    est = tfn.Estimator(ts.K_VGA, "fd", "median")
    a = est.estimate_disparity(d, 60.0).cpu().numpy()
    b = est.estimate_disparity(d, 60.0 * 73).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("f,m", [("prewitt", "median"), ("fd", "mean"), ("fd", "median"), ("sobel", "mean")])
def test_hires_holes_parity(tfn, f, m):
    """config 4 shape: 1080x1920 with ~2 % hole discs + 1 % salt dropout (Z = 0)."""
    sc = ts.random_scenes(2, ts.K_1080, 1080, 1920, seed=7, holes=True, salt=0.01)
    r = ts.render(sc, ts.K_1080, 1080, 1920)
    z = r.depth.numpy()
    assert (z == 0).mean() > 0.02
    check(tfn, z, ts.K_1080, f, m)


def test_4k_frame_parity(tfn):
    sc = ts.random_scenes(1, ts.K_2160, 2160, 3840, seed=9, holes=True, salt=0.01)
    r = ts.render(sc, ts.K_2160, 2160, 3840)
    check(tfn, r.depth.numpy(), ts.K_2160, "prewitt", "median")


# ------------------------------------------------------------------ adversarial planes
@pytest.mark.parametrize("n", [(0.4, -0.4 * (1 + 3e-4), -1.0), (1e-3, 5e-4, -1.0), (0.0, -0.3, -1.0),
                               (0.7, 0.0, -1.0), (0.3, 0.3, -1.0)])
@pytest.mark.parametrize("m", MODES)
def test_adversarial_planes(tfn, n, m):
    """near-diagonal isoline (cancellation in g_u +- g_v), near-fronto, axis-aligned
    (dZ == 0 along rows/columns -> skipped candidates), exactly diagonal."""
    r = ts.render(ts.plane_scene(n, (0, 0, 3.0)), ts.K_VGA, 480, 640)
    for f in ("sobel", "fd"):
        check(tfn, r.depth.numpy(), ts.K_VGA, f, m)


def test_exact_flat_and_apex(tfn):
    """P2/P3 on the GPU: fronto-parallel -> exactly [0,0,-1]; on-axis sphere apex too."""
    z = np.full((1, 64, 68), 2.5, np.float32)
    for f in FILTERS:
        for m in MODES:
            g = run_gpu(tfn, z, ts.K_VGA, f, m)
            inner = g[0, :, 1:-1, 1:-1]
            assert (inner[0] == 0).all() and (inner[1] == 0).all() and (inner[2] == -1).all()
            assert np.isnan(g[0, :, 0, :]).all() and np.isnan(g[0, :, :, -1]).all()
    K = ts.Intrinsics(500.0, 500.0, 320.0, 240.0)
    zz = ts.render(ts.sphere_scene((0, 0, 3), 1.0), K, 480, 644).depth.numpy()
    for f in FILTERS:
        for m in MODES:
            g = run_gpu(tfn, zz, K, f, m)
            assert tuple(g[0, :, 240, 320]) == (0.0, 0.0, -1.0)


# ------------------------------------------------------------------ edge inputs
def test_invalid_values_and_random_masks(tfn, random8):
    z = random8.depth.numpy()[:3].copy()
    rng = np.random.default_rng(5)
    bad = np.array([0.0, -1.0, np.nan, np.inf, -np.inf, 1e-45, -0.0], np.float32)
    sel = rng.random(z.shape) < 0.15
    z[sel] = bad[rng.integers(0, len(bad), sel.sum())]
    for f in FILTERS:
        for m in MODES:
            check(tfn, z, ts.K_VGA, f, m)


def test_quantized_depth(tfn):
    """integer-millimetre depth: dZ == 0 is common, so the k < 8 paths (skips,
    padding, odd-k median) run on many pixels."""
    sc = ts.random_scenes(2, ts.K_VGA, 480, 640, seed=77)
    r = ts.render(sc, ts.K_VGA, 480, 640, keep_depth64=True)
    z = (np.round(r.depth64.numpy() * 1000.0) / 1000.0).astype(np.float32)
    for f in FILTERS:
        for m in MODES:
            check(tfn, z, ts.K_VGA, f, m)


@pytest.mark.parametrize("H,W", [(1, 1), (2, 5), (5, 2), (3, 3), (4, 4), (5, 7), (17, 37), (33, 130),
                                 (40, 132), (9, 256), (70, 260), (31, 1024)])
def test_sizes(tfn, H, W):
    rng = np.random.default_rng(H * 1000 + W)
    sc = ts.random_scenes(2, ts.Intrinsics(200.0, 210.0, W / 2 - 0.3, H / 2 + 0.7), H, W, seed=H + W)
    z = ts.render(sc, ts.Intrinsics(200.0, 210.0, W / 2 - 0.3, H / 2 + 0.7), H, W).depth.numpy()
    z[rng.random(z.shape) < 0.05] = 0.0
    K = ts.Intrinsics(200.0, 210.0, W / 2 - 0.3, H / 2 + 0.7)
    for f in ("sobel", "fd"):
        for m in MODES:
            g, _ = check(tfn, z, K, f, m)
            if W % 4 == 0 and W >= 4:
                gp = run_gpu(tfn, z, K, f, m, kernel="pixel")
                assert np.array_equal(g.view(np.uint32), gp.view(np.uint32))
    # disparity (the FD32 path; Eq. 21 needs fx == fy)
    Kd = ts.Intrinsics(205.0, 205.0, W / 2 - 0.3, H / 2 + 0.7)
    d = np.where(z > 0, 60.0 / np.where(z > 0, z, 1.0), 0.0).astype(np.float32)
    for m in MODES:
        g, _ = check(tfn, d, Kd, "fd", m, disp=True)
        if W % 4 == 0 and W >= 4:
            gp = run_gpu(tfn, d, Kd, "fd", m, disp=True, kernel="pixel")
            assert_kernels_agree(g, gp, True, (H, W, m))


def test_depth_scale_power_of_two_bitwise(tfn, cfg1):
    z = cfg1.depth.numpy()
    for m in MODES:
        a = run_gpu(tfn, z, ts.K_VGA, "sobel", m)
        b = run_gpu(tfn, z * np.float32(8.0), ts.K_VGA, "sobel", m)
        ok = np.all(np.isfinite(a), 1)
        assert np.array_equal(ok, np.all(np.isfinite(b), 1))
        d = metrics.angular_error_deg(np.moveaxis(a, 1, -1)[ok], np.moveaxis(b, 1, -1)[ok])
        assert d.max() < 1e-5


# ------------------------------------------------------------------ ABI behaviour
def test_abi_errors_and_noops(tfn):
    from paper_2005_08165_b200 import tfn as T
    h = T.tfn_create((500.0, 500.0, 320.0, 240.0), 1, 1)
    x = torch.ones(2, 8, 8, device="cuda")
    o = torch.empty(2, 3, 8, 8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert T.tfn_estimate(h, x.data_ptr(), 0, 8, 8, s, o.data_ptr()) == 0          # batch 0: no-op
    assert T.tfn_estimate(h, 0, 2, 8, 8, s, o.data_ptr()) == 1                       # NULL
    assert T.tfn_estimate(h, x.data_ptr(), -1, 8, 8, s, o.data_ptr()) == 1
    assert T.tfn_estimate(h, x.data_ptr(), 2, 0, 8, s, o.data_ptr()) == 1
    assert T.tfn_estimate(h, x.data_ptr(), 2, 8, 8, s, x.data_ptr()) == 1            # overlap
    assert T.tfn_estimate_disparity(h, x.data_ptr(), 0.0, 2, 8, 8, s, o.data_ptr()) == 2
    assert T.tfn_estimate_disparity(h, x.data_ptr(), float("nan"), 2, 8, 8, s, o.data_ptr()) == 2
    with pytest.raises(T.TfnError):
        T.tfn_set_layout(h, 5)
    T.tfn_destroy(h)
    h2 = T.tfn_create((500.0, 501.0, 320.0, 240.0), 0, 0)
    assert T.tfn_estimate_disparity(h2, x.data_ptr(), 1.0, 2, 8, 8, s, o.data_ptr()) == 2   # fx != fy
    T.tfn_destroy(h2)
    assert T.tfn_destroy(0) == 0


def test_host_path_matches_device_path(tfn, random8):
    z = random8.depth[:5].contiguous()
    for layout in ("planar", "packed"):
        est = tfn.Estimator(ts.K_VGA, "sobel", "median", layout=layout)
        dev = est.estimate(z.cuda()).cpu().numpy()
        host = est.estimate_host(z.pin_memory()).numpy()
        assert np.array_equal(dev.view(np.uint32), host.view(np.uint32))
        host2 = est.estimate_host(z.clone()).numpy()           # pageable host memory also works
        assert np.array_equal(dev.view(np.uint32), host2.view(np.uint32))
    d = ts.depth_to_disparity(random8.depth64[:3], 500.0, 0.12)
    est = tfn.Estimator(ts.K_VGA, "fd", "mean")
    a = est.estimate_disparity(d.cuda(), F_TC).cpu().numpy()
    b = est.estimate_host(d.pin_memory(), is_disparity=True, baseline_times_f=F_TC).numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_launch_counter(tfn, cfg1):
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    x = cfg1.depth.cuda()
    n0 = tfn.tfn_kernel_launches()
    for _ in range(3):
        est.estimate(x)
    assert tfn.tfn_kernel_launches() - n0 == 3


# ------------------------------------------------------------------ P8: the device Phi
def test_phi8_probe(tfn):
    rng = np.random.default_rng(8)
    n = 200000
    c = (rng.normal(size=(n, 8)) * 10.0 ** rng.integers(-3, 4, size=(n, 1))).astype(np.float32)
    k = rng.integers(0, 9, size=n)
    k[: n // 2] = 8
    marks = np.array([np.inf, -np.inf, np.nan], np.float32)
    for i in range(n):
        if k[i] < 8:
            idx = rng.choice(8, 8 - k[i], replace=False)
            c[i, idx] = marks[rng.integers(0, 3, size=idx.size)]
    ties = rng.random(n) < 0.1
    c[ties, 1] = c[ties, 0]
    cc = torch.as_tensor(c).cuda()
    med, kk = tfn.debug_phi8(cc, "median")
    mean, _ = tfn.debug_phi8(cc, "mean")
    mex, kx = tfn.debug_phi8(cc, "median_ext")      # the fast variants' NaN-propagating network
    med, kk, mean = med.cpu().numpy(), kk.cpu().numpy(), mean.cpu().numpy()
    assert np.array_equal(kk, np.isfinite(c).sum(1))
    assert np.array_equal(kx.cpu().numpy(), kk)             # finite extremes <=> all 8 finite
    assert np.array_equal(mex.cpu().numpy().view(np.uint32), med.view(np.uint32))
    for i in range(n):
        v = np.sort(c[i][np.isfinite(c[i])].astype(np.float64))
        if v.size == 0:
            continue
        j = v.size
        exp = v[j // 2] if j % 2 else np.float32((v[j // 2 - 1] + v[j // 2]) / 2.0)
        assert med[i] == np.float32(exp), (i, c[i], med[i], exp)
        assert abs(mean[i] - v.mean()) <= 4e-7 * np.abs(v).sum() + 1e-30


# ------------------------------------------------------------------ a8: stats kernel
def test_stats_kernel_vs_oracle_metrics(tfn, random8):
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    x = random8.depth.cuda()
    gt = random8.gt.cuda()
    out = est.estimate(x)
    acc = tfn.stats(out, gt).cpu().numpy()
    ref = metrics.normal_stats(out.cpu().numpy(), random8.gt.numpy())
    assert acc[1] == ref["m"] and acc[5] == ref["n_valid_est"] and acc[6] == ref["n_valid_gt"]
    assert acc[7] == ref["n_pixels"]
    assert abs(acc[0] / 1e6 - ref["sum_psi_deg"]) <= 1e-6 * ref["m"] + 1e-9 * ref["sum_psi_deg"]
    psi = ref["psi"]
    for j, phi in zip((2, 3, 4), (10, 20, 30)):
        near = np.count_nonzero(np.abs(psi - phi) < 1e-9)
        assert abs(int(acc[j]) - ref[f"n_le_{phi}"]) <= near
    # packed layout gives the same stats
    est2 = tfn.Estimator(ts.K_VGA, "sobel", "median", layout="packed")
    acc2 = tfn.stats(est2.estimate(x), gt, layout="packed").cpu().numpy()
    assert np.array_equal(acc, acc2)
    # median beats mean on clean analytic scenes
    estm = tfn.Estimator(ts.K_VGA, "sobel", "mean")
    accm = tfn.stats(estm.estimate(x), gt).cpu().numpy()
    assert acc[0] / acc[1] <= accm[0] / accm[1] + 0.1e6


# ------------------------------------------------------------------ generator CPU == GPU
def test_generator_bitwise_cpu_gpu(tfn):
    sc = ts.random_scenes(3, ts.K_1080, 1080, 1920, seed=4, first_frame=100, holes=True, salt=0.01)
    a = ts.render(sc, ts.K_1080, 1080, 1920, device="cpu")
    b = ts.render(sc, ts.K_1080, 1080, 1920, device="cuda")
    assert torch.equal(a.depth, b.depth.cpu())
    assert torch.equal(torch.nan_to_num(a.gt, 7.0), torch.nan_to_num(b.gt.cpu(), 7.0))


# ------------------------------------------------------------------ full size (configs[1])
def test_full_size_config2_sampled(tfn):
    """BASELINE.json configs[1] at full size in the launch configuration bench.py
    times (1024 frames, one launch, default strip geometry): whole-frame parity on
    2 frames and sampled pixels on 14 more, the oracle fed with the same frames
    re-rendered on the CPU (bit-identical, asserted)."""
    B, H, W = 1024, 480, 640
    sc = ts.random_scenes(B, ts.K_VGA, H, W, seed=0)
    chunks = []
    for lo in range(0, B, 128):
        chunks.append(ts.render(sc.subset(lo, lo + 128), ts.K_VGA, H, W, device="cuda").depth)
    x = torch.cat(chunks)
    del chunks
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    out = est.estimate(x)
    torch.cuda.synchronize()
    frames = [0, 1023, 1, 2, 100, 255, 256, 511, 512, 700, 767, 768, 900, 1000, 1021, 1022]
    rng = np.random.default_rng(0)
    for i, fidx in enumerate(frames):
        cpu = ts.render(sc.subset(fidx, fidx + 1), ts.K_VGA, H, W, device="cpu").depth[0].numpy()
        assert np.array_equal(cpu, x[fidx].cpu().numpy())
        g = out[fidx].cpu().numpy()
        if i < 2:
            r = oracle.estimate(cpu, ts.K_VGA, "sobel", "median")
            assert_parity(compare(g[None], r[None], cpu[None], ts.K_VGA), f"frame {fidx}")
        else:
            pix = [tuple(p) for p in rng.integers(0, (H, W), size=(3000, 2))] + [(0, 0), (H - 1, W - 1), (5, W - 1)]
            r = oracle.estimate_pixels(cpu, ts.K_VGA, pix, "sobel", "median")
            gg = np.stack([g[:, v, u] for v, u in pix])
            res = compare(gg.T[None, :, None, :], r.T[None, :, None, :], np.zeros((1, 1, len(pix))),
                          ts.K_VGA)
            assert res["mask_equal"]
            # recompute the tie test with the true pixel rays
            ok = np.all(np.isfinite(r), 1)
            a = metrics.angular_error_deg(gg[ok], r[ok])
            if a.size:
                p = np.array([[(u - 320.0) / 500.0, (v - 240.0) / 500.0, 1.0] for v, u in pix])[ok]
                p /= np.linalg.norm(p, axis=1, keepdims=True)
                tie = np.abs(np.sum(r[ok] * p, 1)) < 1e-6
                a = np.where(tie, np.minimum(a, metrics.angular_error_deg(-gg[ok], r[ok])), a)
                assert a.max() <= TOL_DEG, (fidx, a.max())


# ------------------------------------------------------------------ general strip variant
def _general_cases(cfg1, random8):
    """(name, input, K, disparity?) covering skips, holes, invalid encodings, quantization,
    flat / apex, borders and ragged sizes."""
    rng = np.random.default_rng(11)
    z8 = random8.depth.numpy()[:3].copy()
    bad = np.array([0.0, -1.0, np.nan, np.inf, -np.inf, 1e-45, -0.0], np.float32)
    sel = rng.random(z8.shape) < 0.15
    z8[sel] = bad[rng.integers(0, len(bad), sel.sum())]
    q = (np.round(random8.depth64.numpy()[:2] * 1000.0) / 1000.0).astype(np.float32)
    holes = ts.render(ts.random_scenes(1, ts.K_1080, 1080, 1920, seed=7, holes=True, salt=0.01),
                      ts.K_1080, 1080, 1920).depth.numpy()
    flat = np.full((1, 64, 68), 2.5, np.float32)
    K33 = ts.Intrinsics(200.0, 210.0, 130 / 2 - 0.3, 33 / 2 + 0.7)
    small = ts.render(ts.random_scenes(2, K33, 33, 132, seed=3), K33, 33, 132).depth.numpy()
    small[rng.random(small.shape) < 0.05] = 0.0
    d = ts.depth_to_disparity(random8.depth64[:2], 500.0, 0.12).numpy()
    # disparity with holes and dropout (Z = 0 -> d = 0, invalid) on a ragged-width crop
    dh = np.where(holes[:, :540, :964] > 0, (1000.0 * 0.12) / np.maximum(holes[:, :540, :964], 1e-30), 0.0)
    dh = dh.astype(np.float32)
    return [("cfg1", cfg1.depth.numpy(), ts.K_VGA, False), ("invalid", z8, ts.K_VGA, False),
            ("quantized", q, ts.K_VGA, False), ("holes1080", holes, ts.K_1080, False),
            ("flat", flat, ts.K_VGA, False), ("small", small, K33, False),
            ("disparity", d, ts.K_VGA, True), ("disparity_holes", dh, ts.K_1080, True)]


def test_general_kernel_bitwise_vs_pixel(tfn, cfg1, random8):
    """kernel=3 (no special path: skips, flat, ties, invalid taps all handled in registers)
    is bit-identical to the per-pixel kernel on every hard case, and parity-green."""
    for name, z, K, disp in _general_cases(cfg1, random8):
        for f in FILTERS:
            for m in MODES:
                gg = run_gpu(tfn, z, K, f, m, disp=disp, kernel="general")
                gp = run_gpu(tfn, z, K, f, m, disp=disp, kernel="pixel")
                assert np.array_equal(gg.view(np.uint32), gp.view(np.uint32)), (name, f, m)
                gk = run_gpu(tfn, z, K, f, m, disp=disp, kernel="general", layout="packed")
                assert np.array_equal(gg.view(np.uint32), gk.view(np.uint32)), (name, f, m, "packed")
    z = random8.depth.numpy()
    for f in ("sobel", "fd"):
        for m in MODES:
            check(tfn, z, ts.K_VGA, f, m, kernel="general")


def test_masked_kernel_bitwise_vs_pixel(tfn, cfg1, random8):
    """kernel=4 (the fast kernel whose special path skips pixels with an invalid Q4 tap —
    their NaN is already exact — and needs no border masks: out-of-image taps are invalid
    taps) is bit-identical to the per-pixel kernel on every hard case, both layouts (disparity
    FD + mean: fp32 gradients, within FD32_TOL_DEG of it — tests/parity.py)."""
    from paper_2005_08165_b200 import tfn as T
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    with pytest.raises(T.TfnError):
        T.tfn_set_option(est.h, T.OPT_KERNEL, 7)          # 0 auto .. 6 fp32 masked
    for name, z, K, disp in _general_cases(cfg1, random8):
        for f in FILTERS:
            for m in MODES:
                gp = run_gpu(tfn, z, K, f, m, disp=disp, kernel="pixel")
                gm = run_gpu(tfn, z, K, f, m, disp=disp, kernel="masked")
                assert_kernels_agree(gm, gp, fd32_variant(disp, f, m), (name, f, m))
                gk = run_gpu(tfn, z, K, f, m, disp=disp, kernel="masked", layout="packed")
                assert np.array_equal(gm.view(np.uint32), gk.view(np.uint32)), (name, f, m, "packed")
                if f == "sobel" and m == "median":
                    for sh in (5, 13):
                        gs = run_gpu(tfn, z, K, f, m, disp=disp, kernel="masked", strip_h=sh)
                        assert np.array_equal(gm.view(np.uint32), gs.view(np.uint32)), (name, sh)


def test_auto_variant_follows_the_special_rate(tfn, cfg1):
    """AUTO starts on the fast strip kernel; on hole-heavy input (config-4 style: ~98 % of the
    fast kernel's row steps need the special path, few of the masked kernel's) it moves to
    the masked kernel; on millimetre-quantized depth (dZ = 0 everywhere, the masked kernel
    fires too) on to the general one; and it stays fast on clean input.  The output is
    bit-identical whichever variant ran."""
    from paper_2005_08165_b200 import tfn as T
    sc = ts.random_scenes(2, ts.K_1080, 1080, 1920, seed=7, holes=True, salt=0.01)
    holes = ts.render(sc, ts.K_1080, 1080, 1920).depth.cuda()
    est = tfn.Estimator(ts.K_1080, "sobel", "median")
    assert T.tfn_auto_variant(est.h) == 2
    ref = run_gpu(tfn, holes.cpu().numpy(), ts.K_1080, "sobel", "median", kernel="pixel")
    for _ in range(40):
        out = est.estimate(holes)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert T.tfn_auto_variant(est.h) == 4
    quant = torch.round(holes * 1000.0) / 1000.0          # fp32 millimetre steps: dZ = 0 is common
    refq = run_gpu(tfn, quant.cpu().numpy(), ts.K_1080, "sobel", "median", kernel="pixel")
    estq = tfn.Estimator(ts.K_1080, "sobel", "median")
    for _ in range(80):
        out = estq.estimate(quant)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), refq.view(np.uint32))
    assert T.tfn_auto_variant(estq.h) == 3
    clean = cfg1.depth.reshape(1, 480, 640).repeat(4, 1, 1).cuda()
    est2 = tfn.Estimator(ts.K_VGA, "sobel", "median")
    for _ in range(40):
        est2.estimate(clean)
        torch.cuda.synchronize()
    assert T.tfn_auto_variant(est2.h) == 2


# ------------------------------------------------------------------ N2: noisy depth
@pytest.mark.parametrize("level", ["low", "high"])
def test_noisy_depth_parity(tfn, random8, level):
    """Gaussian depth noise (S:374 presets) — parity, and the fast, general
    and per-pixel kernels agree bit for bit on it."""
    z = ts.add_gaussian_noise(random8.depth[:3], ts.NOISE_PRESETS[level], seed=11).numpy()
    for f in ("fd", "sobel"):
        for m in MODES:
            g, _ = check(tfn, z, ts.K_VGA, f, m)
            for kernel in ("strip", "masked", "general", "pixel"):
                gk = run_gpu(tfn, z, ts.K_VGA, f, m, kernel=kernel)
                assert np.array_equal(g.view(np.uint32), gk.view(np.uint32)), (level, f, m, kernel)


def test_noise_degrades_accuracy_monotonically(tfn, random8):
    """N2 workload sanity through the a8 stats kernel: the average angular error grows with
    the noise preset (clean < low < medium < high) for both Phi.  (Which Phi wins depends on
    the noise-to-footprint ratio: at these presets, 0.1-1 % of ~3.5 m against a ~7 mm pixel
    footprint, the noise dominates every 3x3 neighbourhood; see tools/noise_table.py.)"""
    gt = random8.gt.cuda()
    for m in MODES:
        est = tfn.Estimator(ts.K_VGA, "fd", m)
        aae = []
        for rel in (0.0, ts.NOISE_PRESETS["low"], ts.NOISE_PRESETS["medium"], ts.NOISE_PRESETS["high"]):
            z = ts.add_gaussian_noise(random8.depth, rel, seed=3).cuda()
            acc = tfn.stats(est.estimate(z), gt).cpu().numpy()
            aae.append(acc[0] / 1e6 / acc[1])
        assert all(a < b for a, b in zip(aae, aae[1:])), (m, aae)


# ------------------------------------------------------------------ N1: run-time (p, q) weights
@pytest.mark.parametrize("w", [(1.0, 4.0), (0.5, 3.7), (2.5, 1.0), (1e-3, 1.0)])
def test_custom_weights_parity(tfn, random8, w):
    """TFN_FILTER_CUSTOM: the [kp k0 kp] family of the paper's 3x3 kernel search
    against the oracle with the same weights; fast, general and per-pixel kernels agree bit
    for bit (holes and quantized depth included)"""
    z = random8.depth.numpy()[:2].copy()
    z[:, 100:140, 200:260] = 0.0
    zq = (np.round(random8.depth64.numpy()[2:3] * 1000.0) / 1000.0).astype(np.float32)
    for m in MODES:
        for x in (z, zq):
            g, _ = check(tfn, x, ts.K_VGA, w, m)
            for kernel in ("strip", "masked", "general", "pixel"):
                gk = run_gpu(tfn, x, ts.K_VGA, w, m, kernel=kernel)
                assert np.array_equal(g.view(np.uint32), gk.view(np.uint32)), (w, m, kernel)


def test_custom_weights_reproduce_named_kernels(tfn, random8):
    """(1,2), (3,10), (1,1) are Sobel, Scharr, Prewitt bit for bit (same fp64 sums)"""
    z = random8.depth.numpy()[:2]
    for name, w in (("sobel", (1.0, 2.0)), ("scharr", (3.0, 10.0)), ("prewitt", (1.0, 1.0))):
        for m in MODES:
            a = run_gpu(tfn, z, ts.K_VGA, name, m)
            b = run_gpu(tfn, z, ts.K_VGA, w, m)
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (name, m)
    from paper_2005_08165_b200 import tfn as T
    est = tfn.Estimator(ts.K_VGA, (1.0, 2.0), "median")
    for bad in ((0.0, 1.0), (1.0, 0.0), (-1.0, 2.0), (float("nan"), 1.0)):
        with pytest.raises(T.TfnError):
            T.tfn_set_filter_weights(est.h, *bad)
    with pytest.raises(T.TfnError):
        T.tfn_set_filter_weights(tfn.Estimator(ts.K_VGA, "sobel", "median").h, 1.0, 2.0)


def test_cuda_graph_capture(tfn, cfg1, random8):
    """the ABI is capture-safe (no host sync / event query while a stream captures): a
    CUDA graph of one estimate call replays to the same bits, also after the input buffer
    is refilled in place; AUTO's choice at capture time is baked in"""
    x = random8.depth[:2].cuda().contiguous()
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    ref = est.estimate(x).clone()
    out = torch.empty_like(ref)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            est.estimate(x, out=out, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
    x.copy_(random8.depth[2:4].cuda())
    g.replay()
    torch.cuda.synchronize()
    ref2 = est.estimate(x)
    assert torch.equal(out.view(torch.int32), ref2.view(torch.int32))


def test_pixel_kernel_large_batch(tfn):
    """more than 65535 frames (grid z limit) through the per-pixel kernel: chunked launches"""
    B, H, W = 70000, 3, 5
    z = torch.full((B, H, W), 2.0, device="cuda")
    z[-1, 1, 1:4] = torch.tensor([2.0, 2.2, 2.4])
    est = tfn.Estimator(ts.K_VGA, "fd", "median", kernel="pixel")
    out = est.estimate(z)
    torch.cuda.synchronize()
    assert torch.equal(out[0, :, 1, 1], torch.tensor([0.0, 0.0, -1.0], device="cuda"))
    assert torch.equal(out[65535, :, 1, 1], torch.tensor([0.0, 0.0, -1.0], device="cuda"))
    assert not torch.equal(out[-1, :, 1, 2], out[0, :, 1, 2])
    p = est.plane_fit(z, "pca")
    torch.cuda.synchronize()
    assert torch.isfinite(p[-1, :, 1, 1]).all() and torch.isnan(p[-1, :, 0, 0]).all()


# ------------------------------------------------------------------ extreme ranges / intrinsics
@pytest.mark.parametrize("scale", [1e-3, 1.0, 3e3])
def test_extreme_depth_scales_and_occlusions(tfn, random8, scale):
    """depth in millimetres-of-a-micro-scene up to kilometres, with occlusion steps of 100x
    (near/far mixes inside one 3x3 window) and tiny / huge focal lengths: parity and the
    three kernels bit-identical"""
    z = random8.depth.numpy()[:2].astype(np.float64) * scale
    rng = np.random.default_rng(int(scale * 1000) % 2**31)
    for _ in range(40):                                  # occluding near / far rectangles
        b, v, u = rng.integers(0, 2), rng.integers(0, 440), rng.integers(0, 600)
        h, w = rng.integers(3, 40), rng.integers(3, 40)
        z[b, v:v + h, u:u + w] *= rng.choice([0.01, 100.0])
    z = z.astype(np.float32)
    for K in (ts.Intrinsics(500.0, 470.0, 321.3, 238.9), ts.Intrinsics(5.0, 5.0, 320.0, 240.0),
              ts.Intrinsics(5e4, 4.5e4, -100.0, 900.0)):
        for f in ("fd", "sobel"):
            for m in MODES:
                g, _ = check(tfn, z, K, f, m)
                for kernel in ("masked", "general", "pixel"):
                    gk = run_gpu(tfn, z, K, f, m, kernel=kernel)
                    assert np.array_equal(g.view(np.uint32), gk.view(np.uint32)), (scale, K, f, m, kernel)


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e3])
def test_extreme_disparity_and_noise(tfn, random8, scale):
    """disparity maps scaled over six decades with 100x occlusion steps, and every filter on
    heavily noisy depth (S:374 high preset): parity and bit-identical kernels (disparity FD +
    mean: within FD32_TOL_DEG, tests/parity.py)"""
    d = ts.depth_to_disparity(random8.depth64[:2], 500.0, 0.12).numpy().astype(np.float64) * scale
    rng = np.random.default_rng(int(scale * 7) + 1)
    for _ in range(40):
        b, v, u = rng.integers(0, 2), rng.integers(0, 440), rng.integers(0, 600)
        d[b, v:v + rng.integers(3, 40), u:u + rng.integers(3, 40)] *= rng.choice([0.01, 100.0])
    d = d.astype(np.float32)
    for f in ("fd", "scharr"):
        for m in MODES:
            g, _ = check(tfn, d, ts.K_VGA, f, m, disp=True)
            gk = run_gpu(tfn, d, ts.K_VGA, f, m, disp=True, kernel="general")
            assert_kernels_agree(g, gk, fd32_variant(True, f, m), (scale, f, m))
    if scale == 1.0:
        z = ts.add_gaussian_noise(random8.depth[:2], ts.NOISE_PRESETS["high"], seed=5).numpy()
        for f in FILTERS:
            for m in MODES:
                check(tfn, z, ts.K_VGA, f, m)


def test_fd32_disparity_cancellation_fallback(tfn):
    """disparity FD runs fp32 gradients with s and t re-paired along the diagonals; a
    saddle d = 1 + 1e-2 (u - v) + kappa (u + v)^2 puts s = g_u + g_v through zero along u + v = c,
    where the two diagonal differences have opposite signs and the pixel takes the fp64 s, t
    (fd_st64): parity with the oracle on both sides of the line, every variant, three curvatures"""
    H, W = 96, 160
    v, u = np.mgrid[0:H, 0:W].astype(np.float64)
    for kappa in (1e-6, 1e-5, 1e-4):
        d = 2.0 + 1e-2 * (u - v) + kappa * (u + v - 120.0) ** 2
        d = d.astype(np.float32)[None]
        for m in MODES:
            g, _ = check(tfn, d, ts.K_VGA, "fd", m, disp=True)
            for k in ("masked", "general", "pixel"):
                gk = run_gpu(tfn, d, ts.K_VGA, "fd", m, disp=True, kernel=k)
                assert_kernels_agree(g, gk, k in ("general", "pixel"), (kappa, m, k))


def test_fd32_noisy_disparity(tfn, random8):
    """noisy disparity (the high noise preset on the depth, then d = f b / Z) puts the FD32 sign
    guard on a large share of pixels: the fallback runs for most row steps; parity and variant
    agreement hold, with holes in the mix"""
    z = ts.add_gaussian_noise(random8.depth[:2], ts.NOISE_PRESETS["high"], seed=11)
    d = ts.depth_to_disparity(z.double(), 500.0, 0.12).numpy().astype(np.float32)
    rng = np.random.default_rng(3)
    d[rng.random(d.shape) < 0.02] = 0.0                     # holes (invalid disparity)
    for m in MODES:
        g, _ = check(tfn, d, ts.K_VGA, "fd", m, disp=True)
        for k in ("masked", "general"):
            gk = run_gpu(tfn, d, ts.K_VGA, "fd", m, disp=True, kernel=k)
            assert_kernels_agree(g, gk, k == "general", (m, k))


def test_graph_counter_never_shared_with_direct_calls(tfn, random8):
    """a launch captured into a CUDA graph keeps its own work counter.  Capture a
    dynamically scheduled launch, make > 4096 direct calls (the direct-call ring wraps), then
    replay the graph on one stream while direct calls run on another: the replayed output is
    bit-identical to the uncaptured result every time."""
    x = random8.depth.cuda().repeat(8, 1, 1)                   # 64 frames: more strips than warps
    est = tfn.Estimator(ts.K_VGA, "sobel", "median", kernel="strip")
    ref = est.estimate(x).clone()
    out = torch.empty_like(ref)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        with torch.cuda.graph(g, stream=s1):
            est.estimate(x, out=out, stream=s1)
    torch.cuda.synchronize()
    small = x[:16]
    scratch = torch.empty((16, 3, 480, 640), device="cuda")
    for _ in range(4100):                                     # the direct ring (4096 pairs) wraps
        est.estimate(small, out=scratch, stream=s2)
    torch.cuda.synchronize()
    for _ in range(6):
        out.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            g.replay()
        for _ in range(4):
            est.estimate(small, out=scratch, stream=s2)      # concurrent direct calls
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
