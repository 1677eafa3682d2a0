"""reduced-byte I/O: uint16 depth codes in (Z = code x scale, code 0
= no measurement; 2 B/px) and IEEE-half normals out (6 B/px), on the GPU through the C ABI.

Parity: the oracle runs on the fp64 depths code * scale (the definition; the scale cancels
from the direction, Appendix A.4, so the kernels work on the codes).  Bit-level checks: the
uint16 path equals the fp32 path on the values (float)code, every kernel variant; the half
output equals the fp32 output rounded to nearest (numpy's float16 conversion).
"""
import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts
from tests.parity import assert_parity, compare

pytestmark = pytest.mark.gpu

FILTERS = ("fd", "sobel", "scharr", "prewitt")
MODES = ("mean", "median")
SCALE = 1e-3          # millimetre codes


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


def mm_codes(frames=3, seed=31, H=480, W=640, K=ts.K_VGA, holes=False):
    """ScanNet-like millimetre depth codes of the analytic scenes (0 = no return)."""
    sc = ts.random_scenes(frames, K, H, W, seed=seed, holes=holes, salt=0.01 if holes else 0.0)
    r = ts.render(sc, K, H, W, keep_depth64=True)
    z = r.depth64.numpy()
    codes = np.where(np.isfinite(z) & (z > 0), np.round(z / SCALE), 0.0)
    return np.clip(codes, 0, 65535).astype(np.uint16)


def run_u16(tfn, codes, K, f, m, **kw):
    est = tfn.Estimator(K, filter=f, nz_mode=m, **kw)
    out = est.estimate(torch.from_numpy(codes).cuda(), depth_scale=SCALE)
    torch.cuda.synchronize()
    return out.cpu()


def run_f32(tfn, z, K, f, m, **kw):
    est = tfn.Estimator(K, filter=f, nz_mode=m, **kw)
    out = est.estimate(torch.from_numpy(np.ascontiguousarray(z, np.float32)).cuda())
    torch.cuda.synchronize()
    return out.cpu()


def same_bits(a: torch.Tensor, b: torch.Tensor) -> bool:
    return np.array_equal(a.numpy().view(np.uint32 if a.dtype == torch.float32 else np.uint16),
                          b.numpy().view(np.uint32 if b.dtype == torch.float32 else np.uint16))


@pytest.mark.parametrize("f", FILTERS)
@pytest.mark.parametrize("m", MODES)
def test_u16_parity_vs_oracle(tfn, f, m):
    codes = mm_codes()
    g = run_u16(tfn, codes, ts.K_VGA, f, m).numpy()
    z64 = codes.astype(np.float64) * SCALE                      # Z = code x scale (definition)
    r = oracle.estimate(z64, ts.K_VGA, f, m, threads=4)
    res = compare(g, r, z64, ts.K_VGA)
    assert_parity(res, f"u16 {f}/{m}")
    assert res["n_valid"] > 0.9 * codes.size


def test_u16_holes_parity_vs_oracle(tfn):
    codes = mm_codes(frames=1, seed=5, H=1080, W=1920, K=ts.K_1080, holes=True)
    assert (codes == 0).mean() > 0.02
    for f, m in (("sobel", "median"), ("fd", "mean")):
        g = run_u16(tfn, codes, ts.K_1080, f, m).numpy()
        z64 = codes.astype(np.float64) * SCALE
        assert_parity(compare(g, oracle.estimate(z64, ts.K_1080, f, m, threads=4), z64, ts.K_1080), f"u16 holes {f}/{m}")


def test_u16_bitwise_equals_f32_of_codes(tfn):
    """the uint16 kernels compute exactly what the fp32 kernels compute on (float)code, for
    every kernel variant and layout, and for a ragged / unaligned (per-pixel kernel) case"""
    codes = mm_codes(frames=2, seed=8)
    zf = codes.astype(np.float32)
    for f in FILTERS:
        for m in MODES:
            ref = run_f32(tfn, zf, ts.K_VGA, f, m, kernel="pixel")
            for kernel in ("auto", "strip", "masked", "general", "pixel"):
                assert same_bits(run_u16(tfn, codes, ts.K_VGA, f, m, kernel=kernel), ref), (f, m, kernel)
            pk = run_u16(tfn, codes, ts.K_VGA, f, m, layout="packed")
            assert same_bits(pk.permute(0, 3, 1, 2).contiguous(), ref), (f, m, "packed")
    # W % 4 != 0 and a 2-byte offset: the per-pixel kernel, same bits
    c = np.ascontiguousarray(codes[:, :101, 3:190])
    ref = run_f32(tfn, c.astype(np.float32), ts.K_VGA, "sobel", "median")
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    buf = torch.from_numpy(np.concatenate([np.zeros(1, np.uint16), c.ravel()])).cuda()
    out = est.estimate(buf[1:].view(c.shape), depth_scale=SCALE)
    assert same_bits(out.cpu(), ref)


def test_f16_output_is_rounded_f32(tfn):
    """half normals == the fp32 normals rounded to nearest (NaN stays NaN), every kernel,
    both layouts, fp32 and uint16 input"""
    sc = ts.random_scenes(2, ts.K_VGA, 480, 640, seed=4, holes=True, salt=0.005)
    z = ts.render(sc, ts.K_VGA, 480, 640).depth.numpy()
    codes = mm_codes(frames=2, seed=9)
    for layout in ("planar", "packed"):
        for kernel in ("auto", "strip", "masked", "general", "pixel"):
            for f, m in (("sobel", "median"), ("fd", "mean")):
                a = run_f32(tfn, z, ts.K_VGA, f, m, kernel=kernel, layout=layout).numpy()
                h = run_f32(tfn, z, ts.K_VGA, f, m, kernel=kernel, layout=layout, out_dtype="f16").numpy()
                assert h.dtype == np.float16
                ref = a.astype(np.float16)
                assert np.array_equal(np.isnan(h), np.isnan(ref))
                ok = ~np.isnan(ref)
                assert np.array_equal(h[ok].view(np.uint16), ref[ok].view(np.uint16)), (layout, kernel, f, m)
                a = run_u16(tfn, codes, ts.K_VGA, f, m, kernel=kernel, layout=layout).numpy()
                h = run_u16(tfn, codes, ts.K_VGA, f, m, kernel=kernel, layout=layout, out_dtype="f16").numpy()
                ref = a.astype(np.float16)
                ok = ~np.isnan(ref)
                assert np.array_equal(np.isnan(h), ~ok) and np.array_equal(h[ok].view(np.uint16), ref[ok].view(np.uint16))


def test_u16_host_path_and_errors(tfn):
    from paper_2005_08165_b200 import tfn as T
    codes = mm_codes(frames=5, seed=12)
    est = tfn.Estimator(ts.K_VGA, "sobel", "median", out_dtype="f16")
    dev = est.estimate(torch.from_numpy(codes).cuda(), depth_scale=SCALE).cpu()
    host = est.estimate_host(torch.from_numpy(codes).pin_memory(), depth_scale=SCALE)
    assert host.dtype == torch.float16 and same_bits(host, dev)
    # depth_scale must be finite and > 0 (validated, then unused)
    x = torch.from_numpy(codes).cuda()
    out = torch.empty((5, 3, 480, 640), dtype=torch.float16, device="cuda")
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        assert T.tfn_estimate_u16(est.h, x.data_ptr(), bad, 5, 480, 640, 0, out.data_ptr()) == T.TFN_ERR_CONFIG
    assert T.tfn_estimate_u16(est.h, x.data_ptr(), 2.5, 5, 480, 640, 0, out.data_ptr()) == T.TFN_OK
    torch.cuda.synchronize()
    assert same_bits(out.cpu(), dev)             # the scale cancels: identical bits
    with pytest.raises(T.TfnError):
        T.tfn_set_option(est.h, T.OPT_OUT_DTYPE, 3)


def test_oct16_normals(tfn):
    """TFN_OUT_OCT16 (4 B/pixel): the decoded direction is within 0.005 deg of the fp32
    normal (snorm16 steps of 1/32767 on the octahedral map), the invalid mask maps to the
    (-32768, -32768) sentinel, and every kernel and layout writes the same bits; uint16
    input works too (2 + 4 = 6 B/pixel end to end)"""
    sc = ts.random_scenes(2, ts.K_VGA, 480, 640, seed=13, holes=True, salt=0.005)
    z = ts.render(sc, ts.K_VGA, 480, 640).depth
    from oracle import metrics
    ref32 = run_f32(tfn, z.numpy(), ts.K_VGA, "sobel", "median").numpy()
    base = None
    for layout in ("planar", "packed"):
        for kernel in ("auto", "strip", "masked", "general", "pixel"):
            q = run_f32(tfn, z.numpy(), ts.K_VGA, "sobel", "median", kernel=kernel, layout=layout,
                        out_dtype="oct16")
            assert q.dtype == torch.int16 and q.shape == ((2, 2, 480, 640) if layout == "planar" else (2, 480, 640, 2))
            qp = q if layout == "planar" else q.permute(0, 3, 1, 2).contiguous()
            if base is None:
                base = qp
            assert torch.equal(qp, base), (layout, kernel)
    n = tfn.decode_oct16(base).numpy()
    ok = np.all(np.isfinite(ref32), 1)
    assert np.array_equal(ok, np.all(np.isfinite(n), 1))
    assert ((base[:, 0] == -32768) & (base[:, 1] == -32768)).numpy().sum() == (~ok).sum()
    a = metrics.angular_error_deg(np.moveaxis(n, 1, -1)[ok], np.moveaxis(ref32, 1, -1)[ok])
    assert a.max() < 0.005, a.max()
    codes = mm_codes(frames=2, seed=14)
    qu = run_u16(tfn, codes, ts.K_VGA, "fd", "median", out_dtype="oct16")
    ru = run_u16(tfn, codes, ts.K_VGA, "fd", "median").numpy()
    nu = tfn.decode_oct16(qu).numpy()
    oku = np.all(np.isfinite(ru), 1)
    assert np.array_equal(oku, np.all(np.isfinite(nu), 1))
    assert metrics.angular_error_deg(np.moveaxis(nu, 1, -1)[oku], np.moveaxis(ru, 1, -1)[oku]).max() < 0.005


@pytest.mark.parametrize("H,W", [(3, 4), (5, 8), (37, 132), (64, 260), (50, 644), (130, 388)])
def test_u16_ring_ragged_bitwise(tfn, H, W):
    """the uint16 strip kernels stage rows through a cp.async shared-memory ring whose
    out-of-image rows, halos and lanes past W are zero-filled (code 0 = invalid): on ragged
    shapes (W % 128 != 0, tiny H) and odd strip heights they still equal the fp32 per-pixel
    kernel on (float)code bit for bit, both layouts, both strip variants"""
    codes = mm_codes(frames=2, seed=40 + H, H=H, W=W, K=ts.Intrinsics(W * 0.8, W * 0.8, W / 2 - 0.5, H / 2 - 0.5),
                     holes=True)
    K = ts.Intrinsics(W * 0.8, W * 0.8, W / 2 - 0.5, H / 2 - 0.5)
    zf = codes.astype(np.float32)
    for f, m in (("sobel", "median"), ("fd", "mean"), ("scharr", "mean")):
        ref = run_f32(tfn, zf, K, f, m, kernel="pixel")
        for kernel in ("strip", "general"):
            for sh in (0, 7, 13):
                assert same_bits(run_u16(tfn, codes, K, f, m, kernel=kernel, strip_h=sh), ref), (f, m, kernel, sh)
        pk = run_u16(tfn, codes, K, f, m, layout="packed", strip_h=5)
        assert same_bits(pk.permute(0, 3, 1, 2).contiguous(), ref), (f, m, "packed")
