"""fused point-cloud output (tfn_estimate_points) on the GPU: points
against the oracle's Eq. 13 image back-projection (fp64), normals bit-identical to
tfn_estimate, every input kind, kernel and layout."""
import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts

pytestmark = pytest.mark.gpu

F_TC = 500.0 * 0.12


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def scene():
    sc = ts.random_scenes(3, ts.K_VGA, 480, 640, seed=21, holes=True, salt=0.005)
    return ts.render(sc, ts.K_VGA, 480, 640, keep_depth64=True)


def check_points(p_gpu: np.ndarray, z64: np.ndarray, K, layout="planar"):
    """fp32 points vs the oracle's fp64 points: identical NaN mask, each coordinate within
    4 ulp-equivalents (4 * 2^-24 relative to |p|) — the documented rounding fl(fl(aZ)/fx)"""
    p = np.asarray(p_gpu, np.float64)
    if layout == "packed":
        p = np.moveaxis(p, -1, 1)
    r = oracle.backproject_image(z64, K)
    assert np.array_equal(np.isnan(p), np.isnan(r))
    ok = ~np.isnan(r)
    norm = np.broadcast_to(np.linalg.norm(np.nan_to_num(r), axis=1, keepdims=True), r.shape)
    err = np.abs(p[ok] - r[ok]) / np.maximum(norm[ok], 1e-30)
    assert err.max() <= 4 * 2.0 ** -24, err.max()


@pytest.mark.parametrize("layout", ["planar", "packed"])
@pytest.mark.parametrize("kernel", ["auto", "strip", "general", "pixel"])
def test_points_depth_f32(tfn, scene, layout, kernel):
    z = scene.depth.cuda()
    est = tfn.Estimator(ts.K_VGA, "sobel", "median", layout=layout, kernel=kernel)
    n, p = est.estimate_points(z, scale=1.0)
    torch.cuda.synchronize()
    ref = est.estimate(z)
    assert torch.equal(n.view(torch.int32), ref.view(torch.int32))
    check_points(p.cpu().numpy(), scene.depth.numpy().astype(np.float64), ts.K_VGA, layout)


def test_points_u16_and_disparity(tfn, scene):
    codes = torch.round(scene.depth * 1000.0).clamp(0, 65535).to(torch.int32).to(torch.uint16)
    est = tfn.Estimator(ts.K_VGA, "fd", "mean", out_dtype="f16")
    n, p = est.estimate_points(codes.cuda(), scale=1e-3)
    torch.cuda.synchronize()
    assert torch.equal(n.view(torch.int16), est.estimate(codes.cuda(), depth_scale=1e-3).view(torch.int16))
    z64 = codes.to(torch.int32).numpy().astype(np.float64) * 1e-3
    # Z = fl(code * fl(1e-3)): one more rounding of the scale
    check_points(p.cpu().numpy(), z64, ts.K_VGA)
    d = ts.depth_to_disparity(scene.depth64, 500.0, 0.12)
    est2 = tfn.Estimator(ts.K_VGA, "scharr", "median")
    n2, p2 = est2.estimate_points(d.cuda(), scale=F_TC, disparity=True)
    torch.cuda.synchronize()
    assert torch.equal(n2.view(torch.int32), est2.estimate_disparity(d.cuda(), F_TC).view(torch.int32))
    dd = d.numpy().astype(np.float64)
    zd = np.where(np.isfinite(dd) & (dd >= np.finfo(np.float32).tiny), F_TC / np.where(dd > 0, dd, 1.0), 0.0)
    check_points(p2.cpu().numpy(), zd, ts.K_VGA)


def test_points_errors(tfn, scene):
    from paper_2005_08165_b200 import tfn as T
    z = scene.depth.cuda()
    est = tfn.Estimator(ts.K_VGA, "sobel", "median")
    n = torch.empty((3, 3, 480, 640), device="cuda")
    p = torch.empty((3, 3, 480, 640), device="cuda")
    args = (3, 480, 640, 0, n.data_ptr(), p.data_ptr())
    assert T.tfn_estimate_points(est.h, z.data_ptr(), 0, 0.0, *args) == T.TFN_ERR_CONFIG
    assert T.tfn_estimate_points(est.h, z.data_ptr(), 7, 1.0, *args) == T.TFN_ERR_INVALID_ARGUMENT
    assert T.tfn_estimate_points(est.h, z.data_ptr(), 0, 1.0, 3, 480, 640, 0, n.data_ptr(), n.data_ptr()) \
        == T.TFN_ERR_INVALID_ARGUMENT                               # points overlap the normals
    assert T.tfn_estimate_points(est.h, z.data_ptr(), 0, 1.0, 3, 480, 640, 0, n.data_ptr(), 0) \
        == T.TFN_ERR_INVALID_ARGUMENT
