"""N2 noise workload generator (tfn_scenes.add_gaussian_noise): SPEC S:357-366 examples and
S:374 presets.  CPU only; no 3F2N arithmetic involved."""
import math

import numpy as np
import torch

import tfn_scenes as ts


def test_sigma_zero_and_determinism():
    z = ts.render(ts.random_scenes(3, ts.K_VGA, 48, 64, seed=2), ts.K_VGA, 48, 64).depth
    assert torch.equal(ts.add_gaussian_noise(z, 0.0, seed=1), z)
    a = ts.add_gaussian_noise(z, 0.003, seed=1)
    b = ts.add_gaussian_noise(z, 0.003, seed=1)
    c = ts.add_gaussian_noise(z, 0.003, seed=2)
    assert torch.equal(a, b) and not torch.equal(a, c)
    # counter-based: a frame's noise depends on (seed, global frame id, pixel) only
    d = ts.add_gaussian_noise(z[1:], 0.003, seed=1, first_frame=1)
    assert torch.equal(d, a[1:])
    # invalid pixels stay invalid
    assert torch.equal(a[z == 0], z[z == 0])


def test_statistics_on_constant_depth():
    """over a 480x640 constant-depth image the sample mean of z'-z is within
    3 sigma / sqrt(N) of 0 and the sample std within 5 % of sigma."""
    z = torch.full((1, 480, 640), 2.0, dtype=torch.float32)
    for name, rel in ts.NOISE_PRESETS.items():
        sigma = rel * 2.0
        d = (ts.add_gaussian_noise(z, rel, seed=7).double() - 2.0).flatten()
        n = d.numel()
        assert abs(float(d.mean())) < 3 * sigma / math.sqrt(n), name
        assert abs(float(d.std()) / sigma - 1.0) < 0.05, name
        # and it is Gaussian, not uniform: ~68.3 % within one sigma, ~95.4 % within two
        assert abs(float((d.abs() < sigma).double().mean()) - 0.6827) < 0.01
        assert abs(float((d.abs() < 2 * sigma).double().mean()) - 0.9545) < 0.005


def test_pushed_below_zero_becomes_invalid():
    z = torch.full((1, 64, 64), 1e-3, dtype=torch.float32)
    zn = ts.add_gaussian_noise(z, 10.0, seed=3)          # sigma = 10x depth: ~half go <= 0
    frac = float((zn == 0).double().mean())
    assert 0.4 < frac < 0.6
    assert bool((zn >= 0).all())


def test_sigma_scales_with_frame_mean_depth():
    z = torch.stack([torch.full((32, 32), 1.0), torch.full((32, 32), 4.0)])
    d = ts.add_gaussian_noise(z, 0.01, seed=5).double() - z.double()
    r = float(d[1].std() / d[0].std())
    assert 3.0 < r < 5.3                                  # 4x the mean depth -> ~4x sigma
