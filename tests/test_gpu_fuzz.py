"""Fuzz parity: structureless random depth (every 3x3 window chaotic: tiny and huge dZ,
candidates of all magnitudes and signs, 10 % invalid samples, optionally millimetre-
quantized) against the fp64 oracle for every filter x Phi, and the three kernels bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import tfn_scenes as ts
from tests.parity import assert_parity, compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tfn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2005_08165_b200 as m
    m.lib()
    return m


@pytest.mark.parametrize("seed", range(4))
def test_white_noise_depth(tfn, seed):
    rng = np.random.default_rng(seed)
    z = rng.uniform(0.5, 5.0, size=(2, 96, 128)).astype(np.float32)
    z[rng.random(z.shape) < 0.1] = 0.0
    if seed % 2:
        z = (np.round(z * 1000) / 1000).astype(np.float32)
    K = ts.Intrinsics(rng.uniform(50, 900), rng.uniform(50, 900), rng.uniform(0, 128), rng.uniform(0, 96))
    x = torch.from_numpy(z).cuda()
    for f in ("fd", "sobel", "scharr", "prewitt", (0.7, 2.9)):
        for m in ("mean", "median"):
            outs = [tfn.Estimator(K, f, m, kernel=k).estimate(x).cpu().numpy() for k in ("strip", "masked", "general", "pixel")]
            for o in outs[1:]:
                assert np.array_equal(outs[0].view(np.uint32), o.view(np.uint32)), (seed, f, m)
            assert_parity(compare(outs[0], oracle.estimate(z, K, f, m), z, K), f"fuzz {seed} {f}/{m}")
