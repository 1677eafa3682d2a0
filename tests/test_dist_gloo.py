"""N>1 host logic on CPU (gloo, world size 2): frame sharding covers every frame
exactly once, and the int64 statistics all-reduce gives the single-process vector
bit for bit.  The per-frame statistics here come from the oracle
and its metrics (CPU); on the GPU the same vector comes from tfn_stats."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_08165_b200 import dist as tdist

H, W, FRAMES = 48, 64, 6
K = (60.0, 60.0, 31.5, 23.5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame_stats(lo, hi):
    """int64 stats vector of frames [lo, hi): oracle normals vs analytic GT."""
    import oracle
    import tfn_scenes as ts
    from oracle import metrics
    Ki = ts.Intrinsics(*K)
    sc = ts.random_scenes(hi - lo, Ki, H, W, seed=3, first_frame=lo)
    r = ts.render(sc, Ki, H, W)
    est = oracle.estimate(r.depth.numpy(), Ki, "sobel", "median")
    st = metrics.normal_stats(est.astype(np.float32), r.gt.numpy())
    psi = st["psi"]
    return torch.tensor([int(np.sum(np.rint(psi * tdist.PSI_SCALE).astype(np.int64))), st["m"],
                         int((psi <= 10).sum()), int((psi <= 20).sum()), int((psi <= 30).sum()),
                         st["n_valid_est"], st["n_valid_gt"], st["n_pixels"]], dtype=torch.int64)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = tdist.shard(FRAMES, rank, world)
        acc = torch.zeros(8, dtype=torch.int64)
        for a, b in tdist.chunks(lo, hi, 2):
            acc += _frame_stats(a, b)
        tdist.allreduce_stats(acc)
        q.put((rank, lo, hi, acc.tolist()))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in (0, 1, 7, 65536, 1023):
        for g in (1, 2, 3, 4, 8):
            rs = [tdist.shard(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        tdist.shard(4, 2, 2)
    assert list(tdist.chunks(3, 10, 4)) == [(3, 7), (7, 10)]


def test_allreduce_world2_bitwise():
    single = torch.zeros(8, dtype=torch.int64)
    for a, b in tdist.chunks(0, FRAMES, 3):
        single += _frame_stats(a, b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert (res[0][1], res[0][2], res[1][1], res[1][2]) == (0, 3, 3, 6)
    for _, _, _, vec in res:
        assert vec == single.tolist()          # identical on every rank, equal to G = 1
    s = tdist.summarize(res[0][3])
    assert 0.0 <= s["aae_deg"] < 5.0 and 0.9 < s["pgp30"] <= 1.0
