"""Multi-GPU plumbing for the 3F2N hot path.

Frames are independent, so a batch shards by frame with no exchange on the hot
path: rank r of G owns the contiguous global frame range shard(n, r, G).  The only
collective is one all-reduce (SUM) of the int64 angular-error statistics vector
that the a8 stats kernel accumulates (tfn_stats); integer sums are associative, so
the reduced vector is bit-identical for any G and any shard order.

torch.distributed is the plumbing: NCCL over NVLink/NVSwitch on the GPU box,
gloo for the CPU tests.
"""
from __future__ import annotations

from typing import Dict, Optional, Sequence, Tuple

import torch

STAT_KEYS = ("sum_psi_micro_deg", "m", "n_le_10", "n_le_20", "n_le_30", "n_valid_est", "n_valid_gt",
             "n_pixels")
PSI_SCALE = 1.0e6


def shard(n_frames: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous frame range [lo, hi) of `rank` out of `world` (sizes differ by <= 1)."""
    if world <= 0 or not (0 <= rank < world) or n_frames < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def chunks(lo: int, hi: int, size: int):
    """Consecutive [a, b) chunks of at most `size` frames covering [lo, hi)."""
    a = lo
    while a < hi:
        b = min(hi, a + size)
        yield a, b
        a = b


def allreduce_stats(acc: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of the int64[8] stats vector (no-op without a process group)."""
    import torch.distributed as dist
    if acc.dtype != torch.int64 or acc.numel() != len(STAT_KEYS):
        raise ValueError("stats vector must be int64[8]")
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def summarize(vec: Sequence[int]) -> Dict[str, float]:
    """PAPER.md Eq. 22-23 from the reduced vector: e_A (AAE, degrees) and e_P at 10/20/30 deg."""
    v = [int(x) for x in vec]
    m = v[1]
    out = dict(zip(STAT_KEYS, v))
    if m > 0:
        out.update(aae_deg=v[0] / PSI_SCALE / m, pgp10=v[2] / m, pgp20=v[3] / m, pgp30=v[4] / m)
    return out
