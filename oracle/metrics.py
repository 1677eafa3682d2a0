"""The paper's accuracy metrics in fp64 numpy — TEST INFRASTRUCTURE ONLY (oracle).

PAPER.md §IV-A, P:293-327:
  Eq. 22  e_A = (1/m) sum_k psi_k            e_P(phi) = (1/m) sum_k delta(psi_k, phi)
  Eq. 23  delta(psi, phi) = 1 iff psi <= phi
  Eq. 24  psi_k = arccos(<n_k, n^_k> / (|n_k| |n^_k|))
  Eq. 25  pi = e_A * t

Reading Q16: psi is evaluated as atan2(|a x b|, a.b) — the same angle as Eq. 24,
but well conditioned near 0 (cos(1e-3 deg) = 1 - 1.5e-10).
Reading Q18: pooled over the pixels valid in both maps, across all frames.
"""
from __future__ import annotations

import numpy as np


def angular_error_deg(a: np.ndarray, b: np.ndarray, axis: int = -1) -> np.ndarray:
    """psi (Eq. 24) in degrees between vectors along `axis` (fp64)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    cr = np.cross(a, b, axis=axis)
    num = np.sqrt(np.sum(cr * cr, axis=axis))
    den = np.sum(a * b, axis=axis)
    return np.degrees(np.arctan2(num, den))


def aae(psi) -> float:
    """Eq. 22 left: average angular error."""
    psi = np.asarray(psi, dtype=np.float64)
    if psi.size == 0:
        raise ValueError("empty error list")
    return float(np.mean(psi))


def pgp(psi, phi: float) -> float:
    """Eq. 22-23: proportion of good pixels, psi <= phi."""
    psi = np.asarray(psi, dtype=np.float64)
    if psi.size == 0:
        raise ValueError("empty error list")
    return float(np.count_nonzero(psi <= phi)) / psi.size


def pi_score(e_a: float, t_ms: float) -> float:
    """Eq. 25."""
    return float(e_a) * float(t_ms)


STAT_PHIS = (10.0, 20.0, 30.0)   # Table IV's tolerances
PSI_SCALE = 1.0e6                # fixed point: 1e-6 degree units


def normal_stats(est: np.ndarray, gt: np.ndarray) -> dict:
    """Pooled stats of estimated vs GT normal maps [B,3,H,W] over pixels valid in
    both (Q18).  Mirrors the vector the GPU stats kernel all-reduces."""
    e = np.moveaxis(np.asarray(est, np.float64), 1, -1).reshape(-1, 3)
    g = np.moveaxis(np.asarray(gt, np.float64), 1, -1).reshape(-1, 3)
    ve = np.all(np.isfinite(e), axis=1)
    vg = np.all(np.isfinite(g), axis=1)
    both = ve & vg
    psi = angular_error_deg(e[both], g[both])
    out = {
        "m": int(both.sum()),
        "sum_psi_deg": float(psi.sum()),
        "n_valid_est": int(ve.sum()),
        "n_valid_gt": int(vg.sum()),
        "n_pixels": int(e.shape[0]),
    }
    for phi in STAT_PHIS:
        out[f"n_le_{int(phi)}"] = int(np.count_nonzero(psi <= phi))
    out["psi"] = psi
    return out
