"""fp64 CPU oracle for the 3F2N hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
`--impl reference`) may import this package.  The product package
(paper_2005_08165_b200) never imports it, and it never imports the product: the
two share no code.

The arithmetic lives in tfn_oracle.c (plain C, fp64, the paper's Eq. 13-21
literally; see its header for citations and the ledger of readings Q1-Q14).
This module only marshals numpy arrays through ctypes, plus the paper's
accuracy metrics (metrics.py, Eq. 22-25).

Parity pins: tests/test_oracle_pins.py, tests/test_oracle_components.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_tfn.so")
_SRC = os.path.join(_HERE, "tfn_oracle.c")

FILTERS = {"fd": 0, "sobel": 1, "scharr": 2, "prewitt": 3}
MODES = {"mean": 0, "median": 1}


class _K(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("u0", ctypes.c_double), ("v0", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (fp64, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-fvisibility=hidden", _SRC, "-o", _SO + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        Kp = ctypes.POINTER(_K)
        L.orc_valid_sample.argtypes = [ctypes.c_double]; L.orc_valid_sample.restype = ctypes.c_int
        L.orc_backproject.argtypes = [Kp, ctypes.c_double, ctypes.c_double, ctypes.c_double, dp]
        L.orc_backproject_image.argtypes = [Kp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        L.orc_smallest_eigvec_sym.argtypes = [dp, ctypes.c_int, dp]; L.orc_smallest_eigvec_sym.restype = ctypes.c_int
        L.orc_plane_fit.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, Kp, ctypes.c_int, dp]
        L.orc_plane_fit.restype = ctypes.c_int
        L.orc_inverse_depth.argtypes = [ctypes.c_double]; L.orc_inverse_depth.restype = ctypes.c_double
        L.orc_disparity_to_depth.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_disparity_to_depth.restype = ctypes.c_double
        L.orc_filter_weights.argtypes = [ctypes.c_int, dp, dp]; L.orc_filter_weights.restype = ctypes.c_int
        L.orc_gradient_at.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, dp, dp]
        L.orc_nz_candidate.argtypes = [dp, dp, ctypes.c_double, ctypes.c_double]
        L.orc_nz_candidate.restype = ctypes.c_double
        L.orc_mean.argtypes = [dp, ctypes.c_int]; L.orc_mean.restype = ctypes.c_double
        L.orc_median.argtypes = [dp, ctypes.c_int]; L.orc_median.restype = ctypes.c_double
        L.orc_orient_toward_camera.argtypes = [dp, dp]
        L.orc_estimate_depth_f64.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, Kp,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_int, dp, dp]
        L.orc_estimate_depth_f64.restype = ctypes.c_int
        L.orc_estimate_disparity_f64.argtypes = [dp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, Kp, ctypes.c_double, ctypes.c_double,
                                                 ctypes.c_int, dp, dp]
        L.orc_estimate_disparity_f64.restype = ctypes.c_int
        L.orc_estimate_f32.argtypes = [fp, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, Kp, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int, dp, dp]
        L.orc_estimate_f32.restype = ctypes.c_int
        L.orc_estimate_pixel_f32.argtypes = [fp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                             ctypes.c_int, Kp, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        L.orc_estimate_pixel_f32.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _kstruct(K) -> _K:
    fx, fy, u0, v0 = (K.as_tuple() if hasattr(K, "as_tuple") else tuple(K))
    return _K(float(fx), float(fy), float(u0), float(v0))


def weights(filter) -> tuple:
    """(k_{+-1}, k_0) of the named kernel (reading Q1)."""
    if isinstance(filter, tuple):
        return filter
    kp, k0 = ctypes.c_double(), ctypes.c_double()
    if lib().orc_filter_weights(FILTERS[filter], ctypes.byref(kp), ctypes.byref(k0)) != 0:
        raise ValueError(filter)
    return kp.value, k0.value


# ---------------------------------------------------------------------- components
def valid_sample(z: float) -> bool:
    return bool(lib().orc_valid_sample(float(z)))


def backproject(K, u, v, z) -> np.ndarray:
    p = np.zeros(3)
    k = _kstruct(K)
    lib().orc_backproject(ctypes.byref(k), float(u), float(v), float(z), _dp(p))
    return p


def backproject_image(depth: np.ndarray, K) -> np.ndarray:
    """fp64 point cloud [B,3,H,W] of fp64 depth [B,H,W] (Eq. 13 per pixel,
    NaN where the sample is invalid, Q5)."""
    z = np.ascontiguousarray(depth, dtype=np.float64)
    if z.ndim == 2:
        z = z[None]
    B, H, W = z.shape
    out = np.empty((B, 3, H, W), dtype=np.float64)
    k = _kstruct(K)
    lib().orc_backproject_image(ctypes.byref(k), _dp(z), B, H, W, _dp(out))
    return out


def smallest_eigvec_sym(M: np.ndarray) -> np.ndarray:
    """SPEC S:276-280 (N4 plumbing): unit eigenvector of the smallest eigenvalue (Jacobi)."""
    m = np.ascontiguousarray(M, dtype=np.float64)
    d = m.shape[0]
    out = np.empty(d)
    if lib().orc_smallest_eigvec_sym(_dp(m), d, _dp(out)) != 0:
        raise ValueError("matrix is not symmetric")
    return out


PLANE_METHODS = {"pca": 0, "svd": 1}


def plane_fit(depth: np.ndarray, K, method: str = "pca") -> np.ndarray:
    """PlanePCA (Eq. 3) / PlaneSVD (Eq. 2) normals [B,3,H,W] fp64 of depth
    [B,H,W] (3x3 window, k >= 3 valid neighbours, border invalid, oriented
    toward the camera)."""
    z = np.ascontiguousarray(depth, dtype=np.float64)
    if z.ndim == 2:
        z = z[None]
    B, H, W = z.shape
    out = np.empty((B, 3, H, W), dtype=np.float64)
    k = _kstruct(K)
    if lib().orc_plane_fit(_dp(z), B, H, W, ctypes.byref(k), PLANE_METHODS[method], _dp(out)) != 0:
        raise ValueError(method)
    return out


def inverse_depth(z: float) -> float:
    return lib().orc_inverse_depth(float(z))


def disparity_to_depth(f_tc: float, d: float) -> float:
    return lib().orc_disparity_to_depth(float(f_tc), float(d))


def gradient_at(x: np.ndarray, v: int, u: int, filter="fd"):
    x = np.ascontiguousarray(x, dtype=np.float64)
    kp, k0 = weights(filter)
    gu, gv = ctypes.c_double(), ctypes.c_double()
    lib().orc_gradient_at(_dp(x), x.shape[0], x.shape[1], int(v), int(u), kp, k0,
                          ctypes.byref(gu), ctypes.byref(gv))
    return gu.value, gv.value


def nz_candidate(p, q, nx, ny) -> float:
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    return lib().orc_nz_candidate(_dp(p), _dp(q), float(nx), float(ny))


def aggregate(values: Sequence[float], mode: str) -> float:
    c = np.ascontiguousarray(values, dtype=np.float64).copy()
    if mode == "mean":
        return lib().orc_mean(_dp(c), len(c))
    return lib().orc_median(_dp(c), len(c))


def orient_toward_camera(n, p) -> np.ndarray:
    n = np.ascontiguousarray(n, dtype=np.float64).copy()
    p = np.ascontiguousarray(p, dtype=np.float64)
    lib().orc_orient_toward_camera(_dp(n), _dp(p))
    return n


# ---------------------------------------------------------------------- estimators
def estimate(sample: np.ndarray, K, filter="sobel", mode="median", disparity: bool = False,
             f_tc: float = 1.0, threads: int = 1) -> np.ndarray:
    """3F2N on a batch.  sample: [B,H,W] or [H,W], float32 (the exact buffer the
    GPU reads) or float64 (analytic input for pins).  Returns fp64 normals
    [B,3,H,W] (or [3,H,W]), NaN = invalid.  `threads` > 1 runs frames in parallel
    (ctypes releases the GIL) — the arithmetic per frame is unchanged."""
    squeeze = sample.ndim == 2
    s = sample[None] if squeeze else sample
    B, H, W = s.shape
    kp, k0 = weights(filter)
    md = MODES[mode]
    k = _kstruct(K)
    out = np.empty((B, 3, H, W), dtype=np.float64)
    L = lib()

    def run(lo, hi):
        work = np.empty(4 * H * W, dtype=np.float64)
        for b in range(lo, hi):
            if s.dtype == np.float32:
                fr = np.ascontiguousarray(s[b])
                rc = L.orc_estimate_f32(_fp(fr), int(disparity), float(f_tc), 1, H, W,
                                        ctypes.byref(k), kp, k0, md, _dp(out[b]), _dp(work))
            else:
                fr = np.ascontiguousarray(s[b], dtype=np.float64)
                if disparity:
                    rc = L.orc_estimate_disparity_f64(_dp(fr), float(f_tc), 1, H, W, ctypes.byref(k),
                                                      kp, k0, md, _dp(out[b]), _dp(work))
                else:
                    rc = L.orc_estimate_depth_f64(_dp(fr), 1, H, W, ctypes.byref(k), kp, k0, md,
                                                  _dp(out[b]), _dp(work))
            if rc != 0:
                raise ValueError(f"oracle rejected the arguments (status {rc})")

    if threads <= 1 or B == 1:
        run(0, B)
    else:
        per = (B + threads - 1) // threads
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: run(i * per, min(B, (i + 1) * per)), range(threads)))
    return out[0] if squeeze else out


def estimate_pixels(frame: np.ndarray, K, pixels, filter="sobel", mode="median",
                    disparity: bool = False, f_tc: float = 1.0) -> np.ndarray:
    """Oracle normals at selected (v,u) pixels of one fp32 frame -> [N,3] fp64."""
    fr = np.ascontiguousarray(frame, dtype=np.float32)
    H, W = fr.shape
    kp, k0 = weights(filter)
    k = _kstruct(K)
    out = np.empty((len(pixels), 3), dtype=np.float64)
    L = lib()
    for i, (v, u) in enumerate(pixels):
        rc = L.orc_estimate_pixel_f32(_fp(fr), int(disparity), float(f_tc), H, W, ctypes.byref(k),
                                      kp, k0, MODES[mode], int(v), int(u), _dp(out[i]))
        if rc != 0:
            raise ValueError(f"oracle rejected the arguments (status {rc})")
    return out
