"""paper_2005_08165_b200 — B200-native 3F2N (three-filters-to-normal) surface-normal
estimation (Fan et al., arXiv 2005.08165): the per-pixel hot path as fused sm_100a
CUDA kernels behind the C ABI include/tfn.h (libtfn.so), with a thin ctypes binding.

    from paper_2005_08165_b200 import Estimator
    est = Estimator((fx, fy, u0, v0), filter="sobel", nz_mode="median")
    normals = est.estimate(depth_cuda_f32)          # [B,3,H,W], NaN = invalid

See DESIGN.md for the method, the boundary and the kernel design.
"""
from .tfn import (ABI_SYMBOLS, Estimator, decode_oct16, TfnError, debug_phi8, debug_sol, lib, stats, tfn_create,  # noqa: F401
                  tfn_debug_phi8, tfn_destroy, tfn_estimate, tfn_estimate_disparity, tfn_estimate_host,
                  tfn_kernel_launches, tfn_set_layout, tfn_set_option, tfn_stats, tfn_status_string,
                  tfn_version, tfn_auto_variant, tfn_estimate_u16, tfn_estimate_host_u16, tfn_estimate_points,
                  tfn_set_filter_weights, tfn_plane_fit, STAT_KEYS,
                  LIB_PATH)

__all__ = ["Estimator", "decode_oct16", "TfnError", "stats", "debug_phi8", "lib", "LIB_PATH", "ABI_SYMBOLS", "STAT_KEYS"]
