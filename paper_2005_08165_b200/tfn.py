"""Thin ctypes binding of libtfn.so (include/tfn.h) — argument marshalling only.

Every step of the 3F2N path runs in the CUDA kernels behind the C ABI; this
module never computes normals itself and has no CPU fallback: if libtfn.so is
missing or the device is not sm_100 the calls raise.  PyTorch is used only for
device memory and streams.

Functions with the ABI's names (tfn_create, tfn_estimate, ...) take raw pointers
exactly like the C calls; `Estimator`, `stats` and `debug_phi8` wrap them for
torch tensors.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TFN_LIB") or os.path.join(_HERE, "libtfn.so")

TFN_OK, TFN_ERR_INVALID_ARGUMENT, TFN_ERR_CONFIG, TFN_ERR_CUDA = 0, 1, 2, 3
FILTERS = {"fd": 0, "sobel": 1, "scharr": 2, "prewitt": 3, "custom": 4}
MODES = {"mean": 0, "median": 1}
LAYOUTS = {"planar": 0, "packed": 1}
KERNELS = {"auto": 0, "pixel": 1, "strip": 2, "general": 3, "masked": 4, "f32": 5, "f32masked": 6}
OUT_DTYPES = {"f32": 0, "f16": 1, "oct16": 2}
OPT_KERNEL, OPT_STRIP_H, OPT_GRID, OPT_DYNAMIC, OPT_OUT_DTYPE, OPT_COUNT_SPECIAL = 0, 1, 2, 3, 4, 5

# every symbol include/tfn.h declares (tests/test_abi.py checks the export table)
ABI_SYMBOLS = (
    "tfn_create", "tfn_set_layout", "tfn_set_option", "tfn_estimate", "tfn_estimate_disparity",
    "tfn_estimate_host", "tfn_stats", "tfn_debug_phi8", "tfn_destroy", "tfn_status_string",
    "tfn_kernel_launches", "tfn_version", "tfn_debug_sol", "tfn_auto_variant", "tfn_estimate_u16",
    "tfn_estimate_host_u16", "tfn_estimate_points", "tfn_set_filter_weights", "tfn_plane_fit",
    "tfn_debug_auto", "tfn_debug_special_count",
)
PLANE_METHODS = {"pca": 0, "svd": 1}
INPUT_KINDS = {"depth": 0, "disparity": 1, "depth_u16": 2}


class TfnError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {tfn_status_string(status)} ({status})")


class tfn_intrinsics(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("u0", ctypes.c_double), ("v0", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libtfn.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built — run `python -m paper_2005_08165_b200.build` "
                              "(the 3F2N path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, d, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
        L.tfn_create.argtypes = [ctypes.POINTER(tfn_intrinsics), i, i, ctypes.POINTER(vp)]
        L.tfn_set_layout.argtypes = [vp, i]
        L.tfn_set_option.argtypes = [vp, i, ll]
        L.tfn_estimate.argtypes = [vp, vp, i, i, i, vp, vp]
        L.tfn_estimate_disparity.argtypes = [vp, vp, d, i, i, i, vp, vp]
        L.tfn_estimate_host.argtypes = [vp, vp, i, d, i, i, i, vp, vp]
        L.tfn_estimate_u16.argtypes = [vp, vp, d, i, i, i, vp, vp]
        L.tfn_estimate_host_u16.argtypes = [vp, vp, d, i, i, i, vp, vp]
        L.tfn_estimate_points.argtypes = [vp, vp, i, d, i, i, i, vp, vp, vp]
        L.tfn_set_filter_weights.argtypes = [vp, d, d]
        L.tfn_plane_fit.argtypes = [vp, vp, i, i, i, i, vp, vp]
        L.tfn_stats.argtypes = [vp, vp, i, i, i, i, vp, vp]
        L.tfn_debug_phi8.argtypes = [vp, ll, i, vp, vp, vp]
        L.tfn_debug_sol.argtypes = [vp, i, i, i, vp, vp]
        L.tfn_destroy.argtypes = [vp]
        L.tfn_auto_variant.argtypes = [vp, ctypes.POINTER(i)]
        L.tfn_debug_auto.argtypes = [i, i, d, ctypes.c_uint, i, ctypes.POINTER(i), ctypes.POINTER(i),
                                     ctypes.POINTER(i)]
        L.tfn_debug_special_count.argtypes = [vp, ctypes.POINTER(ll)]
        L.tfn_status_string.argtypes = [i]
        L.tfn_status_string.restype = ctypes.c_char_p
        L.tfn_kernel_launches.restype = ctypes.c_ulonglong
        for name in ABI_SYMBOLS:
            f = getattr(L, name)
            if f.restype is ctypes.c_int or name in ("tfn_create", "tfn_set_layout", "tfn_set_option",
                                                     "tfn_estimate", "tfn_estimate_disparity",
                                                     "tfn_estimate_host", "tfn_stats", "tfn_debug_phi8",
                                                     "tfn_destroy", "tfn_version", "tfn_debug_sol",
                                                     "tfn_auto_variant", "tfn_estimate_u16",
                                                     "tfn_estimate_host_u16", "tfn_estimate_points",
                                                     "tfn_set_filter_weights", "tfn_plane_fit",
                                                     "tfn_debug_auto", "tfn_debug_special_count"):
                f.restype = ctypes.c_int
        _lib = L
    return _lib


# ----------------------------------------------------------------- ABI-named calls
def tfn_debug_special_count(h: int) -> int:
    n = ctypes.c_longlong()
    _check(lib().tfn_debug_special_count(h, ctypes.byref(n)), "tfn_debug_special_count")
    return n.value


def tfn_status_string(status: int) -> str:
    try:
        return lib().tfn_status_string(int(status)).decode()
    except ImportError:
        return str(status)


def _check(rc: int, where: str):
    if rc != TFN_OK:
        raise TfnError(rc, where)


def tfn_create(K, filter: int, nz_mode: int) -> int:
    fx, fy, u0, v0 = K.as_tuple() if hasattr(K, "as_tuple") else tuple(K)
    k = tfn_intrinsics(float(fx), float(fy), float(u0), float(v0))
    h = ctypes.c_void_p()
    _check(lib().tfn_create(ctypes.byref(k), int(filter), int(nz_mode), ctypes.byref(h)), "tfn_create")
    return h.value


def tfn_plane_fit(h: int, depth_ptr: int, method: int, batch: int, H: int, W: int, stream: int,
                  out_ptr: int) -> int:
    return lib().tfn_plane_fit(h, depth_ptr, int(method), batch, H, W, stream, out_ptr)


def tfn_set_filter_weights(h: int, kp: float, k0: float) -> None:
    _check(lib().tfn_set_filter_weights(h, float(kp), float(k0)), "tfn_set_filter_weights")


def tfn_set_layout(h: int, layout: int) -> None:
    _check(lib().tfn_set_layout(h, int(layout)), "tfn_set_layout")


def tfn_set_option(h: int, option: int, value: int) -> None:
    _check(lib().tfn_set_option(h, int(option), int(value)), "tfn_set_option")


def tfn_estimate(h: int, depth_ptr: int, batch: int, H: int, W: int, stream: int, out_ptr: int) -> int:
    return lib().tfn_estimate(h, depth_ptr, batch, H, W, stream, out_ptr)


def tfn_estimate_u16(h: int, codes_ptr: int, depth_scale: float, batch: int, H: int, W: int, stream: int,
                     out_ptr: int) -> int:
    return lib().tfn_estimate_u16(h, codes_ptr, float(depth_scale), batch, H, W, stream, out_ptr)


def tfn_estimate_host_u16(h: int, host_codes: int, depth_scale: float, batch: int, H: int, W: int,
                          host_out: int, stream: int) -> int:
    return lib().tfn_estimate_host_u16(h, host_codes, float(depth_scale), batch, H, W, host_out, stream)


def tfn_estimate_points(h: int, in_ptr: int, input_kind: int, scale: float, batch: int, H: int, W: int,
                        stream: int, out_ptr: int, pts_ptr: int) -> int:
    return lib().tfn_estimate_points(h, in_ptr, int(input_kind), float(scale), batch, H, W, stream, out_ptr,
                                     pts_ptr)


def tfn_estimate_disparity(h: int, disp_ptr: int, baseline_times_f: float, batch: int, H: int, W: int,
                           stream: int, out_ptr: int) -> int:
    return lib().tfn_estimate_disparity(h, disp_ptr, float(baseline_times_f), batch, H, W, stream, out_ptr)


def tfn_estimate_host(h: int, host_in: int, is_disparity: int, baseline_times_f: float, batch: int,
                      H: int, W: int, host_out: int, stream: int) -> int:
    return lib().tfn_estimate_host(h, host_in, int(is_disparity), float(baseline_times_f), batch, H, W,
                                   host_out, stream)


def tfn_stats(est_ptr: int, gt_ptr: int, batch: int, H: int, W: int, layout: int, stream: int,
              stats_ptr: int) -> int:
    return lib().tfn_stats(est_ptr, gt_ptr, batch, H, W, layout, stream, stats_ptr)


def tfn_debug_phi8(cand_ptr: int, n: int, nz_mode: int, out_ptr: int, k_ptr: int, stream: int) -> int:
    return lib().tfn_debug_phi8(cand_ptr, n, nz_mode, out_ptr, k_ptr, stream)


def tfn_debug_sol(in_ptr: int, batch: int, H: int, W: int, stream: int, out_ptr: int) -> int:
    return lib().tfn_debug_sol(in_ptr, batch, H, W, stream, out_ptr)


def debug_sol(x: torch.Tensor, out: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> None:
    """SOL traffic-mix copy (4 B in, 12 B out per pixel), for the roofline context."""
    B, H, W = _bhw(x)
    _check(tfn_debug_sol(x.data_ptr(), B, H, W, _stream_ptr(stream), out.data_ptr()), "tfn_debug_sol")


def tfn_destroy(h: int) -> int:
    return lib().tfn_destroy(h)


def tfn_kernel_launches() -> int:
    return int(lib().tfn_kernel_launches())


def tfn_version() -> int:
    return int(lib().tfn_version())


def tfn_auto_variant(h: int) -> int:
    """The strip variant AUTO currently picks for handle h: 2 fast, 4 masked, 3 general."""
    v = ctypes.c_int(0)
    _check(lib().tfn_auto_variant(h, ctypes.byref(v)), "tfn_auto_variant")
    return v.value


def tfn_debug_auto(state: int, probed: int, rate: float, call: int, can_probe: bool):
    """Host-only AUTO state machine probe: (next_state, run, probe) — states / runs 0 fast,
    1 masked, 2 general (include/tfn.h)."""
    ns, run, pr = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().tfn_debug_auto(state, probed, rate, call, int(can_probe), ctypes.byref(ns), ctypes.byref(run),
                                ctypes.byref(pr)), "tfn_debug_auto")
    return ns.value, run.value, bool(pr.value)


# ----------------------------------------------------------------- tensor helpers
def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _need(t: torch.Tensor, name: str, device: bool = True, dtype=torch.float32):
    if t.dtype != dtype or not t.is_contiguous():
        raise TfnError(TFN_ERR_INVALID_ARGUMENT, f"{name} must be a contiguous {dtype} tensor")
    if device and not t.is_cuda:
        raise TfnError(TFN_ERR_INVALID_ARGUMENT, f"{name} must be a CUDA tensor")


def _bhw(x: torch.Tensor) -> Tuple[int, int, int]:
    if x.dim() == 2:
        return 1, x.shape[0], x.shape[1]
    if x.dim() == 3:
        return x.shape[0], x.shape[1], x.shape[2]
    raise TfnError(TFN_ERR_INVALID_ARGUMENT, "input must be [H,W] or [B,H,W]")


class Estimator:
    """One tfn handle: intrinsics K=(fx,fy,u0,v0), gradient kernel, Phi, layout."""

    def __init__(self, K, filter: str = "sobel", nz_mode: str = "median", layout: str = "planar",
                 kernel: str = "auto", strip_h: int = 0, grid: int = 0, dynamic: bool = True,
                 out_dtype: str = "f32"):
        self.K = K.as_tuple() if hasattr(K, "as_tuple") else tuple(float(x) for x in K)
        self.filter, self.nz_mode, self.layout = filter, nz_mode, layout
        self.out_dtype = out_dtype
        self._odt = {"f32": torch.float32, "f16": torch.float16, "oct16": torch.int16}[out_dtype]
        self._nc = 2 if out_dtype == "oct16" else 3        # stored components per pixel
        # filter: a name, or the (kp, k0) weights of [kp k0 kp]^T (x) [-1 0 1] (TFN_FILTER_CUSTOM)
        custom = isinstance(filter, (tuple, list))
        self.h = tfn_create(self.K, FILTERS["custom" if custom else filter], MODES[nz_mode])
        if custom:
            tfn_set_filter_weights(self.h, float(filter[0]), float(filter[1]))
        tfn_set_layout(self.h, LAYOUTS[layout])
        tfn_set_option(self.h, OPT_KERNEL, KERNELS[kernel])
        tfn_set_option(self.h, OPT_STRIP_H, strip_h)
        tfn_set_option(self.h, OPT_GRID, grid)
        tfn_set_option(self.h, OPT_DYNAMIC, int(dynamic))
        tfn_set_option(self.h, OPT_OUT_DTYPE, OUT_DTYPES[out_dtype])

    def _shape(self, B, H, W):
        return (B, self._nc, H, W) if self.layout == "planar" else (B, H, W, self._nc)

    def _out(self, B, H, W, like: torch.Tensor, out):
        if out is None:
            out = torch.empty(self._shape(B, H, W), dtype=self._odt, device=like.device)
        _need(out, "out", device=like.is_cuda, dtype=self._odt)
        if out.numel() != self._nc * B * H * W:
            raise TfnError(TFN_ERR_INVALID_ARGUMENT, "out has the wrong size")
        return out

    def estimate(self, depth: torch.Tensor, out: Optional[torch.Tensor] = None,
                 stream: Optional[torch.cuda.Stream] = None, depth_scale: float = 1e-3) -> torch.Tensor:
        """depth: CUDA fp32 [B,H,W] / [H,W], or uint16 depth codes (Z = code * depth_scale;
        the scale is validated and cancels)."""
        B, H, W = _bhw(depth)
        if depth.dtype == torch.uint16:
            _need(depth, "depth", dtype=torch.uint16)
            out = self._out(B, H, W, depth, out)
            _check(tfn_estimate_u16(self.h, depth.data_ptr(), depth_scale, B, H, W, _stream_ptr(stream),
                                    out.data_ptr()), "tfn_estimate_u16")
            return out
        _need(depth, "depth")
        out = self._out(B, H, W, depth, out)
        _check(tfn_estimate(self.h, depth.data_ptr(), B, H, W, _stream_ptr(stream), out.data_ptr()),
               "tfn_estimate")
        return out

    def estimate_disparity(self, disp: torch.Tensor, baseline_times_f: float,
                           out: Optional[torch.Tensor] = None,
                           stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        _need(disp, "disparity")
        B, H, W = _bhw(disp)
        out = self._out(B, H, W, disp, out)
        _check(tfn_estimate_disparity(self.h, disp.data_ptr(), baseline_times_f, B, H, W,
                                      _stream_ptr(stream), out.data_ptr()), "tfn_estimate_disparity")
        return out

    def estimate_points(self, x: torch.Tensor, scale: float = 1.0, disparity: bool = False,
                        out: Optional[torch.Tensor] = None, points: Optional[torch.Tensor] = None,
                        stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
        """N3: normals and the fp32 point cloud (same layout) in one pass.  x: fp32 depth
        (Z = scale * x), fp32 disparity (disparity=True, Z = scale / d, scale = f * t_c) or
        uint16 depth codes (Z = scale * code)."""
        B, H, W = _bhw(x)
        if x.dtype == torch.uint16:
            _need(x, "depth", dtype=torch.uint16)
            kind = INPUT_KINDS["depth_u16"]
        else:
            _need(x, "depth")
            kind = INPUT_KINDS["disparity" if disparity else "depth"]
        out = self._out(B, H, W, x, out)
        if points is None:
            shape = (B, 3, H, W) if self.layout == "planar" else (B, H, W, 3)
            points = torch.empty(shape, dtype=torch.float32, device=x.device)
        _need(points, "points")
        if points.numel() != 3 * B * H * W:
            raise TfnError(TFN_ERR_INVALID_ARGUMENT, "points has the wrong size")
        _check(tfn_estimate_points(self.h, x.data_ptr(), kind, scale, B, H, W, _stream_ptr(stream),
                                   out.data_ptr(), points.data_ptr()), "tfn_estimate_points")
        return out, points

    def plane_fit(self, depth: torch.Tensor, method: str = "pca", out: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """N4 comparator: PlanePCA / PlaneSVD normals (fp32, the handle's layout)."""
        _need(depth, "depth")
        B, H, W = _bhw(depth)
        if out is None:
            shape = (B, 3, H, W) if self.layout == "planar" else (B, H, W, 3)
            out = torch.empty(shape, dtype=torch.float32, device=depth.device)
        _need(out, "out")
        _check(tfn_plane_fit(self.h, depth.data_ptr(), PLANE_METHODS[method], B, H, W, _stream_ptr(stream),
                             out.data_ptr()), "tfn_plane_fit")
        return out

    def estimate_host(self, host_in: torch.Tensor, is_disparity: bool = False, baseline_times_f: float = 1.0,
                      out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None,
                      depth_scale: float = 1e-3) -> torch.Tensor:
        """Host buffers in and out (pinned for full overlap); blocking.  host_in fp32 (depth, or
        disparity with baseline_times_f = f * t_c) or uint16 depth codes (Z = code * depth_scale)."""
        u16 = host_in.dtype == torch.uint16
        _need(host_in, "host_in", device=False, dtype=torch.uint16 if u16 else torch.float32)
        if host_in.is_cuda:
            raise TfnError(TFN_ERR_INVALID_ARGUMENT, "host_in must be a CPU tensor")
        B, H, W = _bhw(host_in)
        if out is None:
            out = torch.empty(self._shape(B, H, W), dtype=self._odt, pin_memory=True)
        _need(out, "out", device=False, dtype=self._odt)
        if out.numel() != self._nc * B * H * W:
            raise TfnError(TFN_ERR_INVALID_ARGUMENT, "out has the wrong size")
        if u16:
            _check(tfn_estimate_host_u16(self.h, host_in.data_ptr(), depth_scale, B, H, W, out.data_ptr(),
                                         _stream_ptr(stream)), "tfn_estimate_host_u16")
        else:
            _check(tfn_estimate_host(self.h, host_in.data_ptr(), int(is_disparity), baseline_times_f, B, H, W,
                                     out.data_ptr(), _stream_ptr(stream)), "tfn_estimate_host")
        return out

    def close(self):
        if getattr(self, "h", None):
            tfn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats(est: torch.Tensor, gt: torch.Tensor, layout: str = "planar", acc: Optional[torch.Tensor] = None,
          stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Accumulate the a8 statistics of est vs gt into acc (int64[8] on the device)."""
    _need(est, "est")
    _need(gt, "gt")
    B, H, W = gt.shape[0], gt.shape[2], gt.shape[3]
    if acc is None:
        acc = torch.zeros(8, dtype=torch.int64, device=est.device)
    _check(tfn_stats(est.data_ptr(), gt.data_ptr(), B, H, W, LAYOUTS[layout], _stream_ptr(stream),
                     acc.data_ptr()), "tfn_stats")
    return acc


def debug_phi8(cand: torch.Tensor, nz_mode: str) -> Tuple[torch.Tensor, torch.Tensor]:
    """P8 probe: device Phi of [n,8] candidates (non-finite = skipped); nz_mode 'mean',
    'median' or 'median_ext' (the strip kernel's fast-path median decision)."""
    _need(cand, "cand")
    n = cand.numel() // 8
    out = torch.empty(n, dtype=torch.float32, device=cand.device)
    k = torch.empty(n, dtype=torch.int32, device=cand.device)
    mode = 2 if nz_mode == "median_ext" else MODES[nz_mode]
    _check(tfn_debug_phi8(cand.data_ptr(), n, mode, out.data_ptr(), k.data_ptr(),
                          _stream_ptr(None)), "tfn_debug_phi8")
    return out, k


def decode_oct16(q: torch.Tensor, layout: str = "planar") -> torch.Tensor:
    """Unit normals (fp32, planar [B,3,H,W] or packed [B,H,W,3]) from TFN_OUT_OCT16 pairs
    (include/tfn.h); the sentinel (-32768, -32768) decodes to NaN.  Plain torch ops."""
    u, v = (q[:, 0], q[:, 1]) if layout == "planar" else (q[..., 0], q[..., 1])
    bad = (u == -32768) & (v == -32768)
    px = (u.float() / 32767.0).clamp(-1, 1)
    py = (v.float() / 32767.0).clamp(-1, 1)
    z = 1.0 - px.abs() - py.abs()
    sx = torch.where(px >= 0, 1.0, -1.0)
    sy = torch.where(py >= 0, 1.0, -1.0)
    fx = torch.where(z < 0, (1.0 - py.abs()) * sx, px)
    fy = torch.where(z < 0, (1.0 - px.abs()) * sy, py)
    vec = torch.stack([fx, fy, z], dim=1 if layout == "planar" else -1)
    vec = vec / vec.norm(dim=1 if layout == "planar" else -1, keepdim=True)
    sign = torch.tensor([1.0, 1.0, -1.0], device=q.device)
    n = vec * (sign.view(1, 3, 1, 1) if layout == "planar" else sign)
    nan = torch.full_like(n, float("nan"))
    return torch.where((bad.unsqueeze(1) if layout == "planar" else bad.unsqueeze(-1)), nan, n)


STAT_KEYS = ("sum_psi_micro_deg", "m", "n_le_10", "n_le_20", "n_le_30", "n_valid_est", "n_valid_gt",
             "n_pixels")
