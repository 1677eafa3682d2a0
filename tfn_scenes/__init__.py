"""Seeded synthetic inputs for the 3F2N hot path — shared by the oracle tests, the
GPU parity tests and bench.py.

This module holds NONE of the 3F2N method's arithmetic (no inverse depth, no
gradient filters, no n_z candidates, no mean/median).  It only draws scenes and
ray-casts them analytically, exactly as SURVEY.md §8(d) "Synthetic inputs"
describes:

* pinhole camera K = (fx, fy, u0, v0), u = column, v = row, 0-based, rays through
  integer pixel centres (Eq. 13; SPEC S:373 — no +0.5 offset);
* analytic planes (Eq. 1: n·p + b = 0) and spheres, intersected in
  fp64, nearest hit kept, depth rounded to fp32 once; misses and holes -> Z = 0;
* exact ground-truth normals, camera-facing (<n, p> <= 0);
* disparity d = f·t_c / Z (Eq. 19), Z = 0 -> d = 0;
* counter-based per-pixel randomness (salt dropout) from an integer hash of
  (seed, global frame index, pixel index), so a frame is bit-identical whichever
  rank or chunk renders it, on CPU or GPU.

Everything is computed with one torch elementwise op per step (no fused ops, no
reductions, no pow), so the same fp64 op sequence runs on CPU and CUDA and gives
bit-identical fp32 depth (IEEE + - * / sqrt are correctly rounded on both).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

__all__ = [
    "Intrinsics", "K_VGA", "K_1080", "K_2160", "SceneBatch", "Rendered",
    "config1_scene", "random_scenes", "render", "depth_to_disparity",
    "plane_scene", "sphere_scene", "hash_uniform",
]


@dataclass(frozen=True)
class Intrinsics:
    """Pinhole intrinsics in pixels (Eq. 13)."""
    fx: float
    fy: float
    u0: float
    v0: float

    def as_tuple(self) -> Tuple[float, float, float, float]:
        return (self.fx, self.fy, self.u0, self.v0)


# config 1/2/3 use K=(500,500,320,240);
# config 4 uses the centred principal points below.
K_VGA = Intrinsics(500.0, 500.0, 320.0, 240.0)
K_1080 = Intrinsics(1000.0, 1000.0, 959.5, 539.5)
K_2160 = Intrinsics(2000.0, 2000.0, 1919.5, 1079.5)


@dataclass
class SceneBatch:
    """Per-frame analytic scene parameters (fp64 numpy arrays).

    plane_n  [F,3]  unit plane normal, camera-facing; plane_q [F,3] a point on it;
    plane_on [F]    bool — frame has a plane;
    sph_c    [F,S,3] sphere centres; sph_r [F,S] radii (0 = no sphere);
    disc     [F,D,3] hole discs (u_c, v_c, radius) in pixels (radius 0 = none);
    salt     probability of per-pixel dropout (Z=0); salt_seed its hash seed;
    frame_ids [F] global frame indices (the counter of the per-pixel hash).
    """
    plane_n: np.ndarray
    plane_q: np.ndarray
    plane_on: np.ndarray
    sph_c: np.ndarray
    sph_r: np.ndarray
    disc: np.ndarray
    salt: float = 0.0
    salt_seed: int = 0
    frame_ids: Optional[np.ndarray] = None

    @property
    def frames(self) -> int:
        return int(self.plane_n.shape[0])

    def subset(self, lo: int, hi: int) -> "SceneBatch":
        fid = self.frame_ids if self.frame_ids is not None else np.arange(self.frames)
        return SceneBatch(self.plane_n[lo:hi], self.plane_q[lo:hi], self.plane_on[lo:hi],
                          self.sph_c[lo:hi], self.sph_r[lo:hi], self.disc[lo:hi],
                          self.salt, self.salt_seed, fid[lo:hi])


@dataclass
class Rendered:
    depth: torch.Tensor          # [F,H,W] float32, 0 = invalid
    gt: torch.Tensor             # [F,3,H,W] float32 camera-facing unit normals, NaN where invalid
    depth64: Optional[torch.Tensor] = None  # [F,H,W] float64 unrounded depth (0 = miss)
    obj: Optional[torch.Tensor] = None      # [F,H,W] int8 object id: 0 none, 1 plane, 2+s sphere s


def _normalise(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def plane_scene(n, q, frames: int = 1) -> SceneBatch:
    """One plane with normal n (any sign; made camera-facing) through point q."""
    n = _normalise(np.asarray(n, dtype=np.float64))
    q = np.asarray(q, dtype=np.float64)
    if float(np.dot(n, q)) > 0.0:        # camera-facing: n·q < 0  <=>  b = -n·q > 0
        n = -n
    F = frames
    return SceneBatch(np.tile(n, (F, 1)), np.tile(q, (F, 1)), np.ones(F, bool),
                      np.zeros((F, 1, 3)), np.zeros((F, 1)), np.zeros((F, 1, 3)),
                      frame_ids=np.arange(F))


def sphere_scene(c, r, plane_n=None, plane_q=None, frames: int = 1) -> SceneBatch:
    """A sphere (centre c, radius r), optionally over a plane."""
    F = frames
    if plane_n is None:
        pn, pq, on = np.zeros((F, 3)), np.zeros((F, 3)), np.zeros(F, bool)
    else:
        base = plane_scene(plane_n, plane_q, F)
        pn, pq, on = base.plane_n, base.plane_q, base.plane_on
    return SceneBatch(pn, pq, on, np.tile(np.asarray(c, np.float64), (F, 1, 1)),
                      np.full((F, 1), float(r)), np.zeros((F, 1, 3)), frame_ids=np.arange(F))


def config1_scene() -> SceneBatch:
    """BASELINE.json configs[0] / SURVEY §8(d) config 1: plane with normal
    ∝ (0.3,-0.2,-1) through (0,0,3) plus sphere C=(0.3,-0.2,2.0), R=0.6."""
    return sphere_scene((0.3, -0.2, 2.0), 0.6, plane_n=(0.3, -0.2, -1.0), plane_q=(0.0, 0.0, 3.0))


def random_scenes(frames: int, K: Intrinsics, H: int, W: int, seed: int = 0,
                  first_frame: int = 0, holes: bool = False, salt: float = 0.0) -> SceneBatch:
    """SURVEY §8(d) config 2 recipe, one numpy Generator per global frame index
    (SeedSequence([seed, frame])) so any shard/chunk reproduces the same frames:
    plane tilted U[0,60°] about a random in-plane axis at distance U[2,6] m on the
    optical axis; 1-3 spheres R~U[0.2,0.8] m with centre depth U[1.5,4] m through a
    uniform random pixel.  holes=True adds ~2 % of the area as random discs
    (config 4); salt adds per-pixel dropout with that probability."""
    F, S, D = frames, 3, 24
    pn = np.zeros((F, 3)); pq = np.zeros((F, 3)); on = np.ones(F, bool)
    sc = np.zeros((F, S, 3)); sr = np.zeros((F, S)); disc = np.zeros((F, D, 3))
    fids = np.arange(first_frame, first_frame + F)
    for i, fid in enumerate(fids):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, int(fid)])))
        tilt = g.uniform(0.0, math.radians(60.0))
        az = g.uniform(0.0, 2.0 * math.pi)
        pn[i] = (math.sin(tilt) * math.cos(az), math.sin(tilt) * math.sin(az), -math.cos(tilt))
        pq[i] = (0.0, 0.0, g.uniform(2.0, 6.0))
        ns = int(g.integers(1, S + 1))
        for s in range(ns):
            r = g.uniform(0.2, 0.8)
            zc = g.uniform(1.5, 4.0)
            uc = g.uniform(0.0, W - 1.0)
            vc = g.uniform(0.0, H - 1.0)
            sc[i, s] = ((uc - K.u0) / K.fx * zc, (vc - K.v0) / K.fy * zc, zc)
            sr[i, s] = r
        if holes:
            mean_r = math.sqrt(0.02 * H * W / (D * math.pi))
            for d in range(D):
                disc[i, d] = (g.uniform(0.0, W - 1.0), g.uniform(0.0, H - 1.0),
                              mean_r * g.uniform(0.5, 1.5) / math.sqrt(13.0 / 12.0))
    return SceneBatch(pn, pq, on, sc, sr, disc, salt=salt, salt_seed=seed, frame_ids=fids)


# ----------------------------------------------------------------------------------
# counter-based hash (lowbias32, C. Wellons) in int64 torch ops without overflow
_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    lo = x & 0xFFFF
    hi = x >> 16
    return ((lo * c) + (((hi * c) & 0xFFFF) << 16)) & _M32


def _hash32(x: torch.Tensor) -> torch.Tensor:
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def hash_uniform(seed: int, frame_ids: torch.Tensor, npix: int, device) -> torch.Tensor:
    """[F, npix] uniform in [0,1) from hash(seed, frame, pixel) — integer ops only."""
    pix = torch.arange(npix, dtype=torch.int64, device=device)[None, :]
    f = frame_ids.to(device=device, dtype=torch.int64)[:, None]
    h = _hash32(pix ^ _hash32(f * 0x9E37 + (seed & 0xFFFF) + ((seed >> 16) & 0x7FFF) * 0x10000))
    h = _hash32(h + (f & 0xFFFF))
    return h.to(torch.float64) * (1.0 / 4294967296.0)


# ----------------------------------------------------------------------------------
def render(scenes: SceneBatch, K: Intrinsics, H: int, W: int, device="cpu",
           keep_depth64: bool = False) -> Rendered:
    """Ray-cast every frame of `scenes` at integer pixel centres (fp64), keep the
    nearest hit, round depth to fp32.  Returns depth [F,H,W] f32 (0 = invalid) and
    camera-facing GT normals [F,3,H,W] f32 (NaN = invalid)."""
    dev = torch.device(device)
    f64 = torch.float64
    F = scenes.frames
    u = torch.arange(W, dtype=f64, device=dev)
    v = torch.arange(H, dtype=f64, device=dev)
    dx = ((u - K.u0) / K.fx)[None, None, :].expand(1, H, W)      # ray (dx, dy, 1)
    dy = ((v - K.v0) / K.fy)[None, :, None].expand(1, H, W)
    inf = torch.tensor(float("inf"), dtype=f64, device=dev)

    def t(a):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=f64, device=dev)

    best = torch.full((F, H, W), float("inf"), dtype=f64, device=dev)
    gnx = torch.zeros((F, H, W), dtype=f64, device=dev)
    gny = torch.zeros_like(gnx)
    gnz = torch.zeros_like(gnx)
    obj = torch.zeros((F, H, W), dtype=torch.int8, device=dev)

    # planes:  Z = (n·q) / (n·dir)
    pn, pq = t(scenes.plane_n), t(scenes.plane_q)
    on = torch.as_tensor(scenes.plane_on, device=dev)
    nx, ny, nz = pn[:, 0, None, None], pn[:, 1, None, None], pn[:, 2, None, None]
    nq = pn[:, 0] * pq[:, 0]
    nq = nq + pn[:, 1] * pq[:, 1]
    nq = nq + pn[:, 2] * pq[:, 2]
    den = nx * dx
    den = den + ny * dy
    den = den + nz
    zp = nq[:, None, None] / den
    hit = (zp > 0) & torch.isfinite(zp) & on[:, None, None]
    zp = torch.where(hit, zp, inf)
    take = zp < best
    best = torch.where(take, zp, best)
    gnx = torch.where(take, nx.expand_as(gnx), gnx)
    gny = torch.where(take, ny.expand_as(gny), gny)
    gnz = torch.where(take, nz.expand_as(gnz), gnz)
    obj = torch.where(take, torch.ones_like(obj), obj)

    # spheres: nearest root of A Z^2 - 2 B Z + Cc = 0
    A = dx * dx
    A = A + dy * dy
    A = A + 1.0
    sc, sr = t(scenes.sph_c), t(scenes.sph_r)
    for s in range(sc.shape[1]):
        cx, cy, cz = sc[:, s, 0, None, None], sc[:, s, 1, None, None], sc[:, s, 2, None, None]
        r = sr[:, s, None, None]
        B = dx * cx
        B = B + dy * cy
        B = B + cz
        cc = cx * cx
        cc = cc + cy * cy
        cc = cc + cz * cz
        cc = cc - r * r
        disc = B * B
        disc = disc - A * cc
        ok = (disc >= 0) & (r > 0)
        root = torch.sqrt(torch.where(ok, disc, torch.zeros_like(disc)))
        zs = (B - root) / A
        ok = ok & (zs > 0)
        zs = torch.where(ok, zs, inf)
        take = zs < best
        best = torch.where(take, zs, best)
        inv_r = 1.0 / r
        gnx = torch.where(take, (zs * dx - cx) * inv_r, gnx)
        gny = torch.where(take, (zs * dy - cy) * inv_r, gny)
        gnz = torch.where(take, (zs - cz) * inv_r, gnz)
        obj = torch.where(take, torch.full_like(obj, 2 + s), obj)

    valid = torch.isfinite(best)
    # hole discs (config 4)
    if scenes.disc.shape[1] and np.any(scenes.disc[:, :, 2] > 0):
        dd = t(scenes.disc)
        uu = u[None, None, :]
        vv = v[:, None][None]
        for k in range(dd.shape[1]):
            du = uu - dd[:, k, 0, None, None]
            dv = vv - dd[:, k, 1, None, None]
            rr = dd[:, k, 2, None, None]
            d2 = du * du
            d2 = d2 + dv * dv
            valid = valid & ~(d2 <= rr * rr)
    if scenes.salt > 0:
        fids = scenes.frame_ids if scenes.frame_ids is not None else np.arange(F)
        hu = hash_uniform(scenes.salt_seed, torch.as_tensor(fids), H * W, dev).view(F, H, W)
        valid = valid & ~(hu < scenes.salt)

    depth64 = torch.where(valid, best, torch.zeros_like(best))
    depth = depth64.to(torch.float32)
    valid = valid & (depth > 0)
    nan = torch.tensor(float("nan"), dtype=f64, device=dev)
    gt = torch.stack([torch.where(valid, gnx, nan), torch.where(valid, gny, nan),
                      torch.where(valid, gnz, nan)], dim=1).to(torch.float32)
    obj = torch.where(valid, obj, torch.zeros_like(obj))
    return Rendered(depth=depth, gt=gt, depth64=depth64 if keep_depth64 else None, obj=obj)


def depth_to_disparity(depth64_or_32: torch.Tensor, f: float, baseline: float) -> torch.Tensor:
    """d = f·t_c / Z (Eq. 19) in fp64, rounded to fp32; Z<=0 -> 0."""
    z = depth64_or_32.to(torch.float64)
    fb = float(f) * float(baseline)
    d = torch.where(z > 0, fb / torch.where(z > 0, z, torch.ones_like(z)), torch.zeros_like(z))
    return d.to(torch.float32)


# ----------------------------------------------------------------------------------
# noise-robustness workload (PAPER.md supplement P:829-831, Table VII
# P:706-758; SPEC S:357-366 add_gaussian_noise, S:374 presets)
NOISE_PRESETS = {"low": 0.001, "medium": 0.003, "high": 0.01}   # sigma / mean valid depth


def add_gaussian_noise(depth: torch.Tensor, sigma_rel: float, seed: int = 0, first_frame: int = 0) -> torch.Tensor:
    """z' = z + sigma * N(0,1) on valid pixels (z > 0, finite), sigma = sigma_rel x the frame's
    mean valid depth; pixels pushed to z' <= 0 become invalid (0).  Deterministic per
    (seed, global frame id, pixel): counter-based uniforms (hash_uniform, integer ops)
    -> Box-Muller in fp64.  No 3F2N arithmetic.  CPU and GPU agree to the last few ulps
    of log/cos (not bit for bit): tests feed both sides the same host-generated frames."""
    if sigma_rel == 0:
        return depth.clone()
    F = depth.shape[0]
    npix = depth[0].numel()
    dev = depth.device
    ids = torch.arange(first_frame, first_frame + F, dtype=torch.int64)
    u1 = hash_uniform(seed * 2 + 1, ids, npix, dev)
    u2 = hash_uniform(seed * 2 + 2, ids, npix, dev)
    g = torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos((2.0 * math.pi) * u2)    # N(0,1), fp64
    z = depth.reshape(F, npix).to(torch.float64)
    valid = torch.isfinite(z) & (z > 0)
    mean = torch.where(valid, z, torch.zeros_like(z)).sum(1) / valid.sum(1).clamp(min=1)
    zn = z + (sigma_rel * mean)[:, None] * g
    zn = torch.where(valid & (zn > 0), zn, torch.zeros_like(zn))
    return zn.to(torch.float32).reshape(depth.shape)
