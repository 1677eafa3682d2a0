// tfn_strip.cuh — the production 3F2N kernel (instantiated per filter in
// tfn_strip_<filter>.cu via tfn_strip_inst.cuh).
//
// Geometry.  One warp owns a strip of 32*PPL columns (PPL = 4: 128) x strip_h rows of one
// frame; each lane owns PPL adjacent columns and walks down the strip with a rolling
// window of three row "slots" (rows v-1, v, v+1).  The row loop is unrolled by 3 and the
// slots rotate by renaming (no register copies).  Per lane-row, fp32 input: rows of 136
// columns x 8 arrive as TMA boxes in a per-warp shared-memory ring (tfn_tma.cuh; the fast and
// masked median variants instead load one LDG.128 + two predicated halo loads three rows
// ahead into registers — measured faster there, except FD); uint16 input: one cp.async of 8 B into a per-warp ring
// TFN_CPA_D rows ahead (halo words by the edge lanes), read back with LDS; out: three STG.128
// (fp32) / STG.64 (half) / one or two vector stores (oct16).  Persistent grid (12 warps/SM;
// FD + mean 16); strips handed out by an atomic work counter (dynamic scheduling).
//
// Arithmetic (bit-identical to tfn_pixel_kernel, see tfn_device.cuh, except FD32 below):
//   fp64:  w = 1/z (faithful, ~2^-66), D_h, D_v, g_u, g_v in the oracle's order,
//          s = g_u + g_v, t = g_v - g_u, rounded once to fp32;
//   fp32:  one MUFU reciprocal per neighbour PAIR (shared by both pixels of the pair),
//          tau = fma(m Z_c, R, +-m), Phi (24-op median network with NaN-propagating
//          min / max and an extreme-magnitude finiteness test / mean), n_z, normalise,
//          orient — packed FMUL2/FFMA2/FADD2 over pixel pairs (0,1), (2,3).
//   FD32:  disparity FD fast / masked only — the gradients in fp32.
// Three variants (KV), bit-identical, picked at run time by AUTO (tfn_abi.cu):
//   fast (0):    all 8 candidates finite and Phi != 0 (no skips, no flat rule, no
//                orientation tie, valid pixel) in registers; anything else ("special":
//                holes, invalid samples, dZ == 0, flat, ties) runs the exact per-pixel
//                routine behind ONE warp vote per row step.  Border pixels are never
//                special: their out-of-image taps are NaN, so the fast path already
//                writes the canonical NaN.
//   general (1): no special path — invalid samples get NaN fp64 x (F2F), skipped
//                candidates are padded in registers (phi_any), flat / none / ties /
//                invalid resolved by finish_tail2: the per-pixel kernel's arithmetic.
//   masked (2):  the fast variant whose special test also requires every Q4 tap to be
//                valid (per-row sign-byte masks of the sanitized samples): a pixel beside
//                a hole is already the canonical NaN, so holes and dropout stay fast.
#pragma once

#ifndef TFN_U16_MINBLOCKS
#define TFN_U16_MINBLOCKS 4      // resident CTAs per SM of the uint16 (ring) instantiations (128 registers: +2.3 % over 3)
#endif
#ifndef TFN_CPA_D
#define TFN_CPA_D 4              // cp.async ring prefetch distance (rows), <= 8 (r02 A/B on config 6: 4 > 8 > 6 by ~1 %)
#endif
#ifndef TFN_STRIP_PPL
#define TFN_STRIP_PPL 4          // pixels (columns) per lane: 4 or 2
#endif
#ifndef TFN_PHI_EXT
#define TFN_PHI_EXT 1            // median fast / masked: finiteness from the network's extremes, no candidate sum
#endif
#ifndef TFN_FD32
#define TFN_FD32 1               // disparity FD fast / masked: fp32 gradients (FD32_ON, fd_dw)
#endif
#ifndef TFN_STRIP_TMA
#define TFN_STRIP_TMA 1          // fp32 input rows through the per-warp TMA ring (tfn_tma.cuh) instead of
#endif                           // the three-rows-ahead register prefetch
#include "tfn_tma.cuh"

namespace tfn {

constexpr int PPL = TFN_STRIP_PPL;
constexpr int STRIP_COLS = 32 * PPL;     // columns per warp strip
static_assert(PPL == 2 || PPL == 4, "TFN_STRIP_PPL must be 2 or 4");

struct Slot {
    float raw[6];      // samples of columns c0-1 .. c0+4 as loaded
    bool rok;          // the row exists (loads were issued)
    float z[6];        // sanitized (invalid -> NaN)
    double w[6];       // x = 1/z (depth) or d (disparity), fp64
    double head[4];    // kp*D_h(row-1) + k0*D_h(row)   (D_h re-derived from w when needed)
    float wf[6];       // FD32: x = 1/z (depth, MUFU) or d (disparity) in fp32
    float rN[4], rNW[4], rNE[4];   // pair reciprocals of the N / NW / NE neighbours (pairs owned by the row above)
    unsigned hb;       // masked variant: byte i bit 7 set iff a sample of columns i..i+2 is invalid
    unsigned cb;       //   (FD) byte i bit 7 set iff the sample of column i+1 is invalid
};

template <class T>
struct StripCtx {
    const T* img;      // frame base (fp32 samples or uint16 depth codes)
    const T* pm;       // frame base + clamped column of the lane's 4-vector
    int cm;            // clamped first column of the lane
    float u0;
    int H, W;
    bool okm, okl, okr;   // lane's columns / left halo / right halo inside the image
    float fx, fy;
    float a[4];        // u - u0 of the 4 columns
    int* fired;        // AUTO probe: += 1 per row step that needed the special path
    int outk;          // normal encoding: 0 fp32, 1 IEEE half, 2 octahedral int16 pair (N1)
    float* pts;        // N3: this lane's point-cloud output (column cm) of the item's frame, or nullptr
    float pscale, ifx, ify;   // Z = pscale * sample (depth) or pscale / d (disparity); 1/fx, 1/fy
    Wts wt;            // CUSTOM filter weights
    float v0;
    int y1;            // end row of the current strip
    unsigned ring;     // shared-memory address of this warp's row ring (uint16 input)
    int lane;
    ring::Ring* rg;    // fp32 input with TFN_STRIP_TMA: this warp's TMA row ring
    const CUtensorMap* tm;
    int ys;            //   first output row of the current strip (ring row = v - ys + 1)
};



// uint16 code -> float, exactly, without a conversion instruction: 2^23 + code has the code
// in its low mantissa bits (PRMT builds the word, one FADD removes the 2^23)
__device__ __forceinline__ float code_lo(unsigned x) { return __uint_as_float(__byte_perm(x, 0x4B00u, 0x5410)) - 8388608.0f; }
__device__ __forceinline__ float code_hi(unsigned x) { return __uint_as_float(__byte_perm(x, 0x4B00u, 0x5432)) - 8388608.0f; }

// Row staging.  fp32 input: register window, LDG three rows ahead (load_raw).  uint16 input
// (N1): a per-warp shared-memory ring filled by cp.async TFN_CPA_D rows ahead — measured
// +20 % on uint16 codes -> half normals (158.8 vs 132.0 Gpx/s), but -5 % on the fp32 fast
// variant and +-0.5 % on the fp32 general one, so fp32 keeps the register window (and 3
// CTAs/SM: 4 with 128 registers runs the general variant 8 % slower).
template <class T, bool GEN> struct Ring { static constexpr bool on = sizeof(T) == 2; };
// The ring: 8 rows per warp, RB bytes per row: [12 B pad | left halo word | the
// strip's 32*PPL samples | right halo word | pad]; lane l's vector at byte 16 + l*PPL*sizeof(T)
constexpr int RING_RB = 16 + 32 * 4 * 4 + 16;

__device__ __forceinline__ void cpa(unsigned dst, const void* src, int bytes_ok, int size) {
    if (size == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(bytes_ok) : "memory");
    else if (size == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(dst), "l"(src), "r"(bytes_ok) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(dst), "l"(src), "r"(bytes_ok) : "memory");
}
__device__ __forceinline__ unsigned ring_base() {
    __shared__ __align__(16) char ring[TFN_STRIP_THREADS / 32][8][RING_RB];
    return (unsigned)__cvta_generic_to_shared(&ring[threadIdx.x >> 5][0][0]);
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// issue row v of the strip into its ring slot; rows outside the image, halos outside the
// image and lanes past W are zero-filled (0 is an invalid sample: Q5), so the sanitize needs
// no position predicates
template <class T>
__device__ __forceinline__ void issue_row(const StripCtx<T>& c, int v) {
    const bool rin = (v >= 0) && (v < c.H);
    const unsigned slot = c.ring + ((v + 1) & 7) * RING_RB;
    TFN_CHECK(c.cm >= 0 && c.cm + PPL <= c.W && 16 + c.lane * PPL * (int)sizeof(T) + PPL * (int)sizeof(T) <= RING_RB - 16);
    const T* row = c.pm + (rin ? v : 0) * c.W;
    constexpr int VB = PPL * sizeof(T);
    cpa(slot + 16 + c.lane * VB, row, (rin && c.okm) ? VB : 0, VB);
    // halo words: fp32 the sample itself; uint16 the aligned pair holding it
    // (zero-filled halos keep an in-image source address: nothing is read from it)
    if (c.lane == 0) cpa(slot + 12, reinterpret_cast<const char*>(row) - (c.okl ? 4 : 0), (rin && c.okl) ? 4 : 0, 4);
    if (c.lane == 31) cpa(slot + 16 + 32 * VB, row + (c.okr ? PPL : 0), (rin && c.okr) ? 4 : 0, 4);
}
__device__ __forceinline__ void fetch_row(Slot& s, const StripCtx<unsigned short>& c, int v) {
    const char* slot = reinterpret_cast<const char*>(__cvta_shared_to_generic(c.ring + ((v + 1) & 7) * RING_RB));
    const char* me = slot + 16 + c.lane * 8;
    const uint2 m = *reinterpret_cast<const uint2*>(me);
    s.raw[1] = code_lo(m.x); s.raw[2] = code_hi(m.x); s.raw[3] = code_lo(m.y); s.raw[4] = code_hi(m.y);
    s.raw[0] = code_hi(*reinterpret_cast<const unsigned*>(me - 4));
    s.raw[5] = code_lo(*reinterpret_cast<const unsigned*>(me + 8));
    s.rok = true;
}

// row v of the lane's window: one LDG.128 (fp32) or LDG.64 (uint16) + two halo loads at
// immediate offsets, predicated off outside the image (never an out-of-bounds address)
__device__ __forceinline__ void load_raw(Slot& s, const StripCtx<float>& c, int v) {
    s.rok = (v >= 0) && (v < c.H);
    const float* row = c.pm + v * c.W;
    TFN_CHECK(c.cm >= 0 && c.cm + PPL <= c.W && (!c.okl || c.cm >= 1) && (!c.okr || c.cm + PPL < c.W));
    if (s.rok) {
        if (PPL == 4) {
            const float4 m = __ldg(reinterpret_cast<const float4*>(row));
            s.raw[1] = m.x; s.raw[2] = m.y; s.raw[3] = m.z; s.raw[4] = m.w;
        } else {
            const float2 m = __ldg(reinterpret_cast<const float2*>(row));
            s.raw[1] = m.x; s.raw[2] = m.y;
        }
    }
    if (s.rok && c.okl) s.raw[0] = __ldg(row - 1);
    if (s.rok && c.okr) s.raw[PPL + 1] = __ldg(row + PPL);
}
__device__ __forceinline__ void load_raw(Slot& s, const StripCtx<unsigned short>& c, int v) {
    s.rok = (v >= 0) && (v < c.H);
    TFN_CHECK(c.cm >= 0 && c.cm + PPL <= c.W && (!c.okl || c.cm >= 1) && (!c.okr || c.cm + PPL < c.W));
    const unsigned short* row = c.pm + v * c.W;
    if (s.rok) {
        if (PPL == 4) {
            const uint2 m = __ldg(reinterpret_cast<const uint2*>(row));
            s.raw[1] = code_lo(m.x); s.raw[2] = code_hi(m.x); s.raw[3] = code_lo(m.y); s.raw[4] = code_hi(m.y);
        } else {
            const unsigned m = __ldg(reinterpret_cast<const unsigned*>(row));
            s.raw[1] = code_lo(m); s.raw[2] = code_hi(m);
        }
    }
    if (s.rok && c.okl) s.raw[0] = code_lo(__ldg(row - 1));
    if (s.rok && c.okr) s.raw[PPL + 1] = code_lo(__ldg(row + PPL));
}

// Q5 for the fast path: valid iff finite and >= FLT_MIN (rejects 0, negatives, NaN,
// +-Inf, subnormals).  An invalid sample becomes NaN, which makes every candidate that
// uses it NaN and so sends the pixel to the exact path.
// VM (masked variant): the NaN carries the sign bit, so an OR of sample bits is negative
// iff one of them is invalid (the special test below)
template <bool VM> constexpr int bad_z() { return VM ? (int)0xffffffff : 0x7fffffff; }
template <bool VM>
__device__ __forceinline__ float sanitize_fast(float z, bool ok) {
    const bool good = valid_bits(z) & ok;      // no short circuit: FSEL, not a branch
    return good ? z : __int_as_float(bad_z<VM>());
}

template <bool DISP, bool GEN, class T, bool VM = false, bool G32 = false>
__device__ __forceinline__ void prepare(Slot& s, const StripCtx<T>& c) {
    // the lane's own columns need only the value test; the halos are outside the image at
    // the first / last lane of a frame row; whole rows outside the image (loads predicated
    // off, stale registers) take a warp-uniform, rare branch — measured +1.9 % over
    // per-sample row predicates.  Lanes past W never store, so their stale samples need no NaN.
    s.z[0] = sanitize_fast<VM>(s.raw[0], Ring<T, GEN>::on || c.okl);
#pragma unroll
    for (int j = 1; j <= PPL; ++j) s.z[j] = valid_bits(s.raw[j]) ? s.raw[j] : __int_as_float(bad_z<VM>());
    s.z[PPL + 1] = sanitize_fast<VM>(s.raw[PPL + 1], Ring<T, GEN>::on || c.okr);
    if (!Ring<T, GEN>::on && __any_sync(0xffffffffu, !s.rok)) {
#pragma unroll
        for (int j = 0; j < PPL + 2; ++j) s.z[j] = s.rok ? s.z[j] : __int_as_float(bad_z<VM>());
    }
    if (VM && PPL == 4) {
        // an invalid sample is a NaN with the sign bit set: OR the row's 3-column windows and
        // gather the four sign bytes (PRMT) — the tap test of the masked variant's vote
        int h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __float_as_int(s.z[i]) | __float_as_int(s.z[i + 1]) | __float_as_int(s.z[i + 2]);
        // (only bit 7 of each byte is ever tested: the other bits are left as gathered)
        s.hb = __byte_perm(__byte_perm(h[0], h[1], 0x0073), __byte_perm(h[2], h[3], 0x0073), 0x5410);
        s.cb = __byte_perm(__byte_perm(__float_as_int(s.z[1]), __float_as_int(s.z[2]), 0x0073),
                           __byte_perm(__float_as_int(s.z[3]), __float_as_int(s.z[4]), 0x0073), 0x5410);
    }
    // exact for every valid sample; invalid ones give finite garbage here, but their
    // NaN z makes the pixel "special", which recomputes it exactly
    if constexpr (G32) {
#pragma unroll
        for (int j = 0; j < PPL + 2; ++j) s.wf[j] = DISP ? s.z[j] : rcp_approx(s.z[j]);
        return;
    }
#pragma unroll
    for (int j = 0; j < PPL + 2; ++j) {
        // fast variant: integer widening (exact for the positive normal floats every valid
        // sample is; invalid ones give garbage, but their NaN z makes the pixel special).
        // General variant: the F2F conversion, so an invalid sample's x is NaN and every
        // gradient that uses it is NaN: the pixel comes out invalid (Q4) without a special
        // path (measured: F2F is 4 % slower in the fast variant, 1 % faster in the general)
        const double x = GEN ? (double)s.z[j] : widen_pos(s.z[j]);
        s.w[j] = DISP ? x : rcp_rn(x);
    }
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// normals are written once and never re-read: streaming (evict-first) stores
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}
__device__ __forceinline__ unsigned h2(float a, float b) {      // RN to half, NaN stays NaN
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const unsigned*>(&h);
}
__device__ __forceinline__ void st4h(void* p, float a, float b, float c, float d) {
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(h2(a, b), h2(c, d)));
}
__device__ __forceinline__ void st2(float* p, float a, float b) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(a, b));
}
__device__ __forceinline__ void st2h(void* p, float a, float b) {
    __stcs(reinterpret_cast<unsigned*>(p), h2(a, b));
}
// N1 octahedral encoding of a unit normal in two int16 snorms (4 B/pixel), camera hemisphere
// (n_z <= 0) in the inner diamond: encode (n_x, n_y, -n_z) by the standard octahedral map,
// fold the far hemisphere, round to nearest of 32767 steps (the FFMA against 1.5 * 2^23 puts
// the rounded integer in the low mantissa bits: no conversion instruction).  NaN (invalid)
// -> the sentinel pair (-32768, -32768), which the encoder never produces otherwise.
__device__ __forceinline__ unsigned oct16(float x, float y, float z) {
    const float zz = -z;
    const float inv = rcp_approx(fabsf(x) + fabsf(y) + fabsf(zz));
    float px = x * inv, py = y * inv;
    if (zz < 0.f) {
        const float ax = fabsf(px), ay = fabsf(py);
        px = copysignf(1.f - ay, px);
        py = copysignf(1.f - ax, py);
    }
    px = fminf(fmaxf(px, -1.f), 1.f);
    py = fminf(fmaxf(py, -1.f), 1.f);
    const unsigned qx = __float_as_uint(__fmaf_rn(px, 32767.f, 12582912.f)) - 0x4B400000u;
    const unsigned qy = __float_as_uint(__fmaf_rn(py, 32767.f, 12582912.f)) - 0x4B400000u;
    const unsigned w = (qx & 0xffffu) | (qy << 16);
    return isnan(x) ? 0x80008000u : w;
}
__device__ __forceinline__ void store_oct(short* o, long long plane, const float* x, const float* y,
                                          const float* z, bool planar) {
    unsigned w[4];
#pragma unroll
    for (int i = 0; i < PPL; ++i) w[i] = oct16(x[i], y[i], z[i]);
    if (planar) {      // u plane, v plane: PPL shorts each
        if (PPL == 4) {
            __stcs(reinterpret_cast<uint2*>(o), make_uint2(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410)));
            __stcs(reinterpret_cast<uint2*>(o + plane), make_uint2(__byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632)));
        } else {
            __stcs(reinterpret_cast<unsigned*>(o), __byte_perm(w[0], w[1], 0x5410));
            __stcs(reinterpret_cast<unsigned*>(o + plane), __byte_perm(w[0], w[1], 0x7632));
        }
    } else {           // packed (u, v) per pixel
        if (PPL == 4) __stcs(reinterpret_cast<uint4*>(o), make_uint4(w[0], w[1], w[2], w[3]));
        else __stcs(reinterpret_cast<uint2*>(o), make_uint2(w[0], w[1]));
    }
}
// one component plane (or the packed triples) of the lane's PPL pixels
__device__ __forceinline__ void store_planar(float* o, const float* x) {
    if (PPL == 4) st4(o, x[0], x[1], x[2], x[3]); else st2(o, x[0], x[1]);
}
__device__ __forceinline__ void store_planar(__half* o, const float* x) {
    if (PPL == 4) st4h(o, x[0], x[1], x[2], x[3]); else st2h(o, x[0], x[1]);
}
__device__ __forceinline__ void store_packed(float* o, const float* x, const float* y, const float* z) {
    if (PPL == 4) {
        st4(o, x[0], y[0], z[0], x[1]);
        st4(o + 4, y[1], z[1], x[2], y[2]);
        st4(o + 8, z[2], x[3], y[3], z[3]);
    } else {
        st2(o, x[0], y[0]); st2(o + 2, z[0], x[1]); st2(o + 4, y[1], z[1]);
    }
}
__device__ __forceinline__ void store_packed(__half* o, const float* x, const float* y, const float* z) {
    if (PPL == 4) {
        st4h(o, x[0], y[0], z[0], x[1]);
        st4h(o + 4, y[1], z[1], x[2], y[2]);
        st4h(o + 8, z[2], x[3], y[3], z[3]);
    } else {
        st2h(o, x[0], y[0]); st2h(o + 2, z[0], x[1]); st2h(o + 4, y[1], z[1]);
    }
}

// One row step: output row v.  P = slot(v-1) (only P.w is read; P.raw holds row v+2 in
// flight), C = slot(v) (C.raw receives row v+3), N = slot(v+1) (N.raw loaded; the rest
// computed here).
// TMA row staging (tfn_tma.cuh) for fp32 input.  A/B on configs[1] (r02, 1024 x 480x640, Sobel):
// median fast 211 (TMA) vs 218 (register prefetch), masked 211 vs 212, general 176 vs 172; mean
// fast 261 vs 252, masked 263 vs 247, general 168 vs 177 Gpx/s — the register window already
// loads every sample once (loads are 1/4 of the traffic), so the ring only removes the prefetch
// registers; it stays off where it measured slower (fast and masked median — configs[3], the
// masked variant's workload: 203.2 vs 199.6 — and general mean), except FD median, whose
// freed registers buy 16 warps/SM.
#ifndef TFN_STRIP_TMA_ALL
#define TFN_STRIP_TMA_ALL 0      // 1: every fp32 variant through the ring (A/B builds)
#endif
#ifndef TFN_FD_MEDIAN16
#define TFN_FD_MEDIAN16 1        // FD + median fast / masked: TMA ring + 16 warps/SM (128 registers, no spills): 220 -> 231 Gpx/s
#endif
template <int F, class T, int MODE, bool GEN, bool VM>
constexpr bool TMA_ON = (TFN_STRIP_TMA != 0) && (sizeof(T) == 4) &&
                        (TFN_STRIP_TMA_ALL || (TFN_FD_MEDIAN16 && F == FD && !GEN) ||
                         (!(MODE == MEDIAN && !GEN) && !(MODE == MEAN && GEN)));

// FD32 (fast / masked FD on fp32 disparity): the gradients in fp32 (fd_dw below) — no fp64, no
// F2F on the XU, which bounds the mean mode.  Measured (r02, configs[1]-sized batches):
// disparity FD + mean 312 -> 336 Gpx/s, FD + median 252 -> 255; on depth each difference costs
// 3 fp32 ops instead of one fp64 subtraction (91 vs 77 instr/px: 265 vs 291 Gpx/s; median 182
// vs 220), so depth keeps the fp64 path
template <int F, int MODE, bool DISP, bool GEN, class T>
constexpr bool FD32_ON = TFN_FD32 && F == FD && DISP && !GEN && sizeof(T) == 4;

// w_b - w_a for two samples: disparity x = d, so d_b - d_a; depth x = 1/z, so
// (z_a - z_b) w_a w_b — the difference of the samples is exact (Sterbenz) or rounded once, and
// every step is a product: a few ulp relative, whatever the cancellation in w_b - w_a
template <bool DISP>
__device__ __forceinline__ float fd_dw(float za, float wa, float zb, float wb) {
    return DISP ? __fsub_rn(zb, za) : __fmul_rn(__fmul_rn(__fsub_rn(za, zb), wa), wb);
}

// the fp64 path's s, t of one FD pixel (out of line: the rare fallback of fd_dw's re-paired sums)
template <bool DISP>
__device__ __noinline__ float2 fd_st64(float zW, float zE, float zN, float zS) {
    auto x64 = [](float z) { return DISP ? widen_pos(z) : rcp_rn(widen_pos(z)); };
    const double gu = __dsub_rn(x64(zE), x64(zW));
    const double gv = __dsub_rn(x64(zS), x64(zN));
    return make_float2(__double2float_rn(__dadd_rn(gu, gv)), __double2float_rn(__dsub_rn(gv, gu)));
}

template <int F, int MODE, bool DISP, int LAYOUT, bool GEN, class T, bool PTS, int OUT, bool VM = false>
__device__ __forceinline__ void row_step(Slot& P, Slot& C, Slot& N, int v, const StripCtx<T>& c,
                                         char* __restrict__ out, long long HW,
                                         unsigned colmask, float vf) {
    if constexpr (Ring<T, GEN>::on) {
        // ring: rows up to v+D-1 in flight; row v+1 is complete once at most D-2 groups are pending
        if (v + TFN_CPA_D - 1 <= c.y1) issue_row(c, v + TFN_CPA_D - 1);
        cpa_commit();
        cpa_wait<TFN_CPA_D - 2>();
        __syncwarp();                                // halo words come from the neighbour lanes' copies
        fetch_row(N, c, v + 1);
    } else if (TMA_ON<F, T, MODE, GEN, VM>) {
        ring::ring_row(c.tm, *c.rg, v + 2 - c.ys, c.lane, N.raw);   // row v+1 from the TMA ring
        N.rok = true;                                // rows outside the image arrive zero-filled
    } else {
        load_raw(C, c, v + 3);                       // prefetch three rows ahead (C.raw is free)
    }
    constexpr bool G32 = FD32_ON<F, MODE, DISP, GEN, T>;
    prepare<DISP, GEN, T, VM, G32>(N, c);
    // masked variant (VM): special (below) = Phi non-finite or zero at a pixel whose Q4 taps (all 9; FD: the plus)
    // are valid.  An invalid sample is a NaN with the sign bit set, so the OR of the taps'
    // bits is negative iff one is invalid — and then the fast path has already produced the
    // canonical NaN (that tap's candidate is NaN).  Image borders (out-of-image taps) and
    // lanes past W need no separate mask.
    unsigned tapok = 0;
    if (VM) {
        // all 9 taps (FD: the plus) valid <=> no sign byte set in the rows' window masks
        const unsigned bad = Taps<F>::corners ? (P.hb | C.hb | N.hb) : (C.hb | P.cb | N.cb);
        tapok = ~bad;                // bit 8i+7 set iff pixel i's taps are all valid
    }

    float gu32[4], gv32[4], s32[4], t32[4];
    if constexpr (G32) {
        // ---- FD gradients in fp32: g_u = w_E - w_W and g_v = w_S - w_N are single
        //      differences; s = g_u + g_v and t = g_v - g_u re-paired along the diagonals,
        //      s = (w_E - w_N) + (w_S - w_W), t = (w_S - w_E) + (w_W - w_N).  A pair of opposite
        //      sign can cancel: those pixels take s, t from the fp64 path (rare on surfaces) ----
        unsigned bad = 0;
#pragma unroll
        for (int i = 0; i < PPL; ++i) {
            const float zW = C.z[i], wW = C.wf[i], zE = C.z[i + 2], wE = C.wf[i + 2];
            const float zN = P.z[i + 1], wN = P.wf[i + 1], zS = N.z[i + 1], wS = N.wf[i + 1];
            gu32[i] = fd_dw<DISP>(zW, wW, zE, wE);
            gv32[i] = fd_dw<DISP>(zN, wN, zS, wS);
            const float d1 = fd_dw<DISP>(zN, wN, zE, wE), d2 = fd_dw<DISP>(zW, wW, zS, wS);
            const float d3 = fd_dw<DISP>(zE, wE, zS, wS), d4 = fd_dw<DISP>(zN, wN, zW, wW);
            s32[i] = __fadd_rn(d1, d2);
            t32[i] = __fadd_rn(d3, d4);
            const unsigned x = (__float_as_uint(d1) ^ __float_as_uint(d2)) | (__float_as_uint(d3) ^ __float_as_uint(d4));
            bad |= (x >> 31) << i;
        }
        if (__any_sync(0xffffffffu, bad != 0)) {
#pragma unroll
            for (int i = 0; i < PPL; ++i) {
                if (bad & (1u << i)) {
                    const float2 st = fd_st64<DISP>(C.z[i], C.z[i + 2], P.z[i + 1], N.z[i + 1]);
                    s32[i] = st.x;
                    t32[i] = st.y;
                }
            }
        }
    } else {
    // ---- fp64 gradients (Eq. 15), oracle order (Q10) ----
    double gu[4], gv[4];
    double dv[6];
#pragma unroll
    for (int j = 0; j < PPL + 2; ++j)
        dv[j] = (Taps<F>::corners || (j >= 1 && j <= PPL)) ? __dsub_rn(N.w[j], P.w[j]) : 0.0;
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        const double dhn = __dsub_rn(N.w[i + 2], N.w[i]);          // D_h(v+1)
        const double dhc = Taps<F>::corners ? __dsub_rn(C.w[i + 2], C.w[i]) : 0.0;   // D_h(v)
        gu[i] = grad_tail<F>(C.head[i], dhn, c.wt);
        N.head[i] = grad_head<F>(dhc, dhn, c.wt);
        gv[i] = grad_tail<F>(grad_head<F>(dv[i], dv[i + 1], c.wt), dv[i + 2], c.wt);
    }
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        gu32[i] = __double2float_rn(gu[i]);
        gv32[i] = __double2float_rn(gv[i]);
        s32[i] = __double2float_rn(__dadd_rn(gu[i], gv[i]));
        t32[i] = __double2float_rn(__dsub_rn(gv[i], gu[i]));
    }
    }

    // ---- rho of the 8 neighbours (order E W S N SE NW SW NE) and the next row's N/NW/NE ----
    // one MUFU reciprocal per neighbour PAIR; index j <-> column c0 + j - 1:
    //   rE[j] (v,j)->(v,j+1), rS (v,c)->(v+1,c), rSE[j] (v,j)->(v+1,j+1), rSW[j] (v,j+1)->(v+1,j)
    const float b = __fsub_rn(vf, c.v0);        // b = v - v0 (same formula as pixel_general)
    float nx[4], ny[4], nz[4];
    unsigned special = 0;
    float rEp = pair_rcp<DISP>(C.z[0], C.z[1]);
    float rSEp = pair_rcp<DISP>(C.z[0], N.z[1]);
    float rSWp = pair_rcp<DISP>(C.z[1], N.z[0]);
#pragma unroll
    for (int q = 0; q < PPL / 2; ++q) {
        float R[2][8];      // pair reciprocals of the 8 neighbours, order E W S N SE NW SW NE
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = 2 * q + h;
            const float zc = C.z[i + 1];
            const float rE = pair_rcp<DISP>(zc, C.z[i + 2]);
            const float rS = pair_rcp<DISP>(zc, N.z[i + 1]);
            const float rSE = pair_rcp<DISP>(zc, N.z[i + 2]);
            const float rSW = pair_rcp<DISP>(C.z[i + 2], N.z[i + 1]);
            R[h][0] = rE;  R[h][1] = rEp;  R[h][2] = rS;  R[h][3] = C.rN[i];
            R[h][4] = rSE; R[h][5] = C.rNW[i]; R[h][6] = rSWp; R[h][7] = C.rNE[i];
            // the next row's N / NW / NE pairs are owned by this row
            N.rN[i] = rS; N.rNW[i] = rSEp; N.rNE[i] = rSW;
            rEp = rE; rSEp = rSE; rSWp = rSW;
        }
        const int i0 = 2 * q, i1 = 2 * q + 1;
        const float2 mu = f2(gu32[i0], gu32[i1]), mv = f2(gv32[i0], gv32[i1]);
        const float2 ms = f2(s32[i0], s32[i1]), mt = f2(t32[i0], t32[i1]);
        const float2 zc2 = f2(C.z[i0 + 1], C.z[i1 + 1]);
        // m~ = m * own sample (tfn_device.cuh: tau_owner / tau_other)
        const float2 xu = __fmul2_rn(mu, zc2), xv = __fmul2_rn(mv, zc2);
        const float2 xs = __fmul2_rn(ms, zc2), xt = __fmul2_rn(mt, zc2);
        float2 tau[8];
        float2 sum8;
        if (MODE == MEAN) {
            // mean numerator by neighbour-direction pairs (tfn_device.cuh, finish32): the
            // +-m of opposite candidates cancel exactly, sum = sum_dir x_dir (R_a + R_b)
            const float2 p23 = __fmul2_rn(xv, __fadd2_rn(f2(R[0][2], R[1][2]), f2(R[0][3], R[1][3])));
            const float2 p67 = __fmul2_rn(xt, __fadd2_rn(f2(R[0][6], R[1][6]), f2(R[0][7], R[1][7])));
            const float2 s0 = __ffma2_rn(xu, __fadd2_rn(f2(R[0][0], R[1][0]), f2(R[0][1], R[1][1])), p23);
            const float2 s1 = __ffma2_rn(xs, __fadd2_rn(f2(R[0][4], R[1][4]), f2(R[0][5], R[1][5])), p67);
            sum8 = __fadd2_rn(s0, s1);
            if (GEN) {       // the general variant's k < 8 fallback needs the candidates
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                    const float2 m = (k < 2) ? mu : (k < 4) ? mv : (k < 6) ? ms : mt;
                    tau[k] = DISP ? __fmul2_rn(x, f2(R[0][k], R[1][k]))
                                  : __ffma2_rn(x, f2(R[0][k], R[1][k]), (k & 1) ? f2(-m.x, -m.y) : m);
                }
            }
        } else if (TFN_PHI_EXT && !GEN) {
            // median, fast / masked: candidates only — finiteness comes from the network (mid_pair8_ext)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                const float2 m = (k < 2) ? mu : (k < 4) ? mv : (k < 6) ? ms : mt;
                tau[k] = DISP ? __fmul2_rn(x, f2(R[0][k], R[1][k]))
                              : __ffma2_rn(x, f2(R[0][k], R[1][k]), (k & 1) ? f2(-m.x, -m.y) : m);
            }
            sum8 = f2(0.f, 0.f);
        } else if (DISP) {
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
                const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                tau[k] = __fmul2_rn(x, f2(R[0][k], R[1][k]));
            }
            // finish32's explicit-FMA sum (median: only its finiteness is used)
            const float2 s01 = __ffma2_rn(xu, f2(R[0][1], R[1][1]), tau[0]);
            const float2 s23 = __ffma2_rn(xv, f2(R[0][3], R[1][3]), tau[2]);
            const float2 s45 = __ffma2_rn(xs, f2(R[0][5], R[1][5]), tau[4]);
            const float2 s67 = __ffma2_rn(xt, f2(R[0][7], R[1][7]), tau[6]);
            sum8 = __fadd2_rn(__fadd2_rn(s01, s23), __fadd2_rn(s45, s67));
#pragma unroll
            for (int k = 1; k < 8; k += 2) {
                const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                tau[k] = __fmul2_rn(x, f2(R[0][k], R[1][k]));
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                const float2 m = (k < 2) ? mu : (k < 4) ? mv : (k < 6) ? ms : mt;
                tau[k] = __ffma2_rn(x, f2(R[0][k], R[1][k]), (k & 1) ? f2(-m.x, -m.y) : m);
            }
            sum8 = __fadd2_rn(__fadd2_rn(__fadd2_rn(tau[0], tau[1]), __fadd2_rn(tau[2], tau[3])),
                              __fadd2_rn(__fadd2_rn(tau[4], tau[5]), __fadd2_rn(tau[6], tau[7])));
        }
        if (GEN) {
            // general variant: skipped candidates, flat, ties and invalid pixels handled in
            // registers by the same arithmetic as the per-pixel kernel (bit-identical results)
            float ph[2];
            bool none[2], okc[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float t[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) t[k] = h ? tau[k].y : tau[k].x;
                int kk;
                ph[h] = phi_any<MODE>(t, h ? sum8.y : sum8.x, kk);
                none[h] = kk == 0;
                okc[h] = !isnan(C.z[2 * q + h + 1]);
            }
            Normal n0, n1;
            finish_tail2(okc, mu, mv, f2(ph[0], ph[1]), none, f2(c.a[i0], c.a[i1]), b, c.fx, c.fy, n0, n1);
            nx[i0] = n0.x; ny[i0] = n0.y; nz[i0] = n0.z;
            nx[i1] = n1.x; ny[i1] = n1.y; nz[i1] = n1.z;
            continue;
        }
        float2 phi;
        if (MODE == MEAN) {
            phi = __fmul2_rn(sum8, f2(0.125f, 0.125f));
            phi = __ffma2_rn(f2(0.f, 0.f), sum8, phi);        // +-inf sum -> NaN Phi (special)
        } else {
            float t0[8], t1[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) { t0[k] = tau[k].x; t1[k] = tau[k].y; }
            float a0, b0, a1, b1;
            if (TFN_PHI_EXT) {
                float e0, e1;
                mid_pair8_ext(t0, a0, b0, e0);
                mid_pair8_ext(t1, a1, b1, e1);
                sum8 = f2(e0, e1);       // finite iff all 8 candidates are
            } else {
                mid_pair8(t0, a0, b0);
                mid_pair8(t1, a1, b1);
            }
            phi = __fmul2_rn(__fadd2_rn(f2(a0, a1), f2(b0, b1)), f2(0.5f, 0.5f));
            // FMNMX drops NaN candidates: make Phi NaN when any candidate is non-finite, so
            // pixels with out-of-image taps (the border, never "special") come out NaN
            phi = __ffma2_rn(f2(0.f, 0.f), sum8, phi);
        }
        // n' = (fx g_u, fy g_v, -(a g_u + b g_v + Phi))
        const float2 nzneg = __ffma2_rn(f2(c.a[i0], c.a[i1]), mu, __ffma2_rn(f2(b, b), mv, phi));
        const float2 px = __fmul2_rn(f2(c.fx, c.fx), mu);
        const float2 py = __fmul2_rn(f2(c.fy, c.fy), mv);
        const float2 pz = f2(-nzneg.x, -nzneg.y);
        const float2 dot = __ffma2_rn(px, px, __ffma2_rn(py, py, __fmul2_rn(pz, pz)));
        // flip iff Phi < 0 (ties Phi == 0 are special): sc = copysign(rsqrt(dot), Phi)
        const float r0 = __uint_as_float(__float_as_uint(rsqrt_approx(dot.x)) | (__float_as_uint(phi.x) & 0x80000000u));
        const float r1 = __uint_as_float(__float_as_uint(rsqrt_approx(dot.y)) | (__float_as_uint(phi.y) & 0x80000000u));
        const float2 sc = f2(r0, r1);
        const float2 ox = __fmul2_rn(px, sc), oy = __fmul2_rn(py, sc), oz = __fmul2_rn(pz, sc);
        nx[i0] = ox.x; nx[i1] = ox.y; ny[i0] = oy.x; ny[i1] = oy.y; nz[i0] = oz.x; nz[i1] = oz.y;
        // special: a non-finite candidate or Phi == 0 at a pixel whose centre is valid (an
        // invalid centre poisons every candidate through m~ = m * NaN: the fast path
        // already wrote the canonical NaN).  Phi is NaN iff a candidate is non-finite (the
        // folds above), so one compare per pixel covers both.
        if (VM) {
            const bool sp0 = !(fabsf(phi.x) > 0.f) && (tapok & (0x80u << (8 * i0)));
            const bool sp1 = !(fabsf(phi.y) > 0.f) && (tapok & (0x80u << (8 * i1)));
            special |= (sp0 ? (1u << i0) : 0u) | (sp1 ? (1u << i1) : 0u);
        } else {
            const bool sp0 = !(fabsf(phi.x) > 0.f) && !isnan(zc2.x);
            const bool sp1 = !(fabsf(phi.y) > 0.f) && !isnan(zc2.y);
            special |= (sp0 ? (1u << i0) : 0u) | (sp1 ? (1u << i1) : 0u);
        }
    }

    // ---- known-invalid pixels (image border, columns past W) are never special: their
    //      out-of-image taps are NaN, so the fast path already produced the canonical NaN ----
    if (!VM) {
        const bool row_border = (v == 0) || (v == c.H - 1);
        special &= row_border ? 0u : ~colmask;
    }
    if (!GEN && __any_sync(0xffffffffu, special != 0)) {
        if (c.fired && (threadIdx.x & 31) == 0) atomicAdd(c.fired, 1);
        // rare: skipped candidates, flat / tie, invalid samples -> exact per-pixel path
        // (re-reads the 3x3 from L1; bit-identical to tfn_pixel_kernel)
        for (int i = 0; i < PPL; ++i) {
            if (special & (1u << i)) {
                const Normal n = pixel_general<F, MODE, DISP>(c.img, c.H, c.W, v, c.cm + i, c.u0, c.v0,
                                                              c.fx, c.fy, c.wt);
                nx[i] = n.x; ny[i] = n.y; nz[i] = n.z;
            }
        }
    }
    // ---- store (16-B / 8-B aligned: W % 4 == 0, c0 % 4 == 0).  OUT: 0 fp32, 1 half, 3 oct16,
    //      2 the handle's choice at run time (general variant); points are general-only ----
    if (c.okm) {
        TFN_CHECK(v >= 0 && v < c.H && c.cm >= 0 && c.cm + PPL <= c.W);
        const int kind = (OUT == 2) ? c.outk : (OUT == 3 ? 2 : OUT);
        if (kind == 2) {
            short* o = reinterpret_cast<short*>(out) + v * c.W * (LAYOUT == 0 ? 1 : 2);
            store_oct(o, HW, nx, ny, nz, LAYOUT == 0);
        } else if (kind == 0) {
            float* o = reinterpret_cast<float*>(out) + v * c.W * (LAYOUT == 0 ? 1 : 3);
            if (LAYOUT == 0) {
                store_planar(o, nx);
                store_planar(o + HW, ny);
                store_planar(o + 2 * HW, nz);
            } else {
                store_packed(o, nx, ny, nz);
            }
        } else {
            __half* o = reinterpret_cast<__half*>(out) + v * c.W * (LAYOUT == 0 ? 1 : 3);
            if (LAYOUT == 0) {
                store_planar(o, nx);
                store_planar(o + HW, ny);
                store_planar(o + 2 * HW, nz);
            } else {
                store_packed(o, nx, ny, nz);
            }
        }
        // ---- N3: the point cloud beside the normals, Eq. 13: p = Z (a/fx, b/fy, 1) ----
        if (PTS) {
            float X[4], Y[4], Z[4];
#pragma unroll
            for (int i = 0; i < PPL; ++i) {
                const float zs = C.z[i + 1];             // NaN for an invalid sample
                Z[i] = DISP ? __fdiv_rn(c.pscale, zs) : __fmul_rn(zs, c.pscale);
                X[i] = __fmul_rn(__fmul_rn(c.a[i], Z[i]), c.ifx);
                Y[i] = __fmul_rn(__fmul_rn(b, Z[i]), c.ify);
            }
            float* q = c.pts + v * c.W * (LAYOUT == 0 ? 1 : 3);
            if (LAYOUT == 0) {
                store_planar(q, X);
                store_planar(q + HW, Y);
                store_planar(q + 2 * HW, Z);
            } else {
                store_packed(q, X, Y, Z);
            }
        }
    }
}

// Rows [ys, y1) of one strip: prologue, then the rolling window down the strip.
template <int F, int MODE, bool DISP, int LAYOUT, bool GEN, class T, bool PTS, int OUT, bool VM = false>
__device__ __forceinline__ void strip_rows(const StripCtx<T>& c, char* out, long long HW,
                                          unsigned colmask, int ys, int y1) {
    Slot S0, S1, S2;
    if constexpr (Ring<T, GEN>::on) {
        // prologue: rows ys-1 .. ys+D-2 issued (one group each), rows ys-1 (S0), ys (S1) prepared.
        // The previous strip's last fetches read neighbour lanes' halo words from slots these
        // copies may overwrite: order them (with dynamic scheduling the item shuffle
        // already did)
        __syncwarp();
    #pragma unroll
        for (int r = -1; r <= TFN_CPA_D - 2; ++r) {
            if (ys + r <= y1) issue_row(c, ys + r);
            cpa_commit();
        }
        cpa_wait<TFN_CPA_D - 2>();
        __syncwarp();
        fetch_row(S0, c, ys - 1);
        fetch_row(S1, c, ys);
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S0, c);
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S1, c);
    } else if (TMA_ON<F, T, MODE, GEN, VM>) {
        // prologue: rows ys-1 (S0), ys (S1) from the ring, prepared
        ring::ring_row(c.tm, *c.rg, 0, c.lane, S0.raw);
        ring::ring_row(c.tm, *c.rg, 1, c.lane, S1.raw);
        S0.rok = S1.rok = true;
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S0, c);
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S1, c);
    } else {
        // prologue: rows ys-1 (S0), ys (S1) prepared; row ys+1 (S2) loaded
        load_raw(S0, c, ys - 1);
        load_raw(S1, c, ys);
        load_raw(S2, c, ys + 1);
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S0, c);
        prepare<DISP, GEN, T, VM, FD32_ON<F, MODE, DISP, GEN, T>>(S1, c);
        load_raw(S0, c, ys + 2);
    }
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        if constexpr (!FD32_ON<F, MODE, DISP, GEN, T>)
            S1.head[i] = grad_head<F>(Taps<F>::corners ? __dsub_rn(S0.w[i + 2], S0.w[i]) : 0.0,
                                      __dsub_rn(S1.w[i + 2], S1.w[i]), c.wt);
        const float zc = S1.z[i + 1];
        S1.rN[i] = pair_rcp<DISP>(S0.z[i + 1], zc);
        S1.rNW[i] = pair_rcp<DISP>(S0.z[i], zc);
        S1.rNE[i] = pair_rcp<DISP>(S0.z[i + 2], zc);
    }
    float vf = __int2float_rn(ys);      // exact row index as float (rows < 2^24)
    for (int v = ys; v < y1; v += 3) {
        row_step<F, MODE, DISP, LAYOUT, GEN, T, PTS, OUT, VM>(S0, S1, S2, v, c, out, HW, colmask, vf);
        if (v + 1 >= y1) break;
        row_step<F, MODE, DISP, LAYOUT, GEN, T, PTS, OUT, VM>(S1, S2, S0, v + 1, c, out, HW, colmask, vf + 1.0f);
        if (v + 2 >= y1) break;
        row_step<F, MODE, DISP, LAYOUT, GEN, T, PTS, OUT, VM>(S2, S0, S1, v + 2, c, out, HW, colmask, vf + 2.0f);
        vf += 3.0f;
    }
}

// resident CTAs per SM the register budget is sized for: 3 (168 registers, 12 warps) by
// default; the uint16 ring instantiations 4 (128); the fp32 FD fast / masked instantiations
// TFN_STRIP_MINBLOCKS_FDMEAN (no corner taps: with the TMA ring for the median they are the
// only ones that fit 128 registers without spills)
#ifndef TFN_STRIP_MINBLOCKS_FDMEAN
#define TFN_STRIP_MINBLOCKS_FDMEAN 4        // measured: FD + mean 274.5 -> 290.7, FD + median 220 -> 231 Gpx/s (16 vs 12 warps/SM, r02)
#endif
template <int F, int MODE, int KV, class T>
constexpr int strip_minblocks() {
    return Ring<T, KV == 1>::on ? TFN_U16_MINBLOCKS
           : (F == FD && MODE == MEAN && KV != 1) ? TFN_STRIP_MINBLOCKS_FDMEAN
           : (TFN_FD_MEDIAN16 && F == FD && KV != 1) ? TFN_STRIP_MINBLOCKS_FDMEAN : TFN_STRIP_MINBLOCKS;
}

// KV (kernel variant): 0 fast path + exact per-pixel special path, 1 general (no special
// path: skips, flat, ties and invalid taps resolved in registers; ~45 % more instructions
// per pixel, but no divergent exact-path calls — the better choice when many row steps
// contain special pixels: holes, salt dropout, integer-quantized depth), 2 masked: the fast
// variant whose special test also requires every Q4 tap to be valid — a pixel next to a hole
// already comes out as the canonical NaN of the fast path, so holes and dropout no longer
// send row steps to the exact path (config 4: 191 vs 164 Gpx/s general, 94 fast), at the
// price of per-row tap-validity masks (clean config 2: 210 vs 217 fast).  The fast and
// masked variants count their special row steps into p.fired (host-side AUTO, tfn_abi.cu).
template <int F, int MODE, bool DISP, int LAYOUT, int KV, class T, bool PTS, int OUT>
#ifdef TFN_STRIP_MAXNREG
__global__ void __maxnreg__(TFN_STRIP_MAXNREG) tfn_strip_kernel(const __grid_constant__ CUtensorMap tm, KernelArgs p) {
#else
__global__ void __launch_bounds__(TFN_STRIP_THREADS, strip_minblocks<F, MODE, KV, T>())
    tfn_strip_kernel(const __grid_constant__ CUtensorMap tm, KernelArgs p) {
#endif
    const int lane = threadIdx.x & 31;
    const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int sx_n = (p.W + STRIP_COLS - 1) / STRIP_COLS;
    const int sy_n = (p.H + p.strip_h - 1) / p.strip_h;
    const int items = sx_n * sy_n * (int)p.B;          // < 2^31, checked by the host
    const long long HW = (long long)p.H * p.W;

    StripCtx<T> c;
    c.H = p.H; c.W = p.W;
    c.fx = p.fx; c.fy = p.fy;
    c.u0 = p.u0; c.v0 = p.v0;
    c.fired = p.fired;
    c.wt.kp = p.kp; c.wt.k0 = p.k0;
    c.outk = (OUT == 2) ? p.out_kind : (OUT == 3 ? 2 : OUT);
    c.lane = lane;
    if constexpr (Ring<T, KV == 1>::on) c.ring = ring_base();
    ring::Ring rg;
    constexpr bool TMA = TMA_ON<F, T, MODE, KV == 1, KV == 2>;
    if constexpr (TMA) {
        __shared__ __align__(128) float slots[TFN_STRIP_THREADS / 32][ring::NS * ring::SLOT_FLOATS];
        __shared__ __align__(8) unsigned long long bars[TFN_STRIP_THREADS / 32][ring::NS];
        ring::ring_init(rg, slots[threadIdx.x >> 5], bars[threadIdx.x >> 5], lane);
        c.rg = &rg;
        c.tm = &tm;
    }
    c.pscale = p.pscale; c.ifx = p.ifx; c.ify = p.ify;
    const int cb = c.outk == 0 ? 4 : 2;          // bytes per stored component
    const int nc = c.outk == 2 ? 2 : 3;          // stored components per pixel

    // first item static, the rest claimed from a work counter (load balance: strips with
    // holes or sky cost more or less than others); static striding without a counter
    for (int it = warp0; it < items;) {
        const int sx = it % sx_n;
        const int t2 = it / sx_n;
        const int sy = t2 % sy_n;
        const long long fb = t2 / sy_n;
        const int c0 = sx * STRIP_COLS + lane * PPL;
        const int y0 = sy * p.strip_h;
        const int y1 = min(y0 + p.strip_h, p.H);
        c.okm = c0 < p.W;
        c.okl = c.okm && c0 >= 1;
        c.okr = c0 + PPL < p.W;
        c.cm = min(c0, p.W - PPL);
        c.img = reinterpret_cast<const T*>(p.in) + fb * HW;
        c.pm = c.img + c.cm;
#pragma unroll
        for (int i = 0; i < PPL; ++i) c.a[i] = __fsub_rn(__int2float_rn(c0 + i), c.u0);   // a = u - u0
        unsigned colmask = 0;
        if (!c.okm) colmask = 0xFu;
        else {
            if (c0 == 0) colmask |= 1u;
            if (c0 + PPL - 1 == p.W - 1) colmask |= 1u << (PPL - 1);
        }
        char* out = reinterpret_cast<char*>(p.out) + cb * (fb * nc * HW + (LAYOUT == 0 ? (long long)c.cm : (long long)nc * c.cm));
        c.pts = p.pts ? p.pts + fb * 3 * HW + (LAYOUT == 0 ? (long long)c.cm : 3LL * c.cm) : nullptr;

        c.y1 = y1;
        if constexpr (TMA) {
            ring::ring_strip(&tm, rg, sx * STRIP_COLS - 4, y0, y1, (int)fb, lane);
            c.ys = y0;
        }
        strip_rows<F, MODE, DISP, LAYOUT, KV == 1, T, PTS, OUT, KV == 2>(c, out, HW, colmask, y0, y1);
        if constexpr (TMA) ring::ring_strip_done(rg);
        if (p.work) {
            int nxt = 0;
            if (lane == 0) nxt = atomicAdd(p.work, 1);
            it = nwarps + __shfl_sync(0xffffffffu, nxt, 0);
        } else {
            it += nwarps;
        }
    }
}

}  // namespace tfn
