// tfn_f32.cuh — the fp32 "unit-step" 3F2N strip kernel (round-2 production path).
//
// Same method as tfn_strip.cuh (Eq. 13-18, through the closed form of
// DESIGN.md §2.1), but with NO fp64: every gradient is assembled from UNIT-STEP inverse-depth
// differences computed with an exact depth difference,
//
//     D(o -> x) = w_x - w_o = -(Z_x - Z_o) * w_o * w_x      (w = 1/Z, Z_x - Z_o exact: Sterbenz)
//
// which carry a few ulps of RELATIVE error each (no cancellation inside a difference), and the
// four candidate multipliers m in {g_u, g_v, s = g_u + g_v, t = g_v - g_u} are summed from
// differences along their OWN direction:
//
//     g_u = kp H2(v-1) + k0 H2(v) + kp H2(v+1),          H2(r) = E(r,c-1) + E(r,c)
//     g_v = sum_c' k_c' (S(v-1,c') + S(v,c'))
//     s   = 2kp (SE(v,c) + SE(v-1,c-1)) + k0 (SE(v-1,c) + SE(v,c-1))
//     t   = 2kp (SW(v,c) + SW(v-1,c+1)) + k0 (SW(v,c+1) + SW(v-1,c))
//
// (E/S/SE/SW = unit differences toward (0,+1)/(+1,0)/(+1,+1)/(+1,-1)).  On a plane every term
// of s has the sign of s, so the isoline cancellation that forced fp64 in round 1
// (s = g_u + g_v of two large opposite numbers) is gone.  What is left — terms of mixed sign,
// i.e. a multiplier that is small against its own terms — is BOUNDED per pixel by a guard: with
// S_m = sum |k D| the abs-sum of m's terms, |m~ - m| <= c1 S_m, and the angular error of the
// pixel is at most
//
//     [ c1 (fx+|a|) S_u + c1 (fy+|b|) S_v + (c1 max_m S_m/|m| + 10u) V ] / |n'|        (*)
//
// (V = max(|x_(4)|, |x_(5)|) for the median, the mean candidate magnitude for the mean; the
// derivation is DESIGN.md §2.5).  A pixel whose bound exceeds the budget (0.4e-3 deg) — and
// every pixel with a skipped candidate, the flat rule, an orientation tie or an out-of-range
// sample — is "special": it is queued per warp in shared memory and recomputed by the exact
// fp64 per-pixel routine (pixel_general, tfn_device.cuh), 32 pixels at a time.
//
// Data movement: the input rows of a warp's 128-column strip (+4 columns each side, so the
// 16-B vectors stay aligned; out-of-image columns/rows are ZERO-filled = invalid, Q3) come
// through a per-warp ring of TMA boxes (cp.async.bulk.tensor, one mbarrier per slot); a lane
// reads its 4 samples with one LDS.128 and the two halo samples with LDS.32.  Normals go out
// with three streaming STG.128 per lane-row.  Persistent grid, strips claimed from a work
// counter.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tfn_device.cuh"
#include "tfn_kernels.h"
#include "tfn_tma.cuh"

#ifndef TFN_F32_MINBLOCKS
#define TFN_F32_MINBLOCKS 4
#endif

namespace tfn {
namespace f32 {

constexpr int PPL = 4;                       // pixels (columns) per lane
constexpr int NW = PPL + 2;                  // window width (1 halo column each side)
using ring::RC;
using ring::NS;
using ring::BOXW;
constexpr int WARPS = TFN_F32_THREADS / 32;
constexpr int QCAP = 32 + 32 * PPL;          // special-pixel queue entries per warp

struct __align__(128) Smem {
    float ring[WARPS][NS][RC][BOXW];         // 544-B rows: 16-B aligned lane vectors (tfn_tma.cuh)
    unsigned long long bar[WARPS][NS];
    int q[WARPS][QCAP];
};
using ring::Ring;

// ---- guard constants.  u = 2^-24; rcp.approx <= 2^-22 relative.
//      depth: D = -(dZ w_o) w_x: 3 roundings + 2 reciprocals = 11u; sums of <= 6 terms: +6u;
//      c1 = 20u (margin) + 2u (n_z rounding) = 22u.  Disparity: D = d_x - d_o (<= 1 rounding),
//      c1 = 12u.  The host folds c1 into Consts (c1fx, c1fy, c1) and computes teff.
constexpr float U24 = 5.9604644775390625e-08f;

// ---- filter weights [kp k0 kp] (Q1) in fp32 (exact for the named kernels) -------------------
template <int F> struct W32 { static constexpr float kp = 1.f, k0 = 1.f; };    // CUSTOM: run time
template <> struct W32<FD> { static constexpr float kp = 0.f, k0 = 1.f; };
template <> struct W32<SOBEL> { static constexpr float kp = 1.f, k0 = 2.f; };
template <> struct W32<SCHARR> { static constexpr float kp = 3.f, k0 = 10.f; };
template <> struct W32<PREWITT> { static constexpr float kp = 1.f, k0 = 1.f; };

// Consts (tfn_kernels.h F32Consts): CUSTOM weights and the guard constants

// ---- samples -------------------------------------------------------------------------------
// Fast-path valid iff 2^-24 <= z < 2^24 (inside Q5's valid set, and far enough from fp32's
// range that no product below under- or overflows).  Outside: a NaN whose SIGN BIT is set for
// +0 and negative samples (certainly invalid: holes, Q5) and clear otherwise (NaN, Inf,
// subnormal, or a valid sample outside the fast range: the exact path decides).
constexpr unsigned LO_BITS = 0x33800000u;            // 2^-24
constexpr unsigned SPAN = 0x4B800000u - LO_BITS;     // below 2^24
__device__ __forceinline__ float sanitize32(float z) {
    const unsigned b = __float_as_uint(z);
    const unsigned bad = 0x7fffffffu | ((b - 1u) & 0x80000000u);
    return (b - LO_BITS) < SPAN ? z : __uint_as_float(bad);
}
__device__ __forceinline__ bool maybe_valid(float zs) { return (int)__float_as_uint(zs) >= 0; }

// Pixel pairs.  A lane owns columns c0..c0+3 (pixels 0..3) and sees the window j = 0..5 =
// columns c0-1 .. c0+4.  Every per-pixel quantity is a float2 over the pixel pairs
// A = (0, 2) and B = (1, 3), and every window quantity a float2 over the column pairs
// (k, k+2), k = 0..3 — so the shifted operands of the stencil (left / right neighbour
// columns) are again aligned register pairs and all arithmetic issues as FFMA2 / FADD2 /
// FMUL2.  Pixel pair p (0 = A, 1 = B) has its centre columns at window pair k = p + 1, its
// left neighbours at k - 1 and its right neighbours at k + 1.
//
// Multipliers.  Each of the four is a 3-term sum of differences along its
// own direction, every difference computed directly with an exact depth difference:
//   g_u = kp (H(v-1) + H(v+1)) + k0 H(v),            H(r)  = w(r,c+1) - w(r,c-1)
//   g_v = kp (V(c-1) + V(c+1)) + k0 V(c),            V(c') = w(v+1,c') - w(v-1,c')
//   s   = 2kp DD1 + k0 (SE(v-1,c) + SE(v,c-1)),      DD1   = w(v+1,c+1) - w(v-1,c-1)
//   t   = 2kp DD2 + k0 (SW(v,c+1) + SW(v-1,c)),      DD2   = w(v+1,c-1) - w(v-1,c+1)
// (SE(r,c') = w(r+1,c'+1) - w(r,c'), SW(r,c') = w(r+1,c'-1) - w(r,c'); expanding shows
// s = g_u + g_v and t = g_v - g_u exactly.)  Each difference carries <= 11u relative error
// (u = 2^-24; rcp.approx <= 2^-22).  If the three terms of a multiplier have one sign — the
// GUARD, one LOP3 per multiplier — the multiplier is accurate to 13u relative, so every
// candidate to 20u, the median / mean to 20u V, and the angle to
//     13u (2 + |a|/fx + |b|/fy) + 30u V/|n'|
// which the kernel checks as V <= Kpix |n'|.  Pixels with a mixed-sign multiplier (a
// directional extremum inside the window, an occlusion edge, noise) are special.
//
// Sign convention.  The kernel carries the NEGATED differences D' = w_o - w_x (depth:
// (Z_x - Z_o) w_o w_x, no negation needed; disparity: d_o - d_x), hence negated multipliers
// m' = -m, candidates tau' = -tau and Phi' = -Phi.  n' is linear in (m, Phi), so n'' = -n',
// and the oriented output n' copysign(1/|n'|, Phi) is unchanged (the guard and the special
// tests are sign-free).
// ---- register pairs.  The packed fp32 ops take 64-bit register pairs; keeping every pair in a
// 64-bit value (inline PTX f32x2 on .b64 operands) stops the front end from splitting float2s
// into scalars and re-pairing them at each use (measured: 56-98 register moves per row step).
typedef unsigned long long P2;                       // .x = low word, .y = high word
__device__ __forceinline__ P2 pk(float x, float y) { P2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float lo(P2 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(P2 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }
__device__ __forceinline__ P2 add2(P2 a, P2 b) { P2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 sub2(P2 a, P2 b) { P2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 mul2(P2 a, P2 b) { P2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 fma2(P2 a, P2 b, P2 c) { P2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ P2 sc2(float a) { return pk(a, a); }
__device__ __forceinline__ P2 abs2(P2 a) { return a & 0x7fffffff7fffffffull; }
__device__ __forceinline__ P2 rcp2(P2 a) { return pk(rcp_approx(lo(a)), rcp_approx(hi(a))); }

struct Win {                   // one row's window pairs (k, k+2), k = 0..3
    P2 Z[4], W[4];             // sanitized samples; w = 1/z (depth) or d (disparity)
    P2 H[2];                   // H of this row per pixel pair
};
struct Link {                  // what row v's step hands to row v+1's step
    P2 RE[3];                  // R of the E pairs (k -> k+1) of row v+1
    P2 RN[2], RNW[2], RNE[2];  // R of the pairs (v,c)->(v+1,c), (v,c-1)->(v+1,c), (v,c+1)->(v+1,c)
    P2 SE[2], SW[2];           // SE(v,c) and SW(v,c) per pixel pair (row v+1's SE(v'-1,c), SW(v'-1,c))
    unsigned cm;               // non-masked: row v+1's centres that may be valid (bit i)
    unsigned hb, cb;           // masked: row v+1's sign bytes (3-column window ORs / centre column)
    unsigned hbp, cbp;         //   and row v's
};

// depth: dz = Z_x - Z_o, R = 1/dz, D' = dz w_o w_x;  disparity: dz = d_o - d_x, R = 1/dz, D' = dz
template <bool DISP> __device__ __forceinline__ P2 dz2(P2 zo, P2 zx) { return DISP ? sub2(zo, zx) : sub2(zx, zo); }
template <bool DISP> __device__ __forceinline__ P2 dd2(P2 dz, P2 wo, P2 wx) { return DISP ? dz : mul2(mul2(dz, wo), wx); }
template <bool DISP> __device__ __forceinline__ P2 diff(P2 zo, P2 zx, P2 wo, P2 wx) { return dd2<DISP>(dz2<DISP>(zo, zx), wo, wx); }

// kp (x + z) + k0 y  and  2kp x + k0 (y + z), the named kernels' constants folded (Q1)
template <int F, bool CUST> struct Wk {
    __device__ static __forceinline__ P2 sym(const F32Consts& k, P2 x, P2 y, P2 z) {
        if (F == FD) return y;
        if (F == SOBEL) return fma2(sc2(2.f), y, add2(x, z));
        if (F == PREWITT) return add2(add2(x, z), y);
        const float kp = CUST ? k.kp : W32<F>::kp, k0 = CUST ? k.k0 : W32<F>::k0;
        return fma2(sc2(k0), y, mul2(sc2(kp), add2(x, z)));
    }
    __device__ static __forceinline__ P2 diag(const F32Consts& k, P2 x, P2 y, P2 z) {
        if (F == FD) return add2(y, z);
        if (F == SOBEL) return mul2(sc2(2.f), add2(x, add2(y, z)));
        if (F == PREWITT) return fma2(sc2(2.f), x, add2(y, z));
        const float kp = CUST ? k.kp : W32<F>::kp, k0 = CUST ? k.k0 : W32<F>::k0;
        return fma2(sc2(2.f * kp), x, mul2(sc2(k0), add2(y, z)));
    }
};
// sign bit set iff the three terms do not share one sign (LOP3 on the 32-bit halves)
__device__ __forceinline__ unsigned mix3(float x, float y, float z) {
    const unsigned a = __float_as_uint(x), b = __float_as_uint(y), c = __float_as_uint(z);
    return (a ^ b) | (b ^ c);
}

// masked variant: sign bytes of (bits - 1) for the row's 3-column windows and centre columns
// (sign set iff the sample is +0 or negative: certainly invalid)
__device__ __forceinline__ void row_masks(const float zr[NW], unsigned& hb, unsigned& cb) {
    int m1[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) m1[j] = (int)(__float_as_uint(zr[j]) - 1u);
    int h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = m1[i] | m1[i + 1] | m1[i + 2];
    hb = __byte_perm(__byte_perm(h[0], h[1], 0x0073), __byte_perm(h[2], h[3], 0x0073), 0x5410);
    cb = __byte_perm(__byte_perm(m1[1], m1[2], 0x0073), __byte_perm(m1[3], m1[4], 0x0073), 0x5410);
}
// non-masked variant: centres that may be valid (not +0 / negative)
__device__ __forceinline__ unsigned centre_mask(const float zr[NW]) {
    unsigned m = 0;
#pragma unroll
    for (int i = 0; i < PPL; ++i) m |= ((int)__float_as_uint(zr[i + 1]) > 0 ? 1u : 0u) << i;
    return m;
}

struct Ctx {
    float fx, fy;
    P2 a2[2];                  // a = u - u0 per pixel pair
    P2 kc[2];                  // the guard's V/|n'| limit per pixel pair before the row term
    unsigned colmask;          // pixels (bit i) on the image's first / last column or past W (never special)
    F32Consts k;
};

// candidates, Phi, n' and the guard tests of one pixel pair.  Returns the pair's failing bits
// (bit 0: .x pixel, bit 1: .y pixel); px, py, nz = n' and sc = the signed 1/|n'| (the caller
// scales into the store vectors).
template <int MODE, bool DISP>
__device__ __forceinline__ unsigned finish_pair(const Ctx& c, P2 mu, P2 mv, P2 ms, P2 mt, P2 zc, const P2 R[8], P2 a,
                                                P2 b2, P2 klim, P2& px, P2& py, P2& nz, P2& sc) {
    const P2 xu = mul2(mu, zc), xv = mul2(mv, zc), xs = mul2(ms, zc), xt = mul2(mt, zc);
    P2 sum8;
    float ph0, ph1, V0, V1;
    if (MODE == MEAN) {
        // numerator by neighbour-direction pairs (as tfn_device.cuh finish32): sum_dir x (R_a + R_b)
        sum8 = add2(fma2(xu, add2(R[0], R[1]), mul2(xv, add2(R[2], R[3]))),
                    fma2(xs, add2(R[4], R[5]), mul2(xt, add2(R[6], R[7]))));
        const P2 phi = mul2(sum8, sc2(0.125f));
        ph0 = lo(phi); ph1 = hi(phi);
        // V >= mean |tau|: (1/8) sum_dir (|x| (|R_a| + |R_b|) + 2|m|)   (disparity: no |m| term)
        P2 acc = fma2(abs2(xu), add2(abs2(R[0]), abs2(R[1])), mul2(abs2(xv), add2(abs2(R[2]), abs2(R[3]))));
        acc = fma2(abs2(xs), add2(abs2(R[4]), abs2(R[5])), fma2(abs2(xt), add2(abs2(R[6]), abs2(R[7])), acc));
        if (!DISP) acc = fma2(add2(add2(abs2(mu), abs2(mv)), add2(abs2(ms), abs2(mt))), sc2(2.f), acc);
        const P2 V = mul2(acc, sc2(0.125f));
        V0 = lo(V); V1 = hi(V);
    } else {
        P2 tau[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const P2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
            const P2 m = (k < 2) ? mu : (k < 4) ? mv : (k < 6) ? ms : mt;
            tau[k] = DISP ? mul2(x, R[k]) : (k & 1) ? sub2(mul2(x, R[k]), m) : fma2(x, R[k], m);
        }
        sum8 = add2(add2(add2(tau[0], tau[1]), add2(tau[2], tau[3])), add2(add2(tau[4], tau[5]), add2(tau[6], tau[7])));
        float t0[8], t1[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { t0[k] = lo(tau[k]); t1[k] = hi(tau[k]); }
        float a0, b0, a1, b1;
        mid_pair8(t0, a0, b0);
        mid_pair8(t1, a1, b1);
        ph0 = __fmul_rn(__fadd_rn(a0, b0), 0.5f);
        ph1 = __fmul_rn(__fadd_rn(a1, b1), 0.5f);
        V0 = fmaxf(fabsf(a0), fabsf(b0));
        V1 = fmaxf(fabsf(a1), fabsf(b1));
    }
    // a non-finite candidate makes Phi NaN (FMNMX drops NaN and keeps +-inf): special
    const P2 phi = fma2(sc2(0.f), sum8, pk(ph0, ph1));
    // n' = (fx g_u, fy g_v, -(a g_u + b g_v + Phi))  (all negated, see the sign convention)
    const P2 nzneg = fma2(a, mu, fma2(b2, mv, phi));
    px = mul2(sc2(c.fx), mu);
    py = mul2(sc2(c.fy), mv);
    nz = sub2(0ull, nzneg);
    const P2 dot = fma2(px, px, fma2(py, py, mul2(nzneg, nzneg)));
    const float r0 = rsqrt_approx(lo(dot)), r1 = rsqrt_approx(hi(dot));
    const float p0 = lo(phi), p1 = hi(phi);
    // flip iff Phi < 0 (Q11; Phi == 0 is special): scale = copysign(rsqrt(dot), Phi)
    sc = pk(__uint_as_float(__float_as_uint(r0) | (__float_as_uint(p0) & 0x80000000u)),
            __uint_as_float(__float_as_uint(r1) | (__float_as_uint(p1) & 0x80000000u)));
    // guard: V <= klim |n'| bounds the angle; |Phi| >= cg |n'| + tb V makes the
    // orientation certain (and rejects Phi == 0 / NaN).  |n'| = dot rsqrt(dot) is NaN when dot
    // is 0 or inf: every compare below then fails.
    const P2 nn = mul2(dot, pk(r0, r1));
    const P2 Vp = pk(V0, V1);
    const P2 q = sub2(mul2(nn, klim), Vp);
    const P2 thr = fma2(nn, sc2(c.k.cg), mul2(sc2(c.k.tb), Vp));
    const bool ok0 = (lo(q) >= 0.f) && (fabsf(p0) >= lo(thr)) && (fabsf(p0) > 0.f);
    const bool ok1 = (hi(q) >= 0.f) && (fabsf(p1) >= hi(thr)) && (fabsf(p1) > 0.f);
    return (ok0 ? 0u : 1u) | (ok1 ? 0u : 2u);
}

// the new row's window pairs: sanitize (Q5 + the fast range; invalid -> NaN), 1/z
template <bool DISP>
__device__ __forceinline__ void new_row(const float zr[NW], Win& r) {
    float z[NW], w[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        const unsigned bb = __float_as_uint(zr[j]);
        z[j] = (bb - LO_BITS) < SPAN ? zr[j] : __uint_as_float(0x7fffffffu);
        w[j] = DISP ? z[j] : rcp_approx(z[j]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) { r.Z[k] = pk(z[k], z[k + 2]); r.W[k] = pk(w[k], w[k + 2]); }
}

// one output row v: windows rm (v-1), rc (v), rn (v+1, filled here from zr), the link from
// row v-1's step (li) and to row v+1's step (lo).  Normals of row v -> ox/oy/oz (pixel 0..3);
// returns the lane's special bits (pixel i).
template <int F, int MODE, bool DISP, bool VM, bool CUST>
__device__ __forceinline__ unsigned row_step(const Ctx& c, const Win& rm, const Win& rc, Win& rn, const Link& li,
                                             Link& lo_, const float zr[NW], float b, float krb,
                                             float ox[PPL], float oy[PPL], float oz[PPL]) {
    using K = Wk<F, CUST>;
    constexpr bool CORN = (F != FD);             // zero-weight taps are never read (Q4)
    new_row<DISP>(zr, rn);
    if (VM) { row_masks(zr, lo_.hb, lo_.cb); lo_.hbp = li.hb; lo_.cbp = li.cb; } else lo_.cm = centre_mask(zr);
    // ---- unit pairs owned by row v: S (R only), SE, SW ----
    P2 RS[2], SEu[3], RSE[3], SWu[4], RSW[4];
#pragma unroll
    for (int k = 1; k < 3; ++k) RS[k - 1] = rcp2(dz2<DISP>(rc.Z[k], rn.Z[k]));
#pragma unroll
    for (int k = 0; k < 3; ++k) {                // SE: (v, col k) -> (v+1, col k+1)
        const P2 dz = dz2<DISP>(rc.Z[k], rn.Z[k + 1]);
        SEu[k] = dd2<DISP>(dz, rc.W[k], rn.W[k + 1]);
        RSE[k] = rcp2(dz);
    }
#pragma unroll
    for (int k = 1; k < 4; ++k) {                // SW: (v, col k) -> (v+1, col k-1)
        const P2 dz = dz2<DISP>(rc.Z[k], rn.Z[k - 1]);
        SWu[k] = dd2<DISP>(dz, rc.W[k], rn.W[k - 1]);
        RSW[k] = rcp2(dz);
    }
    // vertical 2-step differences V(c') for the window columns (only the centre ones for FD)
    P2 V2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (CORN || k == 1 || k == 2) V2[k] = diff<DISP>(rm.Z[k], rn.Z[k], rm.W[k], rn.W[k]);
    const P2 b2 = sc2(b);
    const P2 krb2 = sc2(krb);
    unsigned sp = 0;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int k = p + 1;
        // H of row v+1 (direct 2-step horizontal difference)
        rn.H[p] = diff<DISP>(rn.Z[k - 1], rn.Z[k + 1], rn.W[k - 1], rn.W[k + 1]);
        const P2 gu = CORN ? K::sym(c.k, rm.H[p], rc.H[p], rn.H[p]) : rc.H[p];
        const P2 gv = CORN ? K::sym(c.k, V2[k - 1], V2[k], V2[k + 1]) : V2[k];
        P2 dd1 = 0, dd2 = 0;
        if (CORN) {
            dd1 = diff<DISP>(rm.Z[k - 1], rn.Z[k + 1], rm.W[k - 1], rn.W[k + 1]);   // (v-1,c-1) -> (v+1,c+1)
            dd2 = diff<DISP>(rm.Z[k + 1], rn.Z[k - 1], rm.W[k + 1], rn.W[k - 1]);   // (v-1,c+1) -> (v+1,c-1)
        }
        // s: 2kp DD1 + k0 (SE(v-1,c) + SE(v,c-1));  t: 2kp DD2 + k0 (SW(v,c+1) + SW(v-1,c))
        const P2 gs = K::diag(c.k, dd1, li.SE[p], SEu[k - 1]);
        const P2 gt = K::diag(c.k, dd2, SWu[k + 1], li.SW[p]);
        lo_.SE[p] = SEu[k]; lo_.SW[p] = SWu[k];
        // guard: every multiplier's terms share one sign (FD: two terms of s and t only)
        unsigned mx0, mx1;
        if (CORN) {
            mx0 = mix3(lo(rm.H[p]), lo(rc.H[p]), lo(rn.H[p])) | mix3(lo(V2[k - 1]), lo(V2[k]), lo(V2[k + 1])) |
                  mix3(lo(dd1), lo(li.SE[p]), lo(SEu[k - 1])) | mix3(lo(dd2), lo(SWu[k + 1]), lo(li.SW[p]));
            mx1 = mix3(hi(rm.H[p]), hi(rc.H[p]), hi(rn.H[p])) | mix3(hi(V2[k - 1]), hi(V2[k]), hi(V2[k + 1])) |
                  mix3(hi(dd1), hi(li.SE[p]), hi(SEu[k - 1])) | mix3(hi(dd2), hi(SWu[k + 1]), hi(li.SW[p]));
        } else {
            mx0 = (__float_as_uint(lo(li.SE[p])) ^ __float_as_uint(lo(SEu[k - 1]))) |
                  (__float_as_uint(lo(SWu[k + 1])) ^ __float_as_uint(lo(li.SW[p])));
            mx1 = (__float_as_uint(hi(li.SE[p])) ^ __float_as_uint(hi(SEu[k - 1]))) |
                  (__float_as_uint(hi(SWu[k + 1])) ^ __float_as_uint(hi(li.SW[p])));
        }
        // ---- candidates (order E W S N SE NW SW NE) ----
        P2 R[8];
        R[0] = li.RE[k]; R[1] = li.RE[k - 1]; R[2] = RS[p]; R[3] = li.RN[p];
        R[4] = RSE[k]; R[5] = li.RNW[p]; R[6] = RSW[k]; R[7] = li.RNE[p];
        lo_.RN[p] = RS[p]; lo_.RNW[p] = RSE[k - 1]; lo_.RNE[p] = RSW[k + 1];
        P2 px, py, nz, sc;
        const P2 klim = sub2(c.kc[p], krb2);
        unsigned f2b = finish_pair<MODE, DISP>(c, gu, gv, gs, gt, rc.Z[k], R, c.a2[p], b2, klim, px, py, nz, sc);
        f2b |= ((int)mx0 < 0 ? 1u : 0u) | ((int)mx1 < 0 ? 2u : 0u);
        // pixel pair p = (pixel p, pixel p + 2): scalar products straight into the store vectors
        const float s0 = lo(sc), s1 = hi(sc);
        ox[p] = __fmul_rn(lo(px), s0); ox[p + 2] = __fmul_rn(hi(px), s1);
        oy[p] = __fmul_rn(lo(py), s0); oy[p + 2] = __fmul_rn(hi(py), s1);
        oz[p] = __fmul_rn(lo(nz), s0); oz[p + 2] = __fmul_rn(hi(nz), s1);
        sp |= ((f2b & 1u) << p) | ((f2b >> 1) << (p + 2));
    }
    // ---- E pairs of row v+1 (its E / W candidates) ----
#pragma unroll
    for (int k = 0; k < 3; ++k) lo_.RE[k] = rcp2(dz2<DISP>(rn.Z[k], rn.Z[k + 1]));
    // ---- which failing pixels go to the exact path ----
    if (VM) {
        // all Q4 taps (FD: the plus) free of certainly-invalid samples: a pixel with a hole /
        // out-of-image tap is already the canonical NaN (its candidates are NaN)
        const unsigned bad = CORN ? (li.hbp | li.hb | lo_.hb) : (li.hb | li.cbp | lo_.cb);
        const unsigned tapok = ~bad;             // bit 8i+7: pixel i's taps free of sign-NaNs
        unsigned m = 0;
#pragma unroll
        for (int i = 0; i < PPL; ++i) m |= ((tapok >> (8 * i + 7)) & 1u) << i;
        sp &= m;
    } else {
        sp &= li.cm & ~c.colmask;
    }
    return sp;
}

// first row of a strip (row y0 - 1): its window, H, E-pair reciprocals and masks; the rest of
// the link is only read by the priming step, whose outputs are discarded
template <int F, bool DISP, bool VM>
__device__ __forceinline__ void strip_init(Win& r, Link& l, const float zr[NW]) {
    new_row<DISP>(zr, r);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int k = p + 1;
        r.H[p] = diff<DISP>(r.Z[k - 1], r.Z[k + 1], r.W[k - 1], r.W[k + 1]);
        l.RN[p] = l.RNW[p] = l.RNE[p] = l.SE[p] = l.SW[p] = 0ull;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) l.RE[k] = rcp2(dz2<DISP>(r.Z[k], r.Z[k + 1]));
    if (VM) { row_masks(zr, l.hb, l.cb); l.hbp = l.hb; l.cbp = l.cb; } else l.cm = centre_mask(zr);
}

// normals are written once and never re-read: streaming stores
__device__ __forceinline__ void st4cs(float* p, float a, float b, float c, float d) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}
template <int LAYOUT>
__device__ __forceinline__ void store_row(float* o, long long HW, const float x[PPL], const float y[PPL],
                                          const float z[PPL]) {
    if (LAYOUT == 0) {
        st4cs(o, x[0], x[1], x[2], x[3]);
        st4cs(o + HW, y[0], y[1], y[2], y[3]);
        st4cs(o + 2 * HW, z[0], z[1], z[2], z[3]);
    } else {
        st4cs(o, x[0], y[0], z[0], x[1]);
        st4cs(o + 4, y[1], z[1], x[2], y[2]);
        st4cs(o + 8, z[2], x[3], y[3], z[3]);
    }
}

// ---- special-pixel queue: append this row step's special pixels (warp-collective) -------------
static __device__ __noinline__ void queue_append(int* q, int& qn, unsigned sp, int v, int c0, int lane, int* fired) {
    const int cnt = __popc(sp);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int pos = qn + incl - cnt;
    TFN_CHECK(qn + total <= QCAP && v >= 0 && v < 65536 && c0 >= 0 && c0 + PPL <= 65536);
#pragma unroll
    for (int i = 0; i < PPL; ++i)
        if (sp & (1u << i)) q[pos++] = (v << 16) | (c0 + i);
    qn += total;
    if (fired && lane == 0) atomicAdd(fired, total);
}

// recompute queued pixels exactly (pixel_general: fp64 gradients, skips, flat rule, ties,
// Q4), 32 at a time; all = false leaves fewer than 32 queued
template <int F, int MODE, bool DISP, int LAYOUT>
__device__ __noinline__ void queue_flush(const int* q, int& qn, bool all, const float* img, float* ofr, int H, int W,
                                         float u0, float v0, float fx, float fy, double kp, double k0, int lane) {
    __syncwarp();
    const long long HW = (long long)H * W;
    while (qn >= 32 || (all && qn > 0)) {
        const int nb = qn < 32 ? qn : 32;
        if (lane < nb) {
            const int e = q[qn - nb + lane];
            const int v = e >> 16, u = e & 0xffff;
            TFN_CHECK(qn - nb + lane >= 0 && v < H && u < W);
            const Normal n = pixel_general<F, MODE, DISP>(img, H, W, v, u, u0, v0, fx, fy, Wts{kp, k0});
            const long long pix = (long long)v * W + u;
            if (LAYOUT == 0) {
                ofr[pix] = n.x; ofr[HW + pix] = n.y; ofr[2 * HW + pix] = n.z;
            } else {
                ofr[3 * pix] = n.x; ofr[3 * pix + 1] = n.y; ofr[3 * pix + 2] = n.z;
            }
        }
        qn -= nb;
        __syncwarp();
    }
}

// ---- the kernel --------------------------------------------------------------------------------
// KernelArgs as the strip kernel (tfn_kernels.h); the input is also described by the tensor map
// tm: dims (W, H, B) fp32, box (136, RC, 1), zero OOB fill.
template <int F, int MODE, bool DISP, bool VM, int LAYOUT>
__global__ void __launch_bounds__(TFN_F32_THREADS, TFN_F32_MINBLOCKS)
tfn_f32_kernel(const __grid_constant__ CUtensorMap tm, const KernelArgs p, const Consts kc) {
    __shared__ Smem sm;
    constexpr bool CUST = (F == CUSTOM);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Ring rg;
    ring::ring_init(rg, &sm.ring[wid][0][0][0], &sm.bar[wid][0], lane);
    int* q = sm.q[wid];
    int qn = 0;

    const int warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int sx_n = (p.W + 127) / 128;
    const int sy_n = (p.H + p.strip_h - 1) / p.strip_h;
    const int items = sx_n * sy_n * (int)p.B;
    const long long HW = (long long)p.H * p.W;

    Ctx c;
    c.fx = p.fx; c.fy = p.fy;
    c.k = kc;

    for (int it = warp0; it < items;) {
        const int sx = it % sx_n;
        const int t2 = it / sx_n;
        const int sy = t2 % sy_n;
        const int fb = t2 / sy_n;
        const int c0 = sx * 128 + lane * PPL;
        const int y0 = sy * p.strip_h;
        const int y1 = min(y0 + p.strip_h, p.H);
        const bool okm = c0 < p.W;
        c.colmask = okm ? ((c0 == 0 ? 1u : 0u) | (c0 + PPL == p.W ? (1u << (PPL - 1)) : 0u)) : 0xfu;
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {      // pixel pair q2 = (pixel q2, pixel q2 + 2)
            const float a0 = __fsub_rn(__int2float_rn(c0 + q2), p.u0);
            const float a1 = __fsub_rn(__int2float_rn(c0 + q2 + 2), p.u0);
            c.a2[q2] = pk(a0, a1);
            c.kc[q2] = pk(__fmaf_rn(-kc.kca, fabsf(a0), kc.k0lim), __fmaf_rn(-kc.kca, fabsf(a1), kc.k0lim));
        }
        const float* img = reinterpret_cast<const float*>(p.in) + (long long)fb * HW;
        float* ofr = reinterpret_cast<float*>(p.out) + (long long)fb * 3 * HW;
        float* orow = ofr + (LAYOUT == 0 ? (long long)c0 : 3LL * c0);

        // this strip's rows y0-1 .. y1 through the TMA ring
        ring::ring_strip(&tm, rg, sx * 128 - 4, y0, y1, fb, lane);

        Win win[3];
        Link lk[3];
        float zr[NW];
        ring::ring_row(&tm, rg, 0, lane, zr);
        strip_init<F, DISP, VM>(win[0], lk[0], zr);
        win[2] = win[0];
        float ox[PPL], oy[PPL], oz[PPL];
        // step s outputs row v = y0 - 1 + s (s = 0 only primes the state): windows and links rotate
        // over 3 slots (only two links are ever live) — the body is unrolled 3 times so every slot
        // index is static and the loop stays inside the 32 KB L1.5 instruction cache
#define TFN_F32_STEP(S)                                                                                        \
        {                                                                                                      \
            const int v = y0 - 1 + s;                                                                          \
            ring::ring_row(&tm, rg, s + 1, lane, zr);                                                              \
            const float bf = __fsub_rn(__int2float_rn(v), p.v0);                                               \
            unsigned sp = row_step<F, MODE, DISP, VM, CUST>(c, win[((S) + 2) % 3], win[(S) % 3], win[((S) + 1) % 3], \
                                                            lk[(S) % 3], lk[((S) + 1) % 3], zr, bf,           \
                                                            kc.kr * fabsf(bf), ox, oy, oz);                         \
            if (v >= y0) {                                                                                     \
                TFN_CHECK(v < p.H && (!okm || c0 + PPL <= p.W));                                               \
                if (okm) store_row<LAYOUT>(orow + (long long)v * p.W * (LAYOUT == 0 ? 1 : 3), HW, ox, oy, oz); \
                if (!VM && (v == 0 || v == p.H - 1)) sp = 0;                                                   \
                if (__any_sync(0xffffffffu, sp != 0)) {                                                        \
                    queue_append(q, qn, sp, v, c0, lane, p.fired);                                             \
                    if (qn >= 32)                                                                              \
                        queue_flush<F, MODE, DISP, LAYOUT>(q, qn, false, img, ofr, p.H, p.W, p.u0, p.v0, p.fx, \
                                                           p.fy, p.kp, p.k0, lane);                            \
                }                                                                                              \
            }                                                                                                  \
            if (v + 1 >= y1) break;                                                                            \
            ++s;                                                                                               \
        }
        for (int s = 0;;) {
            TFN_F32_STEP(0) TFN_F32_STEP(1) TFN_F32_STEP(2)
        }
#undef TFN_F32_STEP
        ring::ring_strip_done(rg);
        if (qn > 0)
            queue_flush<F, MODE, DISP, LAYOUT>(q, qn, true, img, ofr, p.H, p.W, p.u0, p.v0, p.fx, p.fy, p.kp, p.k0, lane);
        if (p.work) {
            int nxt = 0;
            if (lane == 0) nxt = atomicAdd(p.work, 1);
            it = nwarps + __shfl_sync(0xffffffffu, nxt, 0);
        } else {
            it += nwarps;
        }
    }
}

}  // namespace f32
}  // namespace tfn
