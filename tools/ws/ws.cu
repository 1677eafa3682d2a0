// Prototype (A/B only): warp-specialised 3F2N fast variant.  Producer warps run the strip
// kernel's register window (loads, sanitize, fp64 1/z, gradients, fp32 m values, pair
// reciprocals) and hand each lane-row to a consumer warp through a shared-memory ring
// (13 float4 per lane: g_u, g_v, s, t, z_c and the 8 neighbour reciprocal groups);
// consumers run candidates, the median network, the tail, the special path and the stores.
// Same device arithmetic as tfn_strip_kernel<..., fast> -> bit-identical output.
#include "../../paper_2005_08165_b200/csrc/tfn_device.cuh"
#include "../../paper_2005_08165_b200/csrc/tfn_kernels.h"
#include "../../paper_2005_08165_b200/csrc/tfn_strip.cuh"

#ifndef WS_NS
#define WS_NS 3                 // ring slots per producer/consumer pair
#endif
#ifndef WS_PAIRS
#define WS_PAIRS 4              // producer/consumer warp pairs per CTA
#endif
#ifndef WS_MINB
#define WS_MINB 2
#endif

namespace tfn {

constexpr int WS_G = 13;                                // float4 groups per lane-row
struct WsShared {
    float4 slot[WS_PAIRS][WS_NS][WS_G][32];
    int meta[WS_PAIRS][WS_NS][2];                       // item, row
    unsigned long long full[WS_PAIRS][WS_NS], empty[WS_PAIRS][WS_NS];
};

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(void* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(void* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(void* b, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}" :: "r"(sa(b)), "r"(parity) : "memory");
}

struct Item { int c0, y0, y1; long long fb; };
__device__ __forceinline__ Item item_geom(int it, const KernelArgs& p) {
    const int sx_n = (p.W + STRIP_COLS - 1) / STRIP_COLS;
    const int sy_n = (p.H + p.strip_h - 1) / p.strip_h;
    Item r;
    const int sx = it % sx_n, t2 = it / sx_n;
    r.c0 = sx * STRIP_COLS + (threadIdx.x & 31) * PPL;
    r.y0 = (t2 % sy_n) * p.strip_h;
    r.y1 = min(r.y0 + p.strip_h, p.H);
    r.fb = t2 / sy_n;
    return r;
}
__device__ __forceinline__ void lane_ctx(StripCtx<float>& c, const KernelArgs& p, const Item& g, unsigned& colmask) {
    c.okm = g.c0 < p.W;
    c.okl = c.okm && g.c0 >= 1;
    c.okr = g.c0 + PPL < p.W;
    c.cm = min(g.c0, p.W - PPL);
    c.img = reinterpret_cast<const float*>(p.in) + g.fb * (long long)p.H * p.W;
    c.pm = c.img + c.cm;
#pragma unroll
    for (int i = 0; i < PPL; ++i) c.a[i] = __fsub_rn(__int2float_rn(g.c0 + i), c.u0);
    colmask = 0;
    if (!c.okm) colmask = 0xFu;
    else {
        if (g.c0 == 0) colmask |= 1u;
        if (g.c0 + PPL - 1 == p.W - 1) colmask |= 1u << (PPL - 1);
    }
}

// producer: one row step up to the pair reciprocals, written to ring slot s
template <int F, bool DISP>
__device__ __forceinline__ void prod_row(Slot& P, Slot& C, Slot& N, int v, const StripCtx<float>& c,
                                         float4 (*slot)[32], int lane) {
    load_raw(C, c, v + 3);
    prepare<DISP, false>(N, c);
    double gu[4], gv[4], dv[6];
#pragma unroll
    for (int j = 0; j < PPL + 2; ++j)
        dv[j] = (Taps<F>::corners || (j >= 1 && j <= PPL)) ? __dsub_rn(N.w[j], P.w[j]) : 0.0;
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        const double dhn = __dsub_rn(N.w[i + 2], N.w[i]);
        const double dhc = Taps<F>::corners ? __dsub_rn(C.w[i + 2], C.w[i]) : 0.0;
        gu[i] = grad_tail<F>(C.head[i], dhn, c.wt);
        N.head[i] = grad_head<F>(dhc, dhn, c.wt);
        gv[i] = grad_tail<F>(grad_head<F>(dv[i], dv[i + 1], c.wt), dv[i + 2], c.wt);
    }
    float gu32[4], gv32[4], s32[4], t32[4];
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        gu32[i] = __double2float_rn(gu[i]);
        gv32[i] = __double2float_rn(gv[i]);
        s32[i] = __double2float_rn(__dadd_rn(gu[i], gv[i]));
        t32[i] = __double2float_rn(__dsub_rn(gv[i], gu[i]));
    }
    float rE[5], rS[4], rSE[5], rSW[5];        // index 0 = the left halo pair (i - 1 of pixel 0)
    rE[0] = pair_rcp<DISP>(C.z[0], C.z[1]);
    rSE[0] = pair_rcp<DISP>(C.z[0], N.z[1]);
    rSW[0] = pair_rcp<DISP>(C.z[1], N.z[0]);
#pragma unroll
    for (int i = 0; i < PPL; ++i) {
        const float zc = C.z[i + 1];
        rE[i + 1] = pair_rcp<DISP>(zc, C.z[i + 2]);
        rS[i] = pair_rcp<DISP>(zc, N.z[i + 1]);
        rSE[i + 1] = pair_rcp<DISP>(zc, N.z[i + 2]);
        rSW[i + 1] = pair_rcp<DISP>(C.z[i + 2], N.z[i + 1]);
    }
    slot[0][lane] = make_float4(gu32[0], gu32[1], gu32[2], gu32[3]);
    slot[1][lane] = make_float4(gv32[0], gv32[1], gv32[2], gv32[3]);
    slot[2][lane] = make_float4(s32[0], s32[1], s32[2], s32[3]);
    slot[3][lane] = make_float4(t32[0], t32[1], t32[2], t32[3]);
    slot[4][lane] = make_float4(C.z[1], C.z[2], C.z[3], C.z[4]);
    // R groups, order E W S N SE NW SW NE
    slot[5][lane] = make_float4(rE[1], rE[2], rE[3], rE[4]);
    slot[6][lane] = make_float4(rE[0], rE[1], rE[2], rE[3]);
    slot[7][lane] = make_float4(rS[0], rS[1], rS[2], rS[3]);
    slot[8][lane] = make_float4(C.rN[0], C.rN[1], C.rN[2], C.rN[3]);
    slot[9][lane] = make_float4(rSE[1], rSE[2], rSE[3], rSE[4]);
    slot[10][lane] = make_float4(C.rNW[0], C.rNW[1], C.rNW[2], C.rNW[3]);
    slot[11][lane] = make_float4(rSW[0], rSW[1], rSW[2], rSW[3]);
    slot[12][lane] = make_float4(C.rNE[0], C.rNE[1], C.rNE[2], C.rNE[3]);
#pragma unroll
    for (int i = 0; i < PPL; ++i) { N.rN[i] = rS[i]; N.rNW[i] = rSE[i]; N.rNE[i] = rSW[i + 1]; }
}

template <int F, int MODE, bool DISP>
__global__ void __launch_bounds__(64 * WS_PAIRS, WS_MINB) tfn_ws_kernel(KernelArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WsShared& sh = *reinterpret_cast<WsShared*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp < WS_PAIRS;
    const int pr = producer ? warp : warp - WS_PAIRS;
    if (threadIdx.x == 0) {
        for (int a = 0; a < WS_PAIRS; ++a)
            for (int s = 0; s < WS_NS; ++s) { mb_init(&sh.full[a][s], 32); mb_init(&sh.empty[a][s], 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int sx_n = (p.W + STRIP_COLS - 1) / STRIP_COLS;
    const int sy_n = (p.H + p.strip_h - 1) / p.strip_h;
    const int items = sx_n * sy_n * (int)p.B;
    const long long HW = (long long)p.H * p.W;
    const int npairs = gridDim.x * WS_PAIRS;
    StripCtx<float> c;
    c.H = p.H; c.W = p.W; c.fx = p.fx; c.fy = p.fy; c.u0 = p.u0; c.v0 = p.v0;
    c.fired = nullptr; c.wt.kp = p.kp; c.wt.k0 = p.k0; c.outk = 0; c.pts = nullptr;
    c.lane = lane;
    unsigned colmask = 0;
    if (producer) {
        int ri = 0;                                  // ring index
        auto put = [&](int it, int v) -> float4 (*)[32] {
            const int s = ri % WS_NS;
            if (ri >= WS_NS) mb_wait(&sh.empty[pr][s], ((ri / WS_NS) - 1) & 1);
            if (lane == 0) { sh.meta[pr][s][0] = it; sh.meta[pr][s][1] = v; }
            return sh.slot[pr][s];
        };
        auto done = [&]() { mb_arrive(&sh.full[pr][ri % WS_NS]); ++ri; };
        for (int it = blockIdx.x * WS_PAIRS + pr; it < items;) {
            const Item g = item_geom(it, p);
            lane_ctx(c, p, g, colmask);
            Slot S0, S1, S2;
            const int ys = g.y0, y1 = g.y1;
            load_raw(S0, c, ys - 1);
            load_raw(S1, c, ys);
            load_raw(S2, c, ys + 1);
            prepare<DISP, false>(S0, c);
            prepare<DISP, false>(S1, c);
            load_raw(S0, c, ys + 2);
#pragma unroll
            for (int i = 0; i < PPL; ++i) {
                S1.head[i] = grad_head<F>(Taps<F>::corners ? __dsub_rn(S0.w[i + 2], S0.w[i]) : 0.0,
                                          __dsub_rn(S1.w[i + 2], S1.w[i]), c.wt);
                const float zc = S1.z[i + 1];
                S1.rN[i] = pair_rcp<DISP>(S0.z[i + 1], zc);
                S1.rNW[i] = pair_rcp<DISP>(S0.z[i], zc);
                S1.rNE[i] = pair_rcp<DISP>(S0.z[i + 2], zc);
            }
            for (int v = ys; v < y1; v += 3) {
                prod_row<F, DISP>(S0, S1, S2, v, c, put(it, v), lane); done();
                if (v + 1 >= y1) break;
                prod_row<F, DISP>(S1, S2, S0, v + 1, c, put(it, v + 1), lane); done();
                if (v + 2 >= y1) break;
                prod_row<F, DISP>(S2, S0, S1, v + 2, c, put(it, v + 2), lane); done();
            }
            if (p.work) {
                int nxt = 0;
                if (lane == 0) nxt = atomicAdd(p.work, 1);
                it = npairs + __shfl_sync(0xffffffffu, nxt, 0);
            } else {
                it += npairs;
            }
        }
        put(-1, 0); done();
        return;
    }
    // ---- consumer ----
    int cur = -1;
    Item g;
    char* out = nullptr;
    for (int ri = 0;; ++ri) {
        const int s = ri % WS_NS;
        mb_wait(&sh.full[pr][s], (ri / WS_NS) & 1);
        const int it = sh.meta[pr][s][0], v = sh.meta[pr][s][1];
        if (it < 0) break;
        if (it != cur) {
            cur = it;
            g = item_geom(it, p);
            lane_ctx(c, p, g, colmask);
            out = reinterpret_cast<char*>(p.out) + 4 * (g.fb * 3 * HW + (long long)c.cm);
        }
        const float4 (*sl)[32] = sh.slot[pr][s];
        const float4 G0 = sl[0][lane], G1 = sl[1][lane], G2 = sl[2][lane], G3 = sl[3][lane], Z = sl[4][lane];
        float4 RR[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) RR[k] = sl[5 + k][lane];
        mb_arrive(&sh.empty[pr][s]);
        const float gu32[4] = {G0.x, G0.y, G0.z, G0.w}, gv32[4] = {G1.x, G1.y, G1.z, G1.w};
        const float s32[4] = {G2.x, G2.y, G2.z, G2.w}, t32[4] = {G3.x, G3.y, G3.z, G3.w};
        const float zcv[4] = {Z.x, Z.y, Z.z, Z.w};
        const float b = __fsub_rn(__int2float_rn(v), c.v0);
        float nx[4], ny[4], nz[4];
        unsigned special = 0;
#pragma unroll
        for (int q = 0; q < PPL / 2; ++q) {
            const int i0 = 2 * q, i1 = 2 * q + 1;
            float R[2][8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                R[0][k] = q ? RR[k].z : RR[k].x;
                R[1][k] = q ? RR[k].w : RR[k].y;
            }
            const float2 mu = f2(gu32[i0], gu32[i1]), mv = f2(gv32[i0], gv32[i1]);
            const float2 ms = f2(s32[i0], s32[i1]), mt = f2(t32[i0], t32[i1]);
            const float2 zc2 = f2(zcv[i0], zcv[i1]);
            const float2 xu = __fmul2_rn(mu, zc2), xv = __fmul2_rn(mv, zc2);
            const float2 xs = __fmul2_rn(ms, zc2), xt = __fmul2_rn(mt, zc2);
            float2 tau[8];
            float2 sum8;
            if (MODE == MEAN) {
                const float2 p23 = __fmul2_rn(xv, __fadd2_rn(f2(R[0][2], R[1][2]), f2(R[0][3], R[1][3])));
                const float2 p67 = __fmul2_rn(xt, __fadd2_rn(f2(R[0][6], R[1][6]), f2(R[0][7], R[1][7])));
                const float2 s0 = __ffma2_rn(xu, __fadd2_rn(f2(R[0][0], R[1][0]), f2(R[0][1], R[1][1])), p23);
                const float2 s1 = __ffma2_rn(xs, __fadd2_rn(f2(R[0][4], R[1][4]), f2(R[0][5], R[1][5])), p67);
                sum8 = __fadd2_rn(s0, s1);
            } else if (DISP) {
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    const float2 x = (k < 2) ? xu : (k < 4) ? xv : (k < 6) ? xs : xt;
                    tau[k] = __fmul2_rn(x, f2(R[0][k], R[1][k]));
                }
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
            float2 phi;
            if (MODE == MEAN) {
                phi = __fmul2_rn(sum8, f2(0.125f, 0.125f));
                phi = __ffma2_rn(f2(0.f, 0.f), sum8, phi);
            } else {
                float t0[8], t1[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) { t0[k] = tau[k].x; t1[k] = tau[k].y; }
                float a0, b0, a1, b1;
                mid_pair8(t0, a0, b0);
                mid_pair8(t1, a1, b1);
                phi = __fmul2_rn(__fadd2_rn(f2(a0, a1), f2(b0, b1)), f2(0.5f, 0.5f));
                phi = __ffma2_rn(f2(0.f, 0.f), sum8, phi);
            }
            const float2 nzneg = __ffma2_rn(f2(c.a[i0], c.a[i1]), mu, __ffma2_rn(f2(b, b), mv, phi));
            const float2 px = __fmul2_rn(f2(c.fx, c.fx), mu);
            const float2 py = __fmul2_rn(f2(c.fy, c.fy), mv);
            const float2 pz = f2(-nzneg.x, -nzneg.y);
            const float2 dot = __ffma2_rn(px, px, __ffma2_rn(py, py, __fmul2_rn(pz, pz)));
            const float r0 = __uint_as_float(__float_as_uint(rsqrt_approx(dot.x)) | (__float_as_uint(phi.x) & 0x80000000u));
            const float r1 = __uint_as_float(__float_as_uint(rsqrt_approx(dot.y)) | (__float_as_uint(phi.y) & 0x80000000u));
            const float2 sc = f2(r0, r1);
            const float2 ox = __fmul2_rn(px, sc), oy = __fmul2_rn(py, sc), oz = __fmul2_rn(pz, sc);
            nx[i0] = ox.x; nx[i1] = ox.y; ny[i0] = oy.x; ny[i1] = oy.y; nz[i0] = oz.x; nz[i1] = oz.y;
            const bool sp0 = !(fabsf(phi.x) > 0.f) && !isnan(zc2.x);
            const bool sp1 = !(fabsf(phi.y) > 0.f) && !isnan(zc2.y);
            special |= (sp0 ? (1u << i0) : 0u) | (sp1 ? (1u << i1) : 0u);
        }
        const bool row_border = (v == 0) || (v == c.H - 1);
        special &= row_border ? 0u : ~colmask;
        if (__any_sync(0xffffffffu, special != 0)) {
            for (int i = 0; i < PPL; ++i) {
                if (special & (1u << i)) {
                    const Normal n = pixel_general<F, MODE, DISP>(c.img, c.H, c.W, v, c.cm + i, c.u0, c.v0,
                                                                  c.fx, c.fy, c.wt);
                    nx[i] = n.x; ny[i] = n.y; nz[i] = n.z;
                }
            }
        }
        if (c.okm) {
            float* o = reinterpret_cast<float*>(out) + v * c.W;
            store_planar(o, nx);
            store_planar(o + HW, ny);
            store_planar(o + 2 * HW, nz);
        }
    }
}

}  // namespace tfn

extern "C" int ws_run(const float* in, int B, int H, int W, float fx, float fy, float u0, float v0,
                      float* out, int strip_h, int* work, int grid, cudaStream_t st) {
    tfn::KernelArgs a{};
    a.in = in; a.out = out; a.B = B; a.H = H; a.W = W; a.fx = fx; a.fy = fy; a.u0 = u0; a.v0 = v0;
    a.strip_h = strip_h; a.work = work; a.kp = 1; a.k0 = 2;
    auto k = tfn::tfn_ws_kernel<tfn::SOBEL, tfn::MEDIAN, false>;
    const int smem = (int)sizeof(tfn::WsShared);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (grid <= 0) {
        int n = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 64 * WS_PAIRS, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        grid = n * sms;
    }
    if (work) cudaMemsetAsync(work, 0, sizeof(int), st);
    k<<<grid, 64 * WS_PAIRS, smem, st>>>(a);
    return (int)cudaGetLastError();
}

extern "C" int ws_occupancy() {
    int n = 0;
    auto k = tfn::tfn_ws_kernel<tfn::SOBEL, tfn::MEDIAN, false>;
    const int smem = (int)sizeof(tfn::WsShared);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 64 * WS_PAIRS, smem);
    return n;
}
