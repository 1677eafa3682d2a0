// tfn_kernels.cu — the fused 3F2N stencil kernels for sm_100a.
//
//   tfn_strip_kernel   the production kernel (W % 4 == 0, 16-B aligned buffers):
//                      one warp owns a 128-column x R-row strip; each lane owns 4
//                      adjacent columns and walks down the strip keeping a rolling
//                      3-row register window (sanitized Z, fp64 1/Z, gradient
//                      partial sums, shared pair reciprocals).  One LDG.128 + two
//                      halo LDG.32 per lane-row in, three STG.128 per lane-row out:
//                      16 B/pixel of HBM traffic (4 read + 12 written).
//   tfn_pixel_kernel   one thread per pixel, any W; same arithmetic (bit-identical
//                      results, checked by tests/test_gpu_parity.py).
//
// Both evaluate PAPER.md Eq. 13-21 as described in tfn_device.cuh and
// DESIGN.md §2; neither shares code with oracle/.
#include "tfn_device.cuh"
#include "tfn_kernels.h"

namespace tfn {

// ------------------------------------------------------------------------------------
// one thread per pixel
// ------------------------------------------------------------------------------------
template <int F, int MODE, bool DISP>
__global__ void __launch_bounds__(256) tfn_pixel_kernel(KernelArgs p) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    const long long b = blockIdx.z;
    if (u >= p.W || v >= p.H) return;
    const float* img = p.in + b * (long long)p.H * p.W;
    float s[3][3];
#pragma unroll
    for (int dv = -1; dv <= 1; ++dv)
#pragma unroll
        for (int du = -1; du <= 1; ++du) {
            const int vv = v + dv, uu = u + du;
            const bool in = (vv >= 0) && (vv < p.H) && (uu >= 0) && (uu < p.W);
            s[dv + 1][du + 1] = sanitize(in ? __ldg(img + (long long)vv * p.W + uu) : 0.f);
        }
    // x = 1/z (depth) or d (disparity, Eq. 21), fp64
    auto X = [&](int r, int c) -> double {
        return DISP ? (double)s[r][c] : inv_depth(s[r][c]);
    };
    double gu, gv;
    {
        const double d0 = __dsub_rn(X(1, 2), X(1, 0));
        double dm = 0.0, dp = 0.0;
        if (Taps<F>::corners) {
            dm = __dsub_rn(X(0, 2), X(0, 0));
            dp = __dsub_rn(X(2, 2), X(2, 0));
        }
        gu = grad_tail<F>(grad_head<F>(dm, d0), dp);
    }
    {
        const double d0 = __dsub_rn(X(2, 1), X(0, 1));
        double dm = 0.0, dp = 0.0;
        if (Taps<F>::corners) {
            dm = __dsub_rn(X(2, 0), X(0, 0));
            dp = __dsub_rn(X(2, 2), X(0, 2));
        }
        gv = grad_tail<F>(grad_head<F>(dm, d0), dp);
    }
    const float c = s[1][1];
    float rho[8];
    // E (owner c), W (owner W), S (owner c), N (owner N), SE, NW, SW, NE
    { float R = pair_rcp<DISP>(c, s[1][2]);    rho[0] = rho_owner<DISP>(c, s[1][2], R); }
    { float R = pair_rcp<DISP>(s[1][0], c);    rho[1] = rho_other<DISP>(s[1][0], c, R); }
    { float R = pair_rcp<DISP>(c, s[2][1]);    rho[2] = rho_owner<DISP>(c, s[2][1], R); }
    { float R = pair_rcp<DISP>(s[0][1], c);    rho[3] = rho_other<DISP>(s[0][1], c, R); }
    { float R = pair_rcp<DISP>(c, s[2][2]);    rho[4] = rho_owner<DISP>(c, s[2][2], R); }
    { float R = pair_rcp<DISP>(s[0][0], c);    rho[5] = rho_other<DISP>(s[0][0], c, R); }
    { float R = pair_rcp<DISP>(c, s[2][0]);    rho[6] = rho_owner<DISP>(c, s[2][0], R); }
    { float R = pair_rcp<DISP>(s[0][2], c);    rho[7] = rho_other<DISP>(s[0][2], c, R); }
    const float a = __double2float_rn((double)u - p.u0);
    const float bb = __double2float_rn((double)v - p.v0);
    const Normal n = finish<MODE>(!isnan(c), gu, gv, rho, a, bb, p.fx, p.fy);
    const long long HW = (long long)p.H * p.W;
    const long long pix = (long long)v * p.W + u;
    if (p.layout == 0) {
        float* o = p.out + b * 3 * HW + pix;
        o[0] = n.x; o[HW] = n.y; o[2 * HW] = n.z;
    } else {
        float* o = p.out + (b * HW + pix) * 3;
        o[0] = n.x; o[1] = n.y; o[2] = n.z;
    }
}

// ------------------------------------------------------------------------------------
// warp-strip kernel
// ------------------------------------------------------------------------------------
struct RowRaw { float4 m; float l, r; };

// sanitized Z of columns c0-1 .. c0+4 of row v (NaN outside the image: Q3)
__device__ __forceinline__ RowRaw load_row(const float* __restrict__ img, int v, int c0,
                                           int H, int W) {
    RowRaw q;
    const float NaN = __int_as_float(0x7fffffff);
    q.m = make_float4(NaN, NaN, NaN, NaN);
    q.l = NaN; q.r = NaN;
    if (v >= 0 && v < H) {
        const float* row = img + (long long)v * W;
        if (c0 < W) q.m = __ldg(reinterpret_cast<const float4*>(row + c0));
        if (c0 >= 1 && c0 - 1 < W) q.l = __ldg(row + c0 - 1);
        if (c0 + 4 < W) q.r = __ldg(row + c0 + 4);
    }
    return q;
}

__device__ __forceinline__ void unpack(const RowRaw& q, float z[6]) {
    z[0] = sanitize(q.l);
    z[1] = sanitize(q.m.x); z[2] = sanitize(q.m.y); z[3] = sanitize(q.m.z); z[4] = sanitize(q.m.w);
    z[5] = sanitize(q.r);
}

template <bool DISP>
__device__ __forceinline__ void xrow(const float z[6], double w[6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i) w[i] = DISP ? (double)z[i] : inv_depth(z[i]);
}

__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d, bool cs) {
    float4 v = make_float4(a, b, c, d);
    if (cs) __stcs(reinterpret_cast<float4*>(p), v);
    else *reinterpret_cast<float4*>(p) = v;
}

template <int F, int MODE, bool DISP>
__global__ void __launch_bounds__(TFN_STRIP_THREADS) tfn_strip_kernel(KernelArgs p) {
    const int lane = threadIdx.x & 31;
    const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int sx_n = (p.W + 127) >> 7;
    const int sy_n = (p.H + p.strip_h - 1) / p.strip_h;
    const long long items = (long long)sx_n * sy_n * p.B;
    const long long HW = (long long)p.H * p.W;
    const float fx = p.fx, fy = p.fy;

    for (long long it = warp0; it < items; it += nwarps) {
        const int sx = (int)(it % sx_n);
        const long long t2 = it / sx_n;
        const int sy = (int)(t2 % sy_n);
        const long long b = t2 / sy_n;
        const int c0 = sx * 128 + lane * 4;
        const int y0 = sy * p.strip_h;
        const int y1 = min(y0 + p.strip_h, p.H);
        const float* img = p.in + b * HW;
        float a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = __double2float_rn((double)(c0 + i) - p.u0);

        // ---- prologue: rows y0-1 (prev) and y0 (cur) ----
        float zp[6], zc[6];
        double wp[6], wc[6];
        unpack(load_row(img, y0 - 1, c0, p.H, p.W), zp);
        unpack(load_row(img, y0, c0, p.H, p.W), zc);
        xrow<DISP>(zp, wp);
        xrow<DISP>(zc, wc);
        // gradient head of g_u for row y0: kp*Dh(y0-1) + k0*Dh(y0)
        double head[4], dhc[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double dprev = Taps<F>::corners ? __dsub_rn(wp[i + 2], wp[i]) : 0.0;
            dhc[i] = __dsub_rn(wc[i + 2], wc[i]);
            head[i] = grad_head<F>(dprev, dhc[i]);
        }
        // rho of the N / NW / NE neighbours of row y0 (pairs owned by row y0-1)
        float rN[4], rNW[4], rNE[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            // N: pair (y0-1, c) -> (y0, c), owner prev
            float R = pair_rcp<DISP>(zp[i + 1], zc[i + 1]);
            rN[i] = rho_other<DISP>(zp[i + 1], zc[i + 1], R);
            // NW: pair (y0-1, c-1) -> (y0, c), owner prev
            R = pair_rcp<DISP>(zp[i], zc[i + 1]);
            rNW[i] = rho_other<DISP>(zp[i], zc[i + 1], R);
            // NE: pair (y0-1, c+1) -> (y0, c), e = SW, owner prev
            R = pair_rcp<DISP>(zp[i + 2], zc[i + 1]);
            rNE[i] = rho_other<DISP>(zp[i + 2], zc[i + 1], R);
        }

        RowRaw nxt = load_row(img, y0 + 1, c0, p.H, p.W);
        for (int v = y0; v < y1; ++v) {
            float zn[6];
            unpack(nxt, zn);
            if (v + 1 < y1) nxt = load_row(img, v + 2, c0, p.H, p.W);   // prefetch
            double wn[6];
            xrow<DISP>(zn, wn);

            const float bb = __double2float_rn((double)v - p.v0);
            double dhn[4], gu[4], gv[4];
            double dv[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) dv[i] = __dsub_rn(wn[i], wp[i]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                dhn[i] = __dsub_rn(wn[i + 2], wn[i]);   // centre-row taps of row v+1
                gu[i] = grad_tail<F>(head[i], dhn[i]);
                const double dm = Taps<F>::corners ? dv[i] : 0.0;
                const double dp = Taps<F>::corners ? dv[i + 2] : 0.0;
                gv[i] = grad_tail<F>(grad_head<F>(dm, dv[i + 1]), dp);
            }
            // shared pair reciprocals of this row step (index j <-> column c0 + j - 1):
            //   E  (v,j)->(v,j+1)      j = 0..4     S  (v,j)->(v+1,j)   j = 1..4
            //   SE (v,j)->(v+1,j+1)    j = 0..4     SW (v,j)->(v+1,j-1) j = 1..5
            float rE[5], rS[4], rSE[5], rSW[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                rE[j] = pair_rcp<DISP>(zc[j], zc[j + 1]);
                rSE[j] = pair_rcp<DISP>(zc[j], zn[j + 1]);
                rSW[j] = pair_rcp<DISP>(zc[j + 1], zn[j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) rS[i] = pair_rcp<DISP>(zc[i + 1], zn[i + 1]);

            float ox[4], oy[4], oz[4];
            float nN[4], nNW[4], nNE[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float c = zc[i + 1];
                float rho[8];
                rho[0] = rho_owner<DISP>(c, zc[i + 2], rE[i + 1]);        // E  (owner c)
                rho[1] = rho_other<DISP>(zc[i], c, rE[i]);                // W  (owner W)
                rho[2] = rho_owner<DISP>(c, zn[i + 1], rS[i]);            // S  (owner c)
                rho[3] = rN[i];                                           // N  (owner N)
                rho[4] = rho_owner<DISP>(c, zn[i + 2], rSE[i + 1]);       // SE (owner c)
                rho[5] = rNW[i];                                          // NW (owner NW)
                rho[6] = rho_owner<DISP>(c, zn[i], rSW[i]);               // SW (owner c): rSW[j=i+1]
                rho[7] = rNE[i];                                          // NE (owner NE)
                // the next row's N / NW / NE come from pairs owned by this row
                nN[i] = rho_other<DISP>(c, zn[i + 1], rS[i]);
                nNW[i] = rho_other<DISP>(zc[i], zn[i + 1], rSE[i]);
                nNE[i] = rho_other<DISP>(zc[i + 2], zn[i + 1], rSW[i + 1]);
                const Normal n = finish<MODE>(!isnan(c), gu[i], gv[i], rho, a[i], bb, fx, fy);
                ox[i] = n.x; oy[i] = n.y; oz[i] = n.z;
            }
            if (c0 < p.W) {
                const long long pix = (long long)v * p.W + c0;
                if (p.layout == 0) {
                    float* o = p.out + b * 3 * HW + pix;
                    st4(o, ox[0], ox[1], ox[2], ox[3], p.streaming);
                    st4(o + HW, oy[0], oy[1], oy[2], oy[3], p.streaming);
                    st4(o + 2 * HW, oz[0], oz[1], oz[2], oz[3], p.streaming);
                } else {
                    float* o = p.out + (b * HW + pix) * 3;
                    st4(o, ox[0], oy[0], oz[0], ox[1], p.streaming);
                    st4(o + 4, oy[1], oz[1], ox[2], oy[2], p.streaming);
                    st4(o + 8, oz[2], ox[3], oy[3], oz[3], p.streaming);
                }
            }
            // ---- roll the window down one row ----
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                head[i] = grad_head<F>(dhc[i], dhn[i]);
                dhc[i] = dhn[i];
                rN[i] = nN[i]; rNW[i] = nNW[i]; rNE[i] = nNE[i];
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) { wp[i] = wc[i]; wc[i] = wn[i]; zc[i] = zn[i]; }
        }
    }
}

// ------------------------------------------------------------------------------------
// dispatch
// ------------------------------------------------------------------------------------
template <int F, int MODE, bool DISP>
static cudaError_t launch_t(const KernelArgs& a, int kernel, int grid_strip, cudaStream_t st) {
    if (kernel == TFN_KERNEL_STRIP) {
        tfn_strip_kernel<F, MODE, DISP><<<grid_strip, TFN_STRIP_THREADS, 0, st>>>(a);
    } else {
        dim3 blk(32, 8, 1);
        dim3 grd((a.W + 31) / 32, (a.H + 7) / 8, (unsigned)a.B);
        tfn_pixel_kernel<F, MODE, DISP><<<grd, blk, 0, st>>>(a);
    }
    return cudaGetLastError();
}

template <int F>
static cudaError_t launch_f(const KernelArgs& a, int mode, bool disp, int kernel, int g,
                            cudaStream_t st) {
    if (mode == MEAN)
        return disp ? launch_t<F, MEAN, true>(a, kernel, g, st) : launch_t<F, MEAN, false>(a, kernel, g, st);
    return disp ? launch_t<F, MEDIAN, true>(a, kernel, g, st) : launch_t<F, MEDIAN, false>(a, kernel, g, st);
}

template <int F, int MODE, bool DISP>
static int occ_t() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tfn_strip_kernel<F, MODE, DISP>,
                                                      TFN_STRIP_THREADS, 0) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return n;
}
template <int F>
static int occ_f(int mode, bool disp) {
    if (mode == MEAN) return disp ? occ_t<F, MEAN, true>() : occ_t<F, MEAN, false>();
    return disp ? occ_t<F, MEDIAN, true>() : occ_t<F, MEDIAN, false>();
}
int strip_occupancy(int filter, int mode, bool disp) {
    switch (filter) {
    case FD: return occ_f<FD>(mode, disp);
    case SOBEL: return occ_f<SOBEL>(mode, disp);
    case SCHARR: return occ_f<SCHARR>(mode, disp);
    default: return occ_f<PREWITT>(mode, disp);
    }
}

cudaError_t launch_3f2n(const KernelArgs& a, int filter, int mode, bool disp, int kernel,
                        int grid_strip, cudaStream_t st) {
    switch (filter) {
    case FD: return launch_f<FD>(a, mode, disp, kernel, grid_strip, st);
    case SOBEL: return launch_f<SOBEL>(a, mode, disp, kernel, grid_strip, st);
    case SCHARR: return launch_f<SCHARR>(a, mode, disp, kernel, grid_strip, st);
    default: return launch_f<PREWITT>(a, mode, disp, kernel, grid_strip, st);
    }
}

}  // namespace tfn
