// tfn_kernels.cu — the per-pixel 3F2N kernel and the launch dispatch for sm_100a (the strip
// kernel's instantiations live in tfn_strip_<filter>.cu).
//
//   tfn_strip_kernel   the production kernel (tfn_strip.cuh; W % 4 == 0, vector-aligned
//                      buffers): warp strips with a rolling 3-row register window,
//                      16 B/pixel of HBM traffic for fp32 in / fp32 normals out.
//   tfn_pixel_kernel   one thread per pixel, any W / alignment; the same device
//                      routines (bit-identical results, tests/test_gpu_parity.py).
//
// Both evaluate PAPER.md Eq. 13-21 as described in tfn_device.cuh and
// DESIGN.md §2; neither shares code with oracle/.
#include <cuda_fp16.h>

#include "tfn_device.cuh"
#include "tfn_kernels.h"
#include "tfn_strip.cuh"      // oct16 (the normal encoding shared with the strip kernel)

namespace tfn {

// ------------------------------------------------------------------------------------
// one thread per pixel
// ------------------------------------------------------------------------------------
template <int F, int MODE, bool DISP, class T>
__global__ void __launch_bounds__(256) tfn_pixel_kernel(KernelArgs p) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    const long long b = blockIdx.z;
    if (u >= p.W || v >= p.H) return;
    const long long HW = (long long)p.H * p.W;
    const Normal n = pixel_general<F, MODE, DISP>(reinterpret_cast<const T*>(p.in) + b * HW, p.H, p.W, v, u,
                                                  p.u0, p.v0, p.fx, p.fy, Wts{p.kp, p.k0});
    const long long pix = (long long)v * p.W + u;
    const long long i0 = p.layout == 0 ? b * 3 * HW + pix : (b * HW + pix) * 3;
    const long long st = p.layout == 0 ? HW : 1;
    if (p.out_kind == 2) {
        const unsigned w = oct16(n.x, n.y, n.z);
        short* o = reinterpret_cast<short*>(p.out) + (p.layout == 0 ? b * 2 * HW + pix : (b * HW + pix) * 2);
        o[0] = (short)(w & 0xffffu);
        o[p.layout == 0 ? HW : 1] = (short)(w >> 16);
    } else if (p.out_kind == 1) {
        __half* o = reinterpret_cast<__half*>(p.out) + i0;
        o[0] = __float2half_rn(n.x); o[st] = __float2half_rn(n.y); o[2 * st] = __float2half_rn(n.z);
    } else {
        float* o = reinterpret_cast<float*>(p.out) + i0;
        o[0] = n.x; o[st] = n.y; o[2 * st] = n.z;
    }
    if (p.pts) {      // N3 point cloud (same formulas as the strip kernel)
        const float zs = sanitize(sample_f(__ldg(reinterpret_cast<const T*>(p.in) + b * HW + pix)));
        const float Z = DISP ? __fdiv_rn(p.pscale, zs) : __fmul_rn(zs, p.pscale);
        const float a = __fsub_rn(__int2float_rn(u), p.u0), bb = __fsub_rn(__int2float_rn(v), p.v0);
        float* q = p.pts + i0;
        q[0] = __fmul_rn(__fmul_rn(a, Z), p.ifx);
        q[st] = __fmul_rn(__fmul_rn(bb, Z), p.ify);
        q[2 * st] = Z;
    }
}

// ------------------------------------------------------------------------------------
// dispatch
// ------------------------------------------------------------------------------------
template <int F, int MODE>
static cudaError_t launch_pixel(const KernelArgs& a0, bool disp, cudaStream_t st) {
    if (a0.in_u16 && disp) return cudaErrorInvalidValue;
    // frames on grid z, at most 65535 per launch: larger batches go in chunks
    const long long HW = (long long)a0.H * a0.W;
    const size_t in_b = a0.in_u16 ? 2 : 4;
    const size_t out_px = a0.out_kind == 0 ? 12 : a0.out_kind == 1 ? 6 : 4;
    for (long long b0 = 0; b0 < a0.B; b0 += 65535) {
        KernelArgs a = a0;
        a.B = (a0.B - b0 < 65535) ? a0.B - b0 : 65535;
        a.in = static_cast<const char*>(a0.in) + b0 * HW * in_b;
        a.out = static_cast<char*>(a0.out) + b0 * HW * out_px;
        if (a0.pts) a.pts = a0.pts + b0 * 3 * HW;
        dim3 blk(32, 8, 1);
        dim3 grd((a.W + 31) / 32, (a.H + 7) / 8, (unsigned)a.B);
        if (a.in_u16) tfn_pixel_kernel<F, MODE, false, unsigned short><<<grd, blk, 0, st>>>(a);
        else if (disp) tfn_pixel_kernel<F, MODE, true, float><<<grd, blk, 0, st>>>(a);
        else tfn_pixel_kernel<F, MODE, false, float><<<grd, blk, 0, st>>>(a);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int F>
static cudaError_t launch_f(const KernelArgs& a, int mode, bool disp, int kernel, int g, cudaStream_t st) {
    if (kernel == TFN_KERNEL_STRIP || kernel == TFN_KERNEL_STRIP_GENERAL || kernel == TFN_KERNEL_STRIP_MASKED)
        return launch_strip<F>(a, mode, disp,
                               kernel == TFN_KERNEL_STRIP_GENERAL ? 1 : kernel == TFN_KERNEL_STRIP_MASKED ? 2 : 0, g, st);
    return mode == MEAN ? launch_pixel<F, MEAN>(a, disp, st) : launch_pixel<F, MEDIAN>(a, disp, st);
}

int strip_occupancy(int filter, int mode, bool disp, int variant, int in_u16) {
    switch (filter) {
    case FD: return occupancy_strip<FD>(mode, disp, variant, in_u16);
    case SOBEL: return occupancy_strip<SOBEL>(mode, disp, variant, in_u16);
    case SCHARR: return occupancy_strip<SCHARR>(mode, disp, variant, in_u16);
    case PREWITT: return occupancy_strip<PREWITT>(mode, disp, variant, in_u16);
    default: return occupancy_strip<CUSTOM>(mode, disp, variant, in_u16);
    }
}

cudaError_t launch_f32_any(const CUtensorMap& tm, const KernelArgs& a, const F32Consts& k, int filter, int mode,
                           bool disp, bool vm, int grid, cudaStream_t st) {
    switch (filter) {
    case FD: return launch_f32<FD>(tm, a, k, mode, disp, vm, grid, st);
    case SOBEL: return launch_f32<SOBEL>(tm, a, k, mode, disp, vm, grid, st);
    case SCHARR: return launch_f32<SCHARR>(tm, a, k, mode, disp, vm, grid, st);
    case PREWITT: return launch_f32<PREWITT>(tm, a, k, mode, disp, vm, grid, st);
    default: return launch_f32<CUSTOM>(tm, a, k, mode, disp, vm, grid, st);
    }
}

int f32_occupancy(int filter, int mode, bool disp, bool vm) {
    switch (filter) {
    case FD: return occupancy_f32<FD>(mode, disp, vm);
    case SOBEL: return occupancy_f32<SOBEL>(mode, disp, vm);
    case SCHARR: return occupancy_f32<SCHARR>(mode, disp, vm);
    case PREWITT: return occupancy_f32<PREWITT>(mode, disp, vm);
    default: return occupancy_f32<CUSTOM>(mode, disp, vm);
    }
}

cudaError_t launch_3f2n(const KernelArgs& a, int filter, int mode, bool disp, int kernel,
                        int grid_strip, cudaStream_t st) {
    switch (filter) {
    case FD: return launch_f<FD>(a, mode, disp, kernel, grid_strip, st);
    case SOBEL: return launch_f<SOBEL>(a, mode, disp, kernel, grid_strip, st);
    case SCHARR: return launch_f<SCHARR>(a, mode, disp, kernel, grid_strip, st);
    case PREWITT: return launch_f<PREWITT>(a, mode, disp, kernel, grid_strip, st);
    default: return launch_f<CUSTOM>(a, mode, disp, kernel, grid_strip, st);
    }
}

}  // namespace tfn
