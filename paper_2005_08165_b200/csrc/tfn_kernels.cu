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
#include "tfn_strip.cuh"

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
    const long long HW = (long long)p.H * p.W;
    const Normal n = pixel_general<F, MODE, DISP>(p.in + b * HW, p.H, p.W, v, u, p.u0, p.v0, p.fx, p.fy);
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
// dispatch
// ------------------------------------------------------------------------------------
template <int F, int MODE, bool DISP>
static cudaError_t launch_t(const KernelArgs& a, int kernel, int grid_strip, cudaStream_t st) {
    if (kernel == TFN_KERNEL_STRIP) {
        if (a.layout == 0) tfn_strip_kernel<F, MODE, DISP, 0, 0><<<grid_strip, TFN_STRIP_THREADS, 0, st>>>(a);
        else tfn_strip_kernel<F, MODE, DISP, 1, 0><<<grid_strip, TFN_STRIP_THREADS, 0, st>>>(a);
    } else if (kernel == TFN_KERNEL_STRIP_GENERAL) {
        if (a.layout == 0) tfn_strip_kernel<F, MODE, DISP, 0, 1><<<grid_strip, TFN_STRIP_THREADS, 0, st>>>(a);
        else tfn_strip_kernel<F, MODE, DISP, 1, 1><<<grid_strip, TFN_STRIP_THREADS, 0, st>>>(a);
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
static int occ_t(int gen) {
    int n = 0;
    const cudaError_t e =
        gen ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tfn_strip_kernel<F, MODE, DISP, 0, 1>,
                                                            TFN_STRIP_THREADS, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tfn_strip_kernel<F, MODE, DISP, 0, 0>,
                                                            TFN_STRIP_THREADS, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return n;
}
template <int F>
static int occ_f(int mode, bool disp, int gen) {
    if (mode == MEAN) return disp ? occ_t<F, MEAN, true>(gen) : occ_t<F, MEAN, false>(gen);
    return disp ? occ_t<F, MEDIAN, true>(gen) : occ_t<F, MEDIAN, false>(gen);
}
int strip_occupancy(int filter, int mode, bool disp, int gen) {
    switch (filter) {
    case FD: return occ_f<FD>(mode, disp, gen);
    case SOBEL: return occ_f<SOBEL>(mode, disp, gen);
    case SCHARR: return occ_f<SCHARR>(mode, disp, gen);
    default: return occ_f<PREWITT>(mode, disp, gen);
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
