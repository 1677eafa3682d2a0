// tfn_stats.cu — SURVEY.md §8(a) row a8 (off the timed path): angular-error
// statistics of an estimated normal map against ground truth, Eq. 22-24
// (P:293-323), with the pooled evaluation mask of reading Q18 and psi evaluated as
// atan2(|a x b|, a.b) (Q16).  Integer fixed-point sums so the NCCL all-reduce over
// ranks is bit-exact for any number of GPUs.
//
// Also the P8 probe kernel: Phi of groups of 8 candidates through the same device
// code the stencil kernels use (tfn_device.cuh).
#include "tfn_device.cuh"
#include "tfn_kernels.h"

namespace tfn {

// stats layout (int64): [0] sum psi in 1e-6 deg, [1] m (both valid), [2..4] psi<=10/20/30,
// [5] valid estimates, [6] valid GT, [7] pixels
__global__ void __launch_bounds__(256) tfn_stats_kernel(const float* __restrict__ est,
                                                        const float* __restrict__ gt,
                                                        long long B, int H, int W, int layout,
                                                        unsigned long long* stats) {
    const long long HW = (long long)H * W;
    const long long N = B * HW;
    unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / HW, pix = i - b * HW;
        float e0, e1, e2;
        if (layout == 0) {
            const float* e = est + b * 3 * HW + pix;
            e0 = e[0]; e1 = e[HW]; e2 = e[2 * HW];
        } else {
            const float* e = est + i * 3;
            e0 = e[0]; e1 = e[1]; e2 = e[2];
        }
        const float* g = gt + b * 3 * HW + pix;
        const float g0 = g[0], g1 = g[HW], g2 = g[2 * HW];
        const bool ve = isfinite(e0) && isfinite(e1) && isfinite(e2);
        const bool vg = isfinite(g0) && isfinite(g1) && isfinite(g2);
        acc[7] += 1;
        acc[5] += ve;
        acc[6] += vg;
        if (ve && vg) {
            const double a0 = e0, a1 = e1, a2 = e2, b0 = g0, b1 = g1, b2 = g2;
            const double c0 = a1 * b2 - a2 * b1, c1 = a2 * b0 - a0 * b2, c2 = a0 * b1 - a1 * b0;
            const double psi = atan2(sqrt(c0 * c0 + c1 * c1 + c2 * c2), a0 * b0 + a1 * b1 + a2 * b2) *
                               (180.0 / 3.14159265358979323846);
            acc[0] += (unsigned long long)llrint(psi * 1.0e6);
            acc[1] += 1;
            acc[2] += psi <= 10.0;
            acc[3] += psi <= 20.0;
            acc[4] += psi <= 30.0;
        }
    }
    __shared__ unsigned long long red[8][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        unsigned long long v = acc[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        unsigned long long v = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
        atomicAdd(stats + threadIdx.x, v);
    }
}

cudaError_t launch_stats(const float* est, const float* gt, long long B, int H, int W,
                         int layout, long long* stats_dev, cudaStream_t st) {
    const long long N = B * (long long)H * W;
    long long blocks = (N + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    tfn_stats_kernel<<<(unsigned)blocks, 256, 0, st>>>(est, gt, B, H, W, layout,
                                                      reinterpret_cast<unsigned long long*>(stats_dev));
    return cudaGetLastError();
}

// Speed-of-light reference for the 3F2N traffic mix: 4 B read + 12 B
// written per pixel with the strip kernel's access pattern (one LDG.128 per lane-row,
// three streaming STG.128 into the planar normal map), no arithmetic.
__global__ void __launch_bounds__(256) tfn_sol_kernel(const float4* __restrict__ in, float4* __restrict__ out,
                                                     long long quads_per_frame, long long frames) {
    const long long n = quads_per_frame * frames;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long f = i / quads_per_frame, q = i - f * quads_per_frame;
        const float4 z = __ldg(in + i);
        float4* o = out + f * 3 * quads_per_frame + q;
        __stcs(o, z);
        __stcs(o + quads_per_frame, z);
        __stcs(o + 2 * quads_per_frame, z);
    }
}

cudaError_t launch_sol(const float* in, float* out, long long B, int H, int W, int sms, cudaStream_t st) {
    const long long qpf = (long long)H * W / 4;
    long long blocks = (qpf * B + 255) / 256;
    if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
    if (blocks < 1) blocks = 1;
    tfn_sol_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in),
                                                      reinterpret_cast<float4*>(out), qpf, B);
    return cudaGetLastError();
}

template <int MODE>
__global__ void tfn_phi8_kernel(const float* __restrict__ cand, long long n, float* out, int* kout) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = cand[i * 8 + j];
    const float sum8 = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
    float phi;
    int k = 8;
    if (MODE == 2) {
        // the strip kernel's fast / masked median (TFN_PHI_EXT): the NaN-propagating network
        // and its extreme-magnitude test decide the fast path instead of the candidate sum
        float u[8], v3, v4, ext;
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = t[j];
        mid_pair8_ext(u, v3, v4, ext);
        if (fabsf(ext) < __int_as_float(0x7f800000)) phi = __fmul_rn(__fadd_rn(v3, v4), 0.5f);
        else phi = phi_general<MEDIAN>(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], &k);
    } else if (fabsf(sum8) < __int_as_float(0x7f800000)) {
        phi = phi_all8<MODE>(t, sum8);
    } else {
        phi = phi_general<MODE>(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], &k);
    }
    out[i] = phi;
    kout[i] = k;
}

cudaError_t launch_phi8(const float* cand, long long n, int mode, float* out, int* k_out,
                        cudaStream_t st) {
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    if (mode == MEAN) tfn_phi8_kernel<MEAN><<<blocks, 256, 0, st>>>(cand, n, out, k_out);
    else if (mode == MEDIAN) tfn_phi8_kernel<MEDIAN><<<blocks, 256, 0, st>>>(cand, n, out, k_out);
    else tfn_phi8_kernel<2><<<blocks, 256, 0, st>>>(cand, n, out, k_out);
    return cudaGetLastError();
}

}  // namespace tfn
