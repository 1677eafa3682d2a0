// tfn_kernels.h — internal launch interface between the C ABI (tfn_abi.cu) and the
// kernels (tfn_kernels.cu + tfn_strip_<filter>.cu, tfn_stats.cu).  Not part of the public
// ABI (include/tfn.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#ifndef TFN_STRIP_THREADS
#define TFN_STRIP_THREADS 128
#endif
#ifndef TFN_STRIP_MINBLOCKS
#define TFN_STRIP_MINBLOCKS 3
#endif
#ifndef TFN_STRIP_PPL
#define TFN_STRIP_PPL 4          // strip kernel: pixels (columns) per lane
#endif
#define TFN_STRIP_COLS (32 * TFN_STRIP_PPL)   // columns per warp strip
#ifndef TFN_F32_THREADS
#define TFN_F32_THREADS 128      // fp32 unit-step kernel: threads per CTA
#endif
#include "tfn_tma.cuh"


namespace tfn {

enum KernelId { TFN_KERNEL_AUTO = 0, TFN_KERNEL_PIXEL = 1, TFN_KERNEL_STRIP = 2, TFN_KERNEL_STRIP_GENERAL = 3,
                TFN_KERNEL_STRIP_MASKED = 4, TFN_KERNEL_F32 = 5, TFN_KERNEL_F32_MASKED = 6 };

enum InDtype { TFN_IN_F32 = 0, TFN_IN_U16 = 1 };

struct KernelArgs {
    const void* in;      // [B,H,W] depth or disparity: fp32, or uint16 depth codes (in_u16)
    void* out;           // normals, layout 0 planar / 1 packed: fp32 or half [B,3,H,W] / [B,H,W,3],
                         // or octahedral int16 pairs [B,2,H,W] / [B,H,W,2] (out_kind)
    int in_u16;
    int out_kind;        // 0 fp32, 1 half, 2 oct16 (TFN_OPT_OUT_DTYPE)
    long long B;
    int H, W;
    float fx, fy;        // n' = (fx g_u, fy g_v, n_z)   (Eq. 18)
    float u0, v0;        // a = u - u0, b = v - v0 (Eq. 13), principal point rounded to fp32
    int layout;
    int strip_h;         // rows per warp strip (strip kernel)
    int* work;           // zeroed work counter for dynamic strip scheduling (nullptr: static)
    int* fired;          // fast strip variant: += its special row steps (nullptr: not counted)
    float* pts;          // N3: fp32 point cloud, same layout as the normals (nullptr: none)
    float pscale;        //   Z = pscale * sample (depth, incl. uint16 codes) or pscale / d (disparity)
    float ifx, ify;      //   1/fx, 1/fy
    double kp, k0;       // CUSTOM filter weights [kp k0 kp] (ignored by the fixed filters)
    const CUtensorMap* tmap;   // strip kernel, fp32 input: TMA descriptor of the input (tfn_tma.cuh)
};

// fp32 unit-step kernel (tfn_f32.cuh): guard constants computed on the host
struct F32Consts {
    float kp, k0;          // CUSTOM weights (fp32)
    float k0lim, kca, kr;  // guard: V <= (k0lim - kca |a| - kr |b|) |n'|
    float cg, tb;          //   and |Phi| >= cg |n'| + tb V (the orientation is certain)
};
namespace f32 { using Consts = F32Consts; }
template <int F>
cudaError_t launch_f32(const CUtensorMap& tm, const KernelArgs& a, const F32Consts& k, int mode, bool disp, bool vm,
                       int grid, cudaStream_t st);
template <int F>
int occupancy_f32(int mode, bool disp, bool vm);
cudaError_t launch_f32_any(const CUtensorMap& tm, const KernelArgs& a, const F32Consts& k, int filter, int mode,
                           bool disp, bool vm, int grid, cudaStream_t st);
int f32_occupancy(int filter, int mode, bool disp, bool vm);

cudaError_t launch_3f2n(const KernelArgs& a, int filter, int mode, bool disp, int kernel,
                        int grid_strip, cudaStream_t st);

// resident CTAs per SM of the strip kernel variant (occupancy query)
int strip_occupancy(int filter, int mode, bool disp, int variant, int in_u16);   // variant 0 fast, 1 general, 2 masked

// per-filter strip instantiations (tfn_strip_<filter>.cu, compiled in parallel)
template <int F>
cudaError_t launch_strip(const KernelArgs& a, int mode, bool disp, int variant, int grid, cudaStream_t st);
template <int F>
int occupancy_strip(int mode, bool disp, int variant, int in_u16);

// N4: PlanePCA (method 0) / PlaneSVD (method 1) comparator, fp32 normals (tfn_planefit.cu)
cudaError_t launch_planefit(const float* depth, float* out, long long B, int H, int W, double fx, double fy,
                            double u0, double v0, int layout, int method, cudaStream_t st);

// a8: angular-error statistics vs ground truth (off the timed path)
cudaError_t launch_stats(const float* est, const float* gt, long long B, int H, int W,
                         int layout, long long* stats_dev, cudaStream_t st);

// SOL reference for the traffic mix (4 B in, 12 B out per pixel)
cudaError_t launch_sol(const float* in, float* out, long long B, int H, int W, int sms, cudaStream_t st);

// P8 probe: Phi of n groups of 8 candidates (non-finite = skipped)
cudaError_t launch_phi8(const float* cand, long long n, int mode, float* out, int* k_out,
                        cudaStream_t st);

}  // namespace tfn
