// tfn_strip_inst.cuh — launch / occupancy wrappers of the strip kernel for ONE gradient
// filter F; each tfn_strip_<filter>.cu instantiates them, so the four filters compile in
// parallel.  Instantiated set: fp32 input x {depth, disparity} x {mean, median} x
// {planar, packed} x {fast, general}; uint16 depth codes (N1) x {mean, median} x
// {planar, packed} x {general} (integer-quantized depth makes dZ = 0 common, so the
// fast variant's special path would run on most row steps); and the general variant with
// the fused point cloud (N3) for every input.  The fast variant is compiled per normal
// encoding (fp32 / half / oct16); the general one reads it at run time; points run the
// general variant (same bits).
#pragma once
#include "tfn_device.cuh"
#include "tfn_kernels.h"
#include "tfn_strip.cuh"

namespace tfn {

template <int F, int MODE, bool DISP, int KV, class T, bool PTS = false, int OUT = 2>
static cudaError_t launch_l(const KernelArgs& a, int grid, cudaStream_t st) {
    if (a.layout == 0) tfn_strip_kernel<F, MODE, DISP, 0, KV, T, PTS, OUT><<<grid, TFN_STRIP_THREADS, 0, st>>>(*a.tmap, a);
    else tfn_strip_kernel<F, MODE, DISP, 1, KV, T, PTS, OUT><<<grid, TFN_STRIP_THREADS, 0, st>>>(*a.tmap, a);
    return cudaGetLastError();
}

template <int F, int MODE, bool DISP, int KV = 0>
static cudaError_t launch_fast(const KernelArgs& a, int grid, cudaStream_t st) {
    return a.out_kind == 1 ? launch_l<F, MODE, DISP, KV, float, false, 1>(a, grid, st)
         : a.out_kind == 2 ? launch_l<F, MODE, DISP, KV, float, false, 3>(a, grid, st)
                           : launch_l<F, MODE, DISP, KV, float, false, 0>(a, grid, st);
}

// variant 0 = fast, 1 = general, 2 = masked (fast + tap-validity special test); uint16
// input and points always run general
template <int F, int MODE>
static cudaError_t launch_m(const KernelArgs& a, bool disp, int variant, int grid, cudaStream_t st) {
    if (a.in_u16) {
        if (disp) return cudaErrorInvalidValue;
        if (a.pts) return launch_l<F, MODE, false, 1, unsigned short, true>(a, grid, st);
        // the normal encoding at compile time (N1's uint16 -> half workload is ALU-bound:
        // no per-store run-time encoding branch)
        return a.out_kind == 1 ? launch_l<F, MODE, false, 1, unsigned short, false, 1>(a, grid, st)
             : a.out_kind == 2 ? launch_l<F, MODE, false, 1, unsigned short, false, 3>(a, grid, st)
                               : launch_l<F, MODE, false, 1, unsigned short, false, 0>(a, grid, st);
    }
    if (a.pts)
        return disp ? launch_l<F, MODE, true, 1, float, true>(a, grid, st)
                    : launch_l<F, MODE, false, 1, float, true>(a, grid, st);
    if (disp) return variant == 1 ? launch_l<F, MODE, true, 1, float>(a, grid, st)
                   : variant == 2 ? launch_fast<F, MODE, true, 2>(a, grid, st) : launch_fast<F, MODE, true>(a, grid, st);
    return variant == 1 ? launch_l<F, MODE, false, 1, float>(a, grid, st)
         : variant == 2 ? launch_fast<F, MODE, false, 2>(a, grid, st) : launch_fast<F, MODE, false>(a, grid, st);
}

template <int F>
cudaError_t launch_strip(const KernelArgs& a, int mode, bool disp, int variant, int grid, cudaStream_t st) {
    return mode == MEAN ? launch_m<F, MEAN>(a, disp, variant, grid, st) : launch_m<F, MEDIAN>(a, disp, variant, grid, st);
}

template <class K>
static int occ(K kernel) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, TFN_STRIP_THREADS, 0) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return n;
}

template <int F, int MODE>
static int occ_m(bool disp, int variant, int in_u16) {
    if (in_u16) return occ(tfn_strip_kernel<F, MODE, false, 0, 1, unsigned short, false, 2>);
    if (disp) return variant == 1 ? occ(tfn_strip_kernel<F, MODE, true, 0, 1, float, false, 2>)
                   : variant == 2 ? occ(tfn_strip_kernel<F, MODE, true, 0, 2, float, false, 0>)
                                  : occ(tfn_strip_kernel<F, MODE, true, 0, 0, float, false, 0>);
    return variant == 1 ? occ(tfn_strip_kernel<F, MODE, false, 0, 1, float, false, 2>)
         : variant == 2 ? occ(tfn_strip_kernel<F, MODE, false, 0, 2, float, false, 0>)
                        : occ(tfn_strip_kernel<F, MODE, false, 0, 0, float, false, 0>);
}

template <int F>
int occupancy_strip(int mode, bool disp, int variant, int in_u16) {
    return mode == MEAN ? occ_m<F, MEAN>(disp, variant, in_u16) : occ_m<F, MEDIAN>(disp, variant, in_u16);
}

}  // namespace tfn

#define TFN_INSTANTIATE_STRIP(F)                                                                        \
    namespace tfn {                                                                                    \
    template cudaError_t launch_strip<F>(const KernelArgs&, int, bool, int, int, cudaStream_t);       \
    template int occupancy_strip<F>(int, bool, int, int);                                              \
    }
