// tfn_f32_inst.cuh — launch / occupancy wrappers of the fp32 unit-step kernel (tfn_f32.cuh)
// for ONE gradient filter F; each tfn_f32_<filter>.cu instantiates them so the filters compile
// in parallel.  Instantiated: fp32 depth / disparity x {mean, median} x {fast, masked} x
// {planar, packed}, fp32 normals.
#pragma once
#include "tfn_f32.cuh"

namespace tfn {
namespace f32 {

template <int F, int MODE, bool DISP, bool VM>
static cudaError_t launch_v(const CUtensorMap& tm, const KernelArgs& a, const Consts& k, int grid, cudaStream_t st) {
    if (a.layout == 0) tfn_f32_kernel<F, MODE, DISP, VM, 0><<<grid, TFN_F32_THREADS, 0, st>>>(tm, a, k);
    else tfn_f32_kernel<F, MODE, DISP, VM, 1><<<grid, TFN_F32_THREADS, 0, st>>>(tm, a, k);
    return cudaGetLastError();
}
template <int F, int MODE>
static cudaError_t launch_m(const CUtensorMap& tm, const KernelArgs& a, const Consts& k, bool disp, bool vm, int grid,
                            cudaStream_t st) {
    if (disp) return vm ? launch_v<F, MODE, true, true>(tm, a, k, grid, st) : launch_v<F, MODE, true, false>(tm, a, k, grid, st);
    return vm ? launch_v<F, MODE, false, true>(tm, a, k, grid, st) : launch_v<F, MODE, false, false>(tm, a, k, grid, st);
}
template <class Kern>
static int occ(Kern kernel) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, TFN_F32_THREADS, 0) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return n;
}

}  // namespace f32

template <int F>
cudaError_t launch_f32(const CUtensorMap& tm, const KernelArgs& a, const f32::Consts& k, int mode, bool disp, bool vm,
                       int grid, cudaStream_t st) {
    return mode == MEAN ? f32::launch_m<F, MEAN>(tm, a, k, disp, vm, grid, st)
                        : f32::launch_m<F, MEDIAN>(tm, a, k, disp, vm, grid, st);
}
template <int F>
int occupancy_f32(int mode, bool disp, bool vm) {
    using namespace f32;
    if (mode == MEAN)
        return disp ? (vm ? occ(tfn_f32_kernel<F, MEAN, true, true, 0>) : occ(tfn_f32_kernel<F, MEAN, true, false, 0>))
                    : (vm ? occ(tfn_f32_kernel<F, MEAN, false, true, 0>) : occ(tfn_f32_kernel<F, MEAN, false, false, 0>));
    return disp ? (vm ? occ(tfn_f32_kernel<F, MEDIAN, true, true, 0>) : occ(tfn_f32_kernel<F, MEDIAN, true, false, 0>))
                : (vm ? occ(tfn_f32_kernel<F, MEDIAN, false, true, 0>) : occ(tfn_f32_kernel<F, MEDIAN, false, false, 0>));
}

}  // namespace tfn

#define TFN_INSTANTIATE_F32(F)                                                                                  \
    namespace tfn {                                                                                            \
    template cudaError_t launch_f32<F>(const CUtensorMap&, const KernelArgs&, const f32::Consts&, int, bool, bool, \
                                       int, cudaStream_t);                                                     \
    template int occupancy_f32<F>(int, bool, bool);                                                            \
    }
