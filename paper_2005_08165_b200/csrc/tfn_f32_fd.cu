// tfn_f32_fd.cu — fp32 unit-step kernel instantiations for the fd filter (see tfn_f32_inst.cuh).
#include "tfn_f32_inst.cuh"
TFN_INSTANTIATE_F32(tfn::FD)
