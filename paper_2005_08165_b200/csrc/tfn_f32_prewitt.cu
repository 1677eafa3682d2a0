// tfn_f32_prewitt.cu — fp32 unit-step kernel instantiations for the prewitt filter (see tfn_f32_inst.cuh).
#include "tfn_f32_inst.cuh"
TFN_INSTANTIATE_F32(tfn::PREWITT)
