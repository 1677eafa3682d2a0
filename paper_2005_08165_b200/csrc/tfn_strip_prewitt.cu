// tfn_strip_prewitt.cu — strip-kernel instantiations for the prewitt gradient filter (see tfn_strip_inst.cuh).
#include "tfn_strip_inst.cuh"
TFN_INSTANTIATE_STRIP(tfn::PREWITT)
