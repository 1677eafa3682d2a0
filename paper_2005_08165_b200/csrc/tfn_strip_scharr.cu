// tfn_strip_scharr.cu — strip-kernel instantiations for the scharr gradient filter (see tfn_strip_inst.cuh).
#include "tfn_strip_inst.cuh"
TFN_INSTANTIATE_STRIP(tfn::SCHARR)
