// tfn_strip_sobel.cu — strip-kernel instantiations for the sobel gradient filter (see tfn_strip_inst.cuh).
#include "tfn_strip_inst.cuh"
TFN_INSTANTIATE_STRIP(tfn::SOBEL)
