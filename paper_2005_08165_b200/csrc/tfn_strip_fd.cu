// tfn_strip_fd.cu — strip-kernel instantiations for the fd gradient filter (see tfn_strip_inst.cuh).
#include "tfn_strip_inst.cuh"
TFN_INSTANTIATE_STRIP(tfn::FD)
