// tfn_strip_custom.cu — strip-kernel instantiations for the run-time-weight gradient filter
// [kp k0 kp]^T (x) [-1 0 1] (see tfn_strip_inst.cuh).
#include "tfn_strip_inst.cuh"
TFN_INSTANTIATE_STRIP(tfn::CUSTOM)
