// tiled_f.cu — instantiations of the tiled gate kernel for target dimensions 16, generic.
#include "tiled_impl.cuh"

SV_TILED_DIM(16, 16)
SV_TILED_DIM(0, 16)
