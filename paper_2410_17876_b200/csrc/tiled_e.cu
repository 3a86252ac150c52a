// tiled_e.cu — instantiations of the tiled gate kernel for target dimensions 12, 15.
#include "tiled_impl.cuh"

SV_TILED_DIM(12, 12)
SV_TILED_DIM(15, 15)
