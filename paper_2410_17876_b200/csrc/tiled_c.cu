// tiled_c.cu — instantiations of the tiled gate kernel for target dimensions 6, 8.
#include "tiled_impl.cuh"

SV_TILED_DIM(6, 6)
SV_TILED_DIM(8, 8)
