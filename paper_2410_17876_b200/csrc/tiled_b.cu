// tiled_b.cu — instantiations of the tiled gate kernel for target dimensions 4, 5.
#include "tiled_impl.cuh"

SV_TILED_DIM(4, 4)
SV_TILED_DIM(5, 5)
