// tiled_a.cu — instantiations of the tiled gate kernel for target dimensions 2, 3.
#include "tiled_impl.cuh"

SV_TILED_DIM(2, 2)
SV_TILED_DIM(3, 3)
