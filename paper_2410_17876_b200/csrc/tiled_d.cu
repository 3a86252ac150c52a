// tiled_d.cu — instantiations of the tiled gate kernel for target dimensions 9, 10.
#include "tiled_impl.cuh"

SV_TILED_DIM(9, 9)
SV_TILED_DIM(10, 10)
