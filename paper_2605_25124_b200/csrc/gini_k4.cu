// Instantiation of the K=4 (N=128 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(4)
}  // namespace gmds
