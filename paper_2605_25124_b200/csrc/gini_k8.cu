// Instantiation of the K=8 (N=256 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(8)
}  // namespace gmds
