// Instantiation of the K=2 (N=64 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(2)
}  // namespace gmds
