// Instantiation of the K=1 (N=32 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(1)
}  // namespace gmds
