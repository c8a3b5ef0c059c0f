// Instantiation of the K=16 (N=512 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(16)
}  // namespace gmds
