// Instantiation of the K=32 (N=1024 keys per pair) warp kernels.
#include "gini_tile.cuh"

namespace gmds {
GMDS_INSTANTIATE_K(32)
}  // namespace gmds
