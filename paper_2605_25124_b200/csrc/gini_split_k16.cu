// Instantiation of the zero-compacting, sign-split Gini kernel with K_MAX = 16.
#include "gini_split.cuh"

namespace gmds {
GMDS_INSTANTIATE_SPLIT(16)
}  // namespace gmds
