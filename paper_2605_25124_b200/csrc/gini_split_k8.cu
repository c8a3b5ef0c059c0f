// Instantiation of the zero-compacting, sign-split Gini kernel with K_MAX = 8.
#include "gini_split.cuh"

namespace gmds {
GMDS_INSTANTIATE_SPLIT(8)
}  // namespace gmds
