// Device-resident DistanceMatrix (metrics.hpp:45-57): packed upper-triangle
// tile image (kPT x kPT blocks, see kernels.cuh) in fp32 or fp64.
#pragma once

#include <memory>

#include "common.cuh"
#include "kernels.cuh"

struct gmds_dmat {
  int64_t n = 0;
  gmds_dtype storage = GMDS_F64;
  gmds::DevBuf<unsigned char> buf;  // packed image, gmds::packed_elems(n) elements
  // alternatively a view into a multi-nu image produced by one launch
  std::shared_ptr<gmds::DevBuf<unsigned char>> shared;
  size_t offset = 0;
  // per-fit constants (computed once by validate/resolve)
  double sum_sq = 0.0;   // sum_{i<j} D_ij^2   (offdiag_squared_sum, embed.cpp:23-30)
  double sum = 0.0;      // sum_{i<j} D_ij
  double min_off = 0.0;  // min_{i<j} D_ij
  double max_val = 0.0;  // max over the full matrix (0 on the diagonal)
  bool stats = false;
  const void* ptr() const { return shared ? static_cast<const void*>(shared->get() + offset) : buf.get(); }
};
