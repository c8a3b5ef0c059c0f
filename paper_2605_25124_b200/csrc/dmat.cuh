// Device-resident DistanceMatrix (metrics.hpp:45-57): packed upper-triangle
// tile image (kPT x kPT blocks, see kernels.cuh) in fp32 or fp64.
#pragma once

#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace gmds {
struct Engine;
}

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
  // stress-pass workspaces cached per embedding dimension (reused across
  // calls; a second concurrent user of the same handle gets a fresh one)
  mutable std::mutex mu;
  mutable std::vector<std::pair<int, std::shared_ptr<gmds::Engine>>> engines;
  mutable std::vector<bool> busy;
  // dense row-major fp64 copy for the single-CTA small-n fit (n <= 1024), built once
  mutable std::shared_ptr<gmds::DevBuf<double>> dense;
  // row-sharded (gmds_dmat_gini_sharded): only packed blocks [blk_lo, blk_hi) are held, in a
  // compact buffer; ptr() is the (virtual) base of the full packed image, so block b lives at
  // ptr() + b * kPT^2 elements for b in range
  int64_t blk_lo = 0, blk_hi = -1;
  bool sharded() const { return blk_hi >= 0; }
  const void* ptr() const {
    if (sharded())
      return buf.get() - static_cast<size_t>(blk_lo) * gmds::kPT * gmds::kPT * gmds::dtype_size(storage);
    return shared ? static_cast<const void*>(shared->get() + offset) : buf.get();
  }
};
