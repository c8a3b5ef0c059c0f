// Device DistanceMatrix utilities (host launchers).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gmds.h"

namespace gmds {

struct DStats {
  double sum_sq;   // sum_{i<j} D_ij^2
  double sum;      // sum_{i<j} D_ij
  double min_off;  // min_{i<j} D_ij
  double max_off;  // max_{i<j} D_ij
};

void pack_full(const double* dfull, int64_t n, gmds_dtype storage, void* dpacked, cudaStream_t st);
void unpack_full(const void* dpacked, gmds_dtype storage, int64_t n, double* dfull, bool square, cudaStream_t st);
// rows [r0, r1) of the full fp64 matrix, row-major into dout ((r1 - r0) x n)
void unpack_rows(const void* dpacked, gmds_dtype storage, int64_t n, int64_t r0, int64_t r1, double* dout,
                 cudaStream_t st);
// statistics over packed blocks [blk_lo, blk_hi) (blk_hi < 0: all)
DStats packed_stats(const void* dpacked, gmds_dtype storage, int64_t n, cudaStream_t st, int64_t blk_lo = 0,
                    int64_t blk_hi = -1);
double packed_median(const void* dpacked, gmds_dtype storage, int64_t n, cudaStream_t st);
void double_center_dev(double* dS, int64_t n, cudaStream_t st);

}  // namespace gmds
