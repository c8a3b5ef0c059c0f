// Instantiation + launcher of the merge-based Gini kernel (gini_merge.cuh)
// and the per-row value sort that feeds it.
#include "gini_merge.cuh"

namespace gmds {

#define GMDS_MERGE_ONE(T, TO)                                                                                \
  do {                                                                                                       \
    GMDS_CUDA(cudaFuncSetAttribute(gini_merge_kernel<T, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                   static_cast<int>(smem)));                                                 \
    gini_merge_kernel<T, TO><<<blocks, merge_detail::kMergeThreads, smem, st>>>(ma, static_cast<const T*>(dX), static_cast<TO*>(dout)); \
  } while (0)

void launch_gini_merge(const MergeArgs& ma, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st) {
  // the 32-bit key construction is exact for fp32 inputs only
  if (xt != GMDS_F32) fail(GMDS_ERROR, "gini_merge_kernel: fp32 inputs only");
  if (ot == GMDS_F32) GMDS_MERGE_ONE(float, float);
  else GMDS_MERGE_ONE(float, double);
}

// warp per row: sort the row's nonzeros (feature order in vals/fidx) by value,
// write their feature indices in ascending value order.
template <int K, typename T>
__global__ void row_sort_kernel(const T* __restrict__ vals, const uint16_t* __restrict__ fidx,
                                const int64_t* __restrict__ rowptr, const int* __restrict__ rows, int nrows,
                                uint16_t* __restrict__ sidx, T* __restrict__ svs) {
  const int lane = threadIdx.x & 31;
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nrows; q += (gridDim.x * blockDim.x) >> 5) {
    const int64_t row = rows[q];
    const int64_t b = rowptr[row];
    const int cnt = static_cast<int>(rowptr[row + 1] - b);
    double key[K];
    Payload<true>::Arr<K> idx;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int e = r * 32 + lane;
      key[r] = (e < cnt) ? static_cast<double>(vals[b + e]) : INFINITY;
      idx[r] = (e < cnt) ? static_cast<int>(fidx[b + e]) : 0;
    }
    warp_bitonic_sort<K, true>(key, idx, lane);
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int g = lane * K + r;
      if (g < cnt) {
        sidx[b + g] = static_cast<uint16_t>(idx[r]);
        svs[b + g] = static_cast<T>(key[r]);  // exact: the key is the widened input value
      }
    }
  }
}

void launch_row_sort(const void* vals, gmds_dtype xt, const uint16_t* fidx, const int64_t* rowptr, const int* rows,
                     int nrows, int K, uint16_t* sidx, void* svs, cudaStream_t st) {
  if (nrows <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::max(1, std::min((nrows + 7) / 8, 148 * 8)));
#define GMDS_RS(KK)                                                                                                \
  case KK:                                                                                                         \
    if (xt == GMDS_F32)                                                                                            \
      row_sort_kernel<KK, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(vals), fidx, rowptr, rows, nrows, sidx, static_cast<float*>(svs)); \
    else                                                                                                           \
      row_sort_kernel<KK, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(vals), fidx, rowptr, rows, nrows, sidx, static_cast<double*>(svs)); \
    break;
  switch (K) {
    GMDS_RS(1) GMDS_RS(2) GMDS_RS(4) GMDS_RS(8) GMDS_RS(16) GMDS_RS(32)
    default: fail(GMDS_ERROR, "row sort: bad K");
  }
#undef GMDS_RS
  count_launch();
  check_launch("row_sort_kernel");
}

}  // namespace gmds
