// Instantiation + launcher of the merge-based Gini kernel (gini_merge.cuh)
// and the per-row value sort that feeds it.
#include "gini_merge.cuh"

namespace gmds {

#define GMDS_MERGE_ONE(T, TO)                                                                                \
  do {                                                                                                       \
    if (ma.fast) {                                                                                           \
      GMDS_CUDA(cudaFuncSetAttribute(gini_merge_kernel<T, TO, true>,                                         \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));  \
      gini_merge_kernel<T, TO, true><<<blocks, merge_detail::kMergeThreads, smem, st>>>(                     \
          ma, static_cast<const T*>(dX), static_cast<TO*>(dout));                                            \
    } else {                                                                                                 \
      GMDS_CUDA(cudaFuncSetAttribute(gini_merge_kernel<T, TO, false>,                                        \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));  \
      gini_merge_kernel<T, TO, false><<<blocks, merge_detail::kMergeThreads, smem, st>>>(                    \
          ma, static_cast<const T*>(dX), static_cast<TO*>(dout));                                            \
    }                                                                                                        \
  } while (0)

void launch_gini_merge(const MergeArgs& ma, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st) {
  // the 32-bit key construction is exact for fp32 inputs only
  if (xt != GMDS_F32) fail(GMDS_ERROR, "gini_merge_kernel: fp32 inputs only");
  if (ot == GMDS_F32) GMDS_MERGE_ONE(float, float);
  else GMDS_MERGE_ONE(float, double);
}

// warp per row: sort the row's nonzeros (feature order in vals/fidx) by value,
// write their feature indices and values in ascending value order, and the
// per-row data of the linear-weight path (gini_merge.cuh, gmd_pair):
// pmap[e] = sorted position of the row's e-th nonzero (feature order),
// suf[k] = sum of the sorted values at positions >= k (fp64), and per row
// s1 = sum of the values, tm = sum_k v_(k) * k (pairs' maxima).
template <int K, typename T>
__global__ void row_sort_kernel(const T* __restrict__ vals, const uint16_t* __restrict__ fidx,
                                const int64_t* __restrict__ rowptr, const int* __restrict__ rows, int nrows,
                                uint16_t* __restrict__ sidx, T* __restrict__ svs, uint16_t* __restrict__ pmap,
                                double* __restrict__ suf, double* __restrict__ s1, double* __restrict__ tm,
                                uint32_t* __restrict__ tiew) {
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
      idx[r] = (e < cnt) ? e : 0;  // feature-order index
    }
    warp_bitonic_sort<K, true>(key, idx, lane);
    double loc[K + 1];
    loc[K] = 0.0;
    double tsum = 0.0;
#pragma unroll
    for (int r = K - 1; r >= 0; --r) {
      const int g = lane * K + r;
      const double v = (g < cnt) ? key[r] : 0.0;
      loc[r] = v + loc[r + 1];
      tsum = fma(v, static_cast<double>(g), tsum);
    }
    // exclusive suffix over lanes: sum of the lanes above
    double incl = loc[0];
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const double o = __shfl_down_sync(0xffffffffu, incl, dd);
      if (lane + dd < 32) incl += o;
    }
    const double above = incl - loc[0];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int g = lane * K + r;
      if (g < cnt) {
        const int e = idx[r];
        sidx[b + g] = fidx[b + e];
        svs[b + g] = static_cast<T>(key[r]);  // exact: the key is the widened input value
        if (pmap) {
          pmap[b + e] = static_cast<uint16_t>(g);
          suf[b + g] = loc[r] + above;
        }
      }
    }
    if (pmap) {
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, dd);
      if (lane == 0) {
        s1[row] = incl;  // lane 0: the whole row
        tm[row] = tsum;
      }
      if constexpr (K <= 8) {  // tie words (rows of <= 256 nonzeros): bit g = (v_(g) == v_(g+1))
        const double nxt0 = __shfl_down_sync(0xffffffffu, key[0], 1);
        uint32_t mine = 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int g = lane * K + r;
          const double nx = (r + 1 < K) ? key[r + 1 < K ? r + 1 : 0] : nxt0;
          if (g + 1 < cnt && key[r] == nx) mine |= 1u << r;
        }
        uint32_t word = mine << ((lane * K) & 31);  // 32 / K lanes per word
#pragma unroll
        for (int dd = 1; dd < 32 / K; dd <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, dd);
        const int w = (lane * K) >> 5;
        if (((lane * K) & 31) == 0 && w < 8) tiew[row * 8 + w] = word;
      }
    }
  }
}

void launch_row_sort(const void* vals, gmds_dtype xt, const uint16_t* fidx, const int64_t* rowptr, const int* rows,
                     int nrows, int K, uint16_t* sidx, void* svs, uint16_t* pmap, double* suf, double* s1,
                     double* tm, uint32_t* tiew, cudaStream_t st) {
  if (nrows <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::max(1, std::min((nrows + 7) / 8, 148 * 8)));
#define GMDS_RS(KK)                                                                                                \
  case KK:                                                                                                         \
    if (xt == GMDS_F32)                                                                                            \
      row_sort_kernel<KK, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(vals), fidx, rowptr, rows, nrows, sidx, static_cast<float*>(svs), pmap, suf, s1, tm, tiew); \
    else                                                                                                           \
      row_sort_kernel<KK, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(vals), fidx, rowptr, rows, nrows, sidx, static_cast<double*>(svs), pmap, suf, s1, tm, tiew); \
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
