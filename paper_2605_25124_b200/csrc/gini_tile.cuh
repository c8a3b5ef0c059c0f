// Templates of the warp-per-pair kernels (K1 midrank, K2 Gini tiles),
// instantiated per keys-per-lane K in gini_k*.cu so the heavy unrolled
// bodies compile in parallel.  See gini_kernels.cu for the arithmetic.
#pragma once

#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "warp_rank.cuh"

namespace gmds {

namespace gini_detail {

__device__ __forceinline__ double clamp_nonneg(double v) {
  // std::max(0.0, v) of metrics.cpp:162: (0 < v) ? v : 0 -- NaN maps to 0.
  return (0.0 < v) ? v : 0.0;
}

// Row-major upper-triangle enumeration of tiles (I <= J) over nbt tile rows.
__device__ __forceinline__ void decode_tile(int64_t t, int64_t nbt, int64_t& I, int64_t& J) {
  const double b = 2.0 * static_cast<double>(nbt) + 1.0;
  int64_t i = static_cast<int64_t>((b - sqrt(b * b - 8.0 * static_cast<double>(t))) * 0.5);
  if (i < 0) i = 0;
  auto start = [nbt](int64_t r) { return r * nbt - (r * (r - 1)) / 2; };
  while (i > 0 && start(i) > t) --i;
  while (start(i + 1) <= t) ++i;
  I = i;
  J = i + (t - start(i));
}

}  // namespace gini_detail
using namespace gini_detail;

__host__ __device__ int64_t packed_offset(int64_t i, int64_t j, int64_t nb);

// Tile epilogue shared by the tile / split / merge kernels.  Store mode:
// otile (per nu, tile x (tile+1)) written coalesced to the full n x n image
// (both triangles) or the packed triangle; negative values mark pairs the
// overflow pass fills.  Score mode: per-nu sums of (dist - D)^2 and D^2,
// reduced in a fixed order (warp xor-trees, then warp partials in order)
// into the CTA accumulator sacc[2 nu].
template <typename TO>
__device__ __forceinline__ void tile_epilogue(const GiniTileArgs& a, const double* otile, int tile, int tstride,
                                              int64_t i0, int64_t j0, TO* out, double* sacc, double* sred) {
  if (a.Y == nullptr) {
    for (int v = 0; v < a.nnu; ++v) {
      const double* ot = otile + static_cast<size_t>(v) * tile * tstride;
      TO* o = out + static_cast<size_t>(v) * a.out_stride;
      if (a.packed) {
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int r = e / tile, c = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = ot[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[packed_offset(i, j, a.nb_packed)] = static_cast<TO>(val);
        }
      } else {
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int r = e / tile, c = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = ot[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[i * a.n + j] = static_cast<TO>(val);
        }
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int c = e / tile, r = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = ot[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[j * a.n + i] = static_cast<TO>(val);
        }
      }
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int v0 = 0; v0 < a.nnu; v0 += 4) {
    const int nv = min(4, a.nnu - v0);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
      const int r = e / tile, c = e % tile;
      const int64_t i = i0 + r, j = j0 + c;
      if (!(j < a.n && i < j)) continue;
      double d2 = 0.0;  // embedded_distance (embed.cpp:32-34)
      for (int k = 0; k < a.q; ++k) {
        const double dy = a.Y[i * a.q + k] - a.Y[j * a.q + k];
        d2 += dy * dy;
      }
      const double dist = sqrt(d2);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (v >= nv) break;
        const double Dv = otile[(static_cast<size_t>(v0 + v) * tile + r) * tstride + c];
        if (Dv < 0.0) atomicOr(a.flag, 2);  // overflow pair: not computed here
        const double ee = dist - Dv;
        acc[2 * v] += ee * ee;
        acc[2 * v + 1] += Dv * Dv;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double x = acc[k];
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) x += __shfl_xor_sync(0xffffffffu, x, dd);
      if (lane == 0) sred[warp * 8 + k] = x;
    }
    __syncthreads();
    if (threadIdx.x < 2 * nv) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += sred[w * 8 + threadIdx.x];
      sacc[2 * v0 + threadIdx.x] += t;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void score_flush(const GiniTileArgs& a, const double* sacc) {
  if (a.Y == nullptr) return;
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * a.nnu; e += blockDim.x)
    a.score_part[static_cast<size_t>(blockIdx.x) * 2 * a.nnu + e] = sacc[e];
}


// ---------------------------------------------------------------------------
// K1: segmented midrank, warp per segment (segment length d <= 32*K).

template <int K, typename T>
__global__ void __launch_bounds__(256) midrank_warp_kernel(const double* __restrict__ v, const T* __restrict__ X,
                                                           const int64_t* __restrict__ pairs, int64_t nseg, int d,
                                                           double* __restrict__ ranks) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t s = warp; s < nseg; s += nwarps) {
    double key[K];
    Payload<true>::Arr<K> idx;
    const T* xi = nullptr;
    const T* xj = nullptr;
    if (pairs) {
      xi = X + pairs[2 * s] * d;
      xj = X + pairs[2 * s + 1] * d;
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int e = r * 32 + lane;
      idx[r] = e;
      if (e < d)
        key[r] = pairs ? (static_cast<double>(xi[e]) - static_cast<double>(xj[e])) : v[s * d + e];
      else
        key[r] = INFINITY;
    }
    warp_bitonic_sort<K, true>(key, idx, lane);
    int h[K];
    warp_tie_groups<K>(key, h, lane);
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (idx[r] < d) ranks[s * d + idx[r]] = 0.5 * static_cast<double>(h[r] + 1);
  }
}

// ---------------------------------------------------------------------------
// K2: Gini distance tiles.  CTA = 8 warps on a tile x tile block of pairs.

template <int K, typename T, typename TO>
__global__ void __launch_bounds__(256) gini_tile_kernel(GiniTileArgs a, const T* __restrict__ X, TO* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tile = a.tile;
  const int d = a.d;
  T* rowsI = reinterpret_cast<T*>(smem_raw);
  T* rowsJ = rowsI + static_cast<size_t>(tile) * d;
  size_t panel_bytes = 2 * static_cast<size_t>(tile) * d * sizeof(T);
  panel_bytes = (panel_bytes + 15) & ~static_cast<size_t>(15);
  double* otile = reinterpret_cast<double*>(smem_raw + panel_bytes);  // [nnu][tile][tile+1]
  const int tstride = tile + 1;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const double half_p = 0.5 * static_cast<double>(d);
  __shared__ double s_score[2 * kMaxScoreNu];
  __shared__ double s_red[32 * 8];
  for (int e = threadIdx.x; e < 2 * kMaxScoreNu; e += blockDim.x) s_score[e] = 0.0;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * tile, j0 = J * tile;
    const bool diag = (I == J);
    // stage the two row panels (coalesced; rows past n are zero)
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(tile) * d; e += blockDim.x) {
      const int64_t r = e / d, c = e % d;
      rowsI[e] = (i0 + r < a.n) ? X[(i0 + r) * d + c] : T(0);
      if (!diag) rowsJ[e] = (j0 + r < a.n) ? X[(j0 + r) * d + c] : T(0);
    }
    __syncthreads();
    const T* pj = diag ? rowsI : rowsJ;

    // Every warp runs the same trip count with no data-dependent branch
    // around the shuffles (a divergent-looking region makes ptxas wrap each
    // shuffle in WARPSYNC/collective fallback code); invalid pairs (i >= j,
    // j >= n) are computed on the zero row pair and simply not stored.
    const int per_warp = (tile * tile + nwarps - 1) / nwarps;
    for (int it = 0; it < per_warp; ++it) {
      const int k = warp + it * nwarps;
      const int kk = (k < tile * tile) ? k : 0;
      const int r = kk / tile, c = kk % tile;
      const int64_t i = i0 + r, j = j0 + c;
      const bool valid = (k < tile * tile) && (j < a.n) && (i < j);
      const T* xi = rowsI + static_cast<size_t>(r) * d;
      const T* xj = valid ? pj + static_cast<size_t>(c) * d : xi;
      double key[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int e = q * 32 + lane;
        key[q] = (e < d) ? (static_cast<double>(xi[e]) - static_cast<double>(xj[e])) : INFINITY;
      }
      Payload<false>::Arr<K> nop;
      warp_bitonic_sort<K, false>(key, nop, lane);
      int h[K];
      warp_tie_groups<K>(key, h, lane);
      for (int v = 0; v < a.nnu; ++v) {
        const double* L = a.lut + static_cast<size_t>(v) * 2 * d;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (lane * K + q < d) acc = fma(key[q], __ldg(L + h[q]), acc);
        acc = warp_sum(acc);
        const double val = clamp_nonneg(half_p * acc);
        if (lane == 0 && valid) {
          otile[(static_cast<size_t>(v) * tile + r) * tstride + c] = val;
          if (isinf(val)) atomicOr(a.flag, 1);
        }
      }
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, tile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}


// Overflow pairs of the split kernel (more than 512 nonzeros): warp per
// listed pair, full N = 32K sort straight from the row-major X in HBM/L2.
template <int K, typename T, typename TO>
__global__ void __launch_bounds__(256) gini_list_kernel(GiniTileArgs a, const T* __restrict__ X,
                                                        const int64_t* __restrict__ pairs, int64_t npairs,
                                                        TO* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int d = a.d;
  const double half_p = 0.5 * static_cast<double>(d);
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = w0; q < npairs; q += nw) {
    const int64_t i = pairs[2 * q], j = pairs[2 * q + 1];
    double key[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int e = r * 32 + lane;
      key[r] = (e < d) ? static_cast<double>(X[i * d + e]) - static_cast<double>(X[j * d + e]) : INFINITY;
    }
    Payload<false>::Arr<K> nop;
    warp_bitonic_sort<K, false>(key, nop, lane);
    int h[K];
    warp_tie_groups<K>(key, h, lane);
    for (int v = 0; v < a.nnu; ++v) {
      const double* L = a.lut + static_cast<size_t>(v) * 2 * d;
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (lane * K + r < d) acc = fma(key[r], __ldg(L + h[r]), acc);
      acc = warp_sum(acc);
      const double val = clamp_nonneg(half_p * acc);
      if (lane == 0) {
        TO* o = out + static_cast<size_t>(v) * a.out_stride;
        if (a.packed) {
          o[packed_offset(i, j, a.nb_packed)] = static_cast<TO>(val);
        } else {
          o[i * a.n + j] = static_cast<TO>(val);
          o[j * a.n + i] = static_cast<TO>(val);
        }
        if (isinf(val)) atomicOr(a.flag, 1);
      }
    }
  }
}

template <int K>
void launch_gini_list(GiniTileArgs a, const void* dX, gmds_dtype xt, const int64_t* pairs, int64_t npairs, void* dout,
                      gmds_dtype ot, cudaStream_t st);

template <int K>
void launch_midrank_warp(const double* dv, const void* dX, gmds_dtype xt, const int64_t* dpairs, int64_t nseg, int d,
                         double* dranks, dim3 g, int threads, cudaStream_t st);
template <int K>
void launch_gini_tile(GiniTileArgs a, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                      unsigned blocks, cudaStream_t st);

#define GMDS_INSTANTIATE_K(KK)                                                                                    \
  template <>                                                                                                     \
  void launch_midrank_warp<KK>(const double* dv, const void* dX, gmds_dtype xt, const int64_t* dpairs,            \
                               int64_t nseg, int d, double* dranks, dim3 g, int threads, cudaStream_t st) {       \
    if (xt == GMDS_F32)                                                                                           \
      midrank_warp_kernel<KK, float><<<g, threads, 0, st>>>(dv, static_cast<const float*>(dX), dpairs, nseg, d,  \
                                                            dranks);                                             \
    else                                                                                                          \
      midrank_warp_kernel<KK, double><<<g, threads, 0, st>>>(dv, static_cast<const double*>(dX), dpairs, nseg, d, \
                                                             dranks);                                            \
  }                                                                                                               \
  template <typename T, typename TO>                                                                              \
  static void gini_tile_##KK(GiniTileArgs a, const void* dX, void* dout, size_t smem, unsigned blocks,            \
                             cudaStream_t st) {                                                                   \
    GMDS_CUDA(cudaFuncSetAttribute(gini_tile_kernel<KK, T, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                   static_cast<int>(smem)));                                                      \
    gini_tile_kernel<KK, T, TO><<<blocks, 256, smem, st>>>(a, static_cast<const T*>(dX), static_cast<TO*>(dout)); \
  }                                                                                                               \
  template <typename T, typename TO>                                                                              \
  static void gini_list_##KK(GiniTileArgs a, const void* dX, const int64_t* pairs, int64_t np, void* dout,        \
                             cudaStream_t st) {                                                                   \
    const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((np + 7) / 8, 148 * 8))); \
    gini_list_kernel<KK, T, TO><<<blocks, 256, 0, st>>>(a, static_cast<const T*>(dX), pairs, np,                 \
                                                       static_cast<TO*>(dout));                                  \
  }                                                                                                               \
  template <>                                                                                                     \
  void launch_gini_list<KK>(GiniTileArgs a, const void* dX, gmds_dtype xt, const int64_t* pairs, int64_t np,     \
                            void* dout, gmds_dtype ot, cudaStream_t st) {                                         \
    if (xt == GMDS_F32 && ot == GMDS_F32) gini_list_##KK<float, float>(a, dX, pairs, np, dout, st);               \
    else if (xt == GMDS_F32) gini_list_##KK<float, double>(a, dX, pairs, np, dout, st);                           \
    else if (ot == GMDS_F32) gini_list_##KK<double, float>(a, dX, pairs, np, dout, st);                           \
    else gini_list_##KK<double, double>(a, dX, pairs, np, dout, st);                                              \
  }                                                                                                               \
  template <>                                                                                                     \
  void launch_gini_tile<KK>(GiniTileArgs a, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem, \
                            unsigned blocks, cudaStream_t st) {                                                   \
    if (xt == GMDS_F32 && ot == GMDS_F32) gini_tile_##KK<float, float>(a, dX, dout, smem, blocks, st);            \
    else if (xt == GMDS_F32) gini_tile_##KK<float, double>(a, dX, dout, smem, blocks, st);                        \
    else if (ot == GMDS_F32) gini_tile_##KK<double, float>(a, dX, dout, smem, blocks, st);                        \
    else gini_tile_##KK<double, double>(a, dX, dout, smem, blocks, st);                                           \
  }

}  // namespace gmds
