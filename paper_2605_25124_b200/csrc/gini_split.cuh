// K2 v2: Gini distance tiles with zero compaction and sign-split sorts.
//
// Per pair (one warp), z = x_i - x_j is classified into negatives, exact
// zeros and positives.  Zeros contribute nothing to sum_k z_k L[h_k] and
// only shift positions, and every negative ranks below every zero below
// every positive, so (exactly, tie rule included):
//   * negatives and positives are compacted into a per-warp scratch
//     (negatives from slot 0 up, positives from slot 511 down);
//   * either the two sign classes are sorted as two independent halves of
//     one register array (bitonic network stopped at s = H), or all nonzeros
//     are sorted together, whichever network is shorter;
//   * tie groups are found on the sorted registers and shifted back to
//     their real positions (positives by n_neg + #zeros, or #zeros in the
//     single-array mode) before the LUT lookup.
// Pairs with more than 512 nonzeros go to an overflow list handled by the
// full 1024-key kernel (gini_tile_kernel).
//
// Row panels come in two formats: dense (T[p] per row) and bitmask-sparse
// (32-bit presence mask + running popcount per 32 features, then the
// nonzero values in feature order) -- 4x fewer bytes per row for the
// 80%-zero image-like data, which keeps the tile edge at 32 rows.
#pragma once

#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "gini_tile.cuh"

namespace gmds {

constexpr int kSplitCap = 512;  // scratch slots per warp (K_MAX = 16)

struct SplitArgs {
  GiniTileArgs g;
  // sparse row store (format 1)
  const uint32_t* masks;   // [n][W]
  const uint16_t* prefix;  // [n][W] popcount of the row's mask words before w
  const int64_t* rowptr;   // [n+1] into vals
  const void* vals;        // nonzero values (input dtype) in feature order
  int W;                   // ceil(p / 32)
  int maxnnz;              // max nonzeros in any row (panel stride)
  int sparse;              // 1: sparse panels
  // overflow list
  int64_t* ovf_pairs;      // [cap][2]
  unsigned long long* ovf_count;
  int64_t ovf_cap;
};

namespace split_detail {

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }
__device__ __forceinline__ int npow2(int v) { return v <= 1 ? 1 : 1 << (32 - __clz(v - 1)); }

// sum over s = 2..smax of log2(s) = L(L+1)/2 stages, N/2 compare-exchanges each
__device__ __forceinline__ int net_cost(int N, int smax) {
  const int L = ilog2(smax);
  return (N / 2) * (L * (L + 1) / 2);
}

// Bitonic network over N = 32K blocked keys, stopped after merge size smax
// (smax = N: full sort; smax = N/2: the two halves sorted independently).
template <int K>
__device__ __forceinline__ void warp_bitonic_upto(double (&v)[K], int lane, int smax) {
  constexpr int N = 32 * K;
#pragma unroll
  for (int s = 2; s <= N; s <<= 1) {
    // (a guarded body, not a break, so the loop stays fully unrolled and v[] stays in registers)
    if (s <= smax) {
    if (s <= K) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const int r2 = r ^ (s - 1);
        if (r < r2) ce_asc(v[r], v[r2]);
      }
    } else {
      const int m = s / K - 1;
      const bool keep_lo = !(lane & (s / (2 * K)));
#pragma unroll
      for (int r = 0; r < (K + 1) / 2; ++r) {
        const int r2 = K - 1 - r;
        const double o1 = __shfl_xor_sync(kFull, v[r2], m);
        if (r2 != r) {
          const double o2 = __shfl_xor_sync(kFull, v[r], m);
          const bool lt2 = o2 < v[r2], gt2 = v[r2] < o2;
          v[r2] = sel64(keep_lo ? lt2 : gt2, o2, v[r2]);
        }
        const bool lt1 = o1 < v[r], gt1 = v[r] < o1;
        v[r] = sel64(keep_lo ? lt1 : gt1, o1, v[r]);
      }
    }
#pragma unroll
    for (int t = s / 4; t > 0; t >>= 1) {
      if (t < K) {
#pragma unroll
        for (int r = 0; r < K; ++r)
          if (!(r & t)) ce_asc(v[r], v[r + t]);
      } else {
        const int m = t / K;
        const bool keep_lo = !(lane & m);
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const double o = __shfl_xor_sync(kFull, v[r], m);
          const bool lt = o < v[r], gt = v[r] < o;
          v[r] = sel64(keep_lo ? lt : gt, o, v[r]);
        }
      }
    }
    }
  }
}

// Bitonic merge of 2H = 32K blocked keys whose halves are each a bitonic
// sequence (ascending run, +inf padding, descending run): the half-cleaner
// cascade t = H/2 .. 1 (partners stay inside their half).
template <int K>
__device__ __forceinline__ void warp_bitonic_merge(double (&v)[K], int lane) {
  constexpr int H = 16 * K;
#pragma unroll
  for (int t = H / 2; t > 0; t >>= 1) {
    if (t < K) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (!(r & t)) ce_asc(v[r], v[r + t]);
    } else {
      const int m = t / K;
      const bool keep_lo = !(lane & m);
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const double o = __shfl_xor_sync(kFull, v[r], m);
        const bool lt = o < v[r], gt = v[r] < o;
        v[r] = sel64(keep_lo ? lt : gt, o, v[r]);
      }
    }
  }
}

// Tie groups of the sorted split array (negatives in half A, positives in
// half B), shifted to real positions, and the LUT sum for every nu.
template <int K>
__device__ __forceinline__ void finish_split(double (&key)[K], int n_neg, int n_pos, int zeros, int lane,
                                             const double* __restrict__ lut, int d, int nnu, double half_p, bool store,
                                             double* out, size_t ostride, int* flag) {
  constexpr int H = 16 * K;
  int h[K];
  warp_tie_groups<K>(key, h, lane);
  const int shiftB = 2 * (n_neg + zeros) - 2 * H;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int g = lane * K + r;
    int hh = -1;
    if (g < n_neg) hh = h[r];
    else if (g >= H && g < H + n_pos) hh = h[r] + shiftB;
    h[r] = hh;
  }
  for (int v = 0; v < nnu; ++v) {
    const double* L = lut + static_cast<size_t>(v) * 2 * d;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (h[r] >= 0) acc = fma(key[r], __ldg(L + h[r]), acc);
    acc = warp_sum(acc);
    const double val = clamp_nonneg(half_p * acc);
    if (lane == 0 && store) {
      out[v * ostride] = val;
      if (isinf(val)) atomicOr(flag, 1);
    }
  }
}

// Load the compacted nonzeros into blocked registers, sort, find tie groups,
// and for every nu reduce (p/2) * sum_k z_k L[h_k] across the warp; lane 0
// writes the clamped distance to *out (stride ostride between nu values).
template <int K>
__device__ __forceinline__ void sort_and_sum(const double* __restrict__ scr, int n_neg, int n_pos, int zeros,
                                             bool split, int lane, const double* __restrict__ lut, int d, int nnu,
                                             double half_p, bool store, double* out, size_t ostride, int* flag) {
  constexpr int N = 32 * K;
  constexpr int H = N / 2;
  double key[K];
  if (split) {
    const bool hiB = lane >= 16;
    const int l16 = lane & 15;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int e = r * 16 + l16;  // element index within the half
      double v = INFINITY;
      if (!hiB) {
        if (e < n_neg) v = scr[e];
      } else {
        if (e < n_pos) v = scr[kSplitCap - 1 - e];
      }
      key[r] = v;
    }
  } else {
    const int nnz = n_neg + n_pos;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int e = r * 32 + lane;
      double v = INFINITY;
      if (e < n_neg)
        v = scr[e];
      else if (e < nnz)
        v = scr[kSplitCap - 1 - (e - n_neg)];
      key[r] = v;
    }
  }
  warp_bitonic_upto<K>(key, lane, split ? H : N);
  int h[K];
  warp_tie_groups<K>(key, h, lane);
  // real position of each slot's tie group: h -> h' (or -1 for padding)
  const int shiftB = 2 * (n_neg + zeros) - 2 * H;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int g = lane * K + r;
    int hh = -1;
    if (split) {
      if (g < n_neg) hh = h[r];
      else if (g >= H && g < H + n_pos) hh = h[r] + shiftB;
    } else {
      if (g < n_neg) hh = h[r];
      else if (g < n_neg + n_pos) hh = h[r] + 2 * zeros;
    }
    h[r] = hh;
  }
  for (int v = 0; v < nnu; ++v) {
    const double* L = lut + static_cast<size_t>(v) * 2 * d;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (h[r] >= 0) acc = fma(key[r], __ldg(L + h[r]), acc);
    acc = warp_sum(acc);
    const double val = clamp_nonneg(half_p * acc);
    if (lane == 0 && store) {
      out[v * ostride] = val;
      if (isinf(val)) atomicOr(flag, 1);
    }
  }
}

}  // namespace split_detail

// One CTA = 8 warps on a tile x tile block of pairs.  SPARSE selects the panel format.
// CTAs per SM: 3 for K <= 8 (80 registers, no spills; measured equal or up to
// 30% faster than 2 on dense p = 32..256 inputs), 2 for K = 16 (spills at 85)
constexpr int split_min_blocks(int km) { return km <= 8 ? 3 : 2; }
template <int KMAX, bool SPARSE, typename T, typename TO>
__global__ void __launch_bounds__(256, split_min_blocks(KMAX)) gini_split_kernel(SplitArgs sa, const T* __restrict__ X, TO* __restrict__ out) {
  using namespace split_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const GiniTileArgs& a = sa.g;
  const int tile = a.tile;
  const int d = a.d;
  const int W = sa.W;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  // shared layout: [scratch: nwarps x 512 double][otile: nnu x tile x (tile+1) double][panels]
  double* scratch = reinterpret_cast<double*>(smem_raw) + warp * kSplitCap;
  double* otile = reinterpret_cast<double*>(smem_raw) + nwarps * kSplitCap;
  const int tstride = tile + 1;
  unsigned char* pbase = reinterpret_cast<unsigned char*>(otile + static_cast<size_t>(a.nnu) * tile * tstride);
  // dense panel: rows [2*tile][d] of T; sparse panel: masks [2*tile][W] u32, prefix [2*tile][W] u16,
  // vals [2*tile][maxnnz] T
  T* dpanel = reinterpret_cast<T*>(pbase);
  uint32_t* smask = reinterpret_cast<uint32_t*>(pbase);
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + 2 * tile * W);
  T* svals = reinterpret_cast<T*>(
      pbase + ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)));
  const T* sv = static_cast<const T*>(sa.vals);
  const double half_p = 0.5 * static_cast<double>(d);
  const unsigned lt = (1u << lane) - 1u;
  __shared__ double s_score[2 * kMaxScoreNu];
  __shared__ double s_red[32 * 8];
  for (int e = threadIdx.x; e < 2 * kMaxScoreNu; e += blockDim.x) s_score[e] = 0.0;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * tile, j0 = J * tile;
    // ---- stage panels: rows 0..tile-1 = block I, tile..2tile-1 = block J
    if constexpr (!SPARSE) {
      for (int64_t e = threadIdx.x; e < 2 * static_cast<int64_t>(tile) * d; e += blockDim.x) {
        const int64_t r = e / d, c = e % d;
        const int64_t row = (r < tile) ? i0 + r : j0 + (r - tile);
        dpanel[e] = (row < a.n) ? X[row * d + c] : T(0);
      }
    } else {
      for (int e = threadIdx.x; e < 2 * tile * W; e += blockDim.x) {
        const int r = e / W, w = e % W;
        const int64_t row = (r < tile) ? i0 + r : j0 + (r - tile);
        smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
        spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
      }
      for (int r = warp; r < 2 * tile; r += nwarps) {
        const int64_t row = (r < tile) ? i0 + r : j0 + (r - tile);
        if (row < a.n) {
          const int64_t b = sa.rowptr[row], e1 = sa.rowptr[row + 1];
          for (int64_t k = b + lane; k < e1; k += 32) svals[static_cast<size_t>(r) * sa.maxnnz + (k - b)] = sv[k];
        }
      }
    }
    __syncthreads();

    const int per_warp = (tile * tile + nwarps - 1) / nwarps;
    for (int it = 0; it < per_warp; ++it) {
      const int k = warp + it * nwarps;
      const int kk = (k < tile * tile) ? k : 0;
      const int r = kk / tile, c = kk % tile;
      const int64_t i = i0 + r, j = j0 + c;
      const bool valid = (k < tile * tile) && (j < a.n) && (i < j);
      const int ri = r, rj = valid ? tile + c : r;  // invalid: the zero pair (i, i)
      // ---- build z, classify, compact (negatives up from 0, positives down from 511)
      int n_neg = 0, n_pos = 0;
      for (int w = 0; w < W; ++w) {
        const int e = w * 32 + lane;
        double z = 0.0;
        if constexpr (!SPARSE) {
          if (e < d) z = static_cast<double>(dpanel[ri * d + e]) - static_cast<double>(dpanel[rj * d + e]);
        } else {
          const uint32_t mi = smask[ri * W + w], mj = smask[rj * W + w];
          T av = T(0), bv = T(0);
          if ((mi >> lane) & 1u) av = svals[static_cast<size_t>(ri) * sa.maxnnz + spre[ri * W + w] + __popc(mi & lt)];
          if ((mj >> lane) & 1u) bv = svals[static_cast<size_t>(rj) * sa.maxnnz + spre[rj * W + w] + __popc(mj & lt)];
          z = static_cast<double>(av) - static_cast<double>(bv);
        }
        const unsigned mn = __ballot_sync(kFull, z < 0.0);
        const unsigned mp = __ballot_sync(kFull, z > 0.0);
        if (z < 0.0) {
          const int slot = n_neg + __popc(mn & lt);
          if (slot < kSplitCap) scratch[slot] = z;
        } else if (z > 0.0) {
          const int slot = kSplitCap - 1 - (n_pos + __popc(mp & lt));
          if (slot >= 0) scratch[slot] = z;
        }
        n_neg += __popc(mn);
        n_pos += __popc(mp);
      }
      __syncwarp();
      const int nnz = n_neg + n_pos;
      const int zeros = d - nnz;
      // ---- choose the shorter network
      const int Nf = max(32, npow2(nnz));
      const int Hs = max(16, npow2(max(n_neg, n_pos)));
      const int Ns = 2 * Hs;
      const bool split = net_cost(Ns, Hs) <= net_cost(Nf, Nf);
      const int Nsel = split ? Ns : Nf;
      const bool overflow = nnz > kSplitCap || Nsel > 32 * KMAX;
      double* ot = otile + static_cast<size_t>(r) * tstride + c;
      const size_t ostride = static_cast<size_t>(tile) * tstride;
      if (overflow) {
        if (valid && lane == 0) {
          const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
          if (static_cast<int64_t>(slot) < sa.ovf_cap) {
            sa.ovf_pairs[2 * slot] = i;
            sa.ovf_pairs[2 * slot + 1] = j;
          }
          for (int v = 0; v < a.nnu; ++v) ot[v * ostride] = -1.0;  // filled by the overflow pass
        }
      } else if (nnz == 0) {
        if (valid && lane == 0)
          for (int v = 0; v < a.nnu; ++v) ot[v * ostride] = 0.0;
      } else {
        switch (Nsel / 32) {
          case 1: sort_and_sum<1>(scratch, n_neg, n_pos, zeros, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
          case 2: sort_and_sum<2>(scratch, n_neg, n_pos, zeros, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
          case 4: sort_and_sum<4>(scratch, n_neg, n_pos, zeros, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
          case 8:
            if constexpr (KMAX >= 8)
              sort_and_sum<8>(scratch, n_neg, n_pos, zeros, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag);
            break;
          default:
            if constexpr (KMAX >= 16)
              sort_and_sum<16>(scratch, n_neg, n_pos, zeros, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag);
            break;
        }
      }
      __syncwarp();  // scratch reuse
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, tile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}

template <int KMAX>
void launch_gini_split(const SplitArgs& sa, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st);

#define GMDS_SPLIT_ONE(KM, SP, T, TO)                                                                                \
  do {                                                                                                               \
    GMDS_CUDA(cudaFuncSetAttribute(gini_split_kernel<KM, SP, T, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   static_cast<int>(smem)));                                                         \
    gini_split_kernel<KM, SP, T, TO><<<blocks, 256, smem, st>>>(sa, static_cast<const T*>(dX), static_cast<TO*>(dout)); \
  } while (0)

#define GMDS_INSTANTIATE_SPLIT(KM)                                                                                  \
  template <>                                                                                                       \
  void launch_gini_split<KM>(const SplitArgs& sa, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot,        \
                             size_t smem, unsigned blocks, cudaStream_t st) {                                       \
    if (sa.sparse) {                                                                                                \
      if (xt == GMDS_F32 && ot == GMDS_F32) GMDS_SPLIT_ONE(KM, true, float, float);                                \
      else if (xt == GMDS_F32) GMDS_SPLIT_ONE(KM, true, float, double);                                            \
      else if (ot == GMDS_F32) GMDS_SPLIT_ONE(KM, true, double, float);                                            \
      else GMDS_SPLIT_ONE(KM, true, double, double);                                                               \
    } else {                                                                                                        \
      if (xt == GMDS_F32 && ot == GMDS_F32) GMDS_SPLIT_ONE(KM, false, float, float);                               \
      else if (xt == GMDS_F32) GMDS_SPLIT_ONE(KM, false, float, double);                                           \
      else if (ot == GMDS_F32) GMDS_SPLIT_ONE(KM, false, double, float);                                           \
      else GMDS_SPLIT_ONE(KM, false, double, double);                                                              \
    }                                                                                                               \
  }

}  // namespace gmds
