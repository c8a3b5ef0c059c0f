// Rank and distance kernels (sm_100a):
//   K1 midrank_warp_kernel / midrank_block_kernel -- exact segmented midranks
//      (public midrank API and the pair-rank verification path),
//   K2 gini_tile_kernel  -- Gini distance matrix, one sort per pair shared by
//      every nu, warp per pair, X tile panels staged in shared memory,
//   K2b gini_block_kernel -- same for p > 1024 (CTA per pair, keys in smem
//      or global scratch),
//   euclid_kernel -- pairwise_matrix's Euclidean branch, bit-exact fp64.
// Reference arithmetic: metrics.cpp:42-93 (ranks / directed distance),
// 157-163 (symmetrised, clamped), 193-237 (pairwise loop).  The closed form
// used here:
//   D_ij = max(0, (p/2) * sum_k z_k * L[h_k]),  h_k = 2 R_k - 1 = a + b
//   L[h] = (pow(S'(R), nu-1) - c) - (pow(S(R), nu-1) - c),
// with S(R) = 1 - (R - 1/2)/p (forward) and S'(R) = S(p + 1 - R) (backward
// direction, whose midranks are exactly p + 1 - R).  L is built on the host
// with the reference's own expressions and std::pow, so every per-term
// factor is bit-identical to the reference's; only the summation order
// differs (round-off, well inside the 1e-6 contract).
#include <math.h>

#include "gini_tile.cuh"

namespace gmds {


__host__ __device__ int64_t packed_offset(int64_t i, int64_t j, int64_t nb) {
  // (i < j) -> offset in the packed upper-triangle tile image (kPT x kPT blocks).
  const int64_t I = i / kPT, J = j / kPT;
  const int64_t blk = I * nb - (I * (I - 1)) / 2 + (J - I);
  return blk * (kPT * kPT) + (i % kPT) * kPT + (j % kPT);
}

int64_t packed_elems(int64_t n) {
  const int64_t nb = (n + kPT - 1) / kPT;
  return nb * (nb + 1) / 2 * kPT * kPT;
}

// Block-level bitonic sort of n2 (power of two) keys (+ optional int payload)
// in memory `key` (shared or global scratch), direction-free form.
__device__ void block_bitonic(double* key, int* idx, int n2) {
  for (int s = 2; s <= n2; s <<= 1) {
    for (int t = s / 2; t > 0; t >>= 1) {
      for (int g = threadIdx.x; g < n2 / 2; g += blockDim.x) {
        int i, j;
        if (t == s / 2) {
          const int blk = g / t, off = g % t;
          i = blk * s + off;
          j = blk * s + s - 1 - off;
        } else {
          const int blk = g / t, off = g % t;
          i = blk * 2 * t + off;
          j = i + t;
        }
        const double a = key[i], b = key[j];
        if (b < a) {
          key[i] = b;
          key[j] = a;
          if (idx) {
            const int ti = idx[i];
            idx[i] = idx[j];
            idx[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

// h = a + b of slot g's tie group in a sorted array (binary searches).
__device__ __forceinline__ int group_h(const double* key, int n2, int g) {
  const double x = key[g];
  int lo = 0, hi = g;  // first index with key == x (key[lo..g] ; key < x before)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key[mid] < x) lo = mid + 1; else hi = mid;
  }
  int lo2 = g + 1, hi2 = n2;  // first index > g with key > x
  while (lo2 < hi2) {
    const int mid = (lo2 + hi2) >> 1;
    if (x < key[mid]) hi2 = mid; else lo2 = mid + 1;
  }
  return lo + lo2;
}

template <typename T>
__global__ void midrank_block_kernel(const double* __restrict__ v, const T* __restrict__ X,
                                     const int64_t* __restrict__ pairs, int64_t nseg, int d, int n2,
                                     double* __restrict__ scratch_keys, int* __restrict__ scratch_idx,
                                     double* __restrict__ ranks) {
  extern __shared__ unsigned char smem_raw[];
  double* key;
  int* idx;
  if (scratch_keys) {
    key = scratch_keys + static_cast<int64_t>(blockIdx.x) * n2;
    idx = scratch_idx + static_cast<int64_t>(blockIdx.x) * n2;
  } else {
    key = reinterpret_cast<double*>(smem_raw);
    idx = reinterpret_cast<int*>(key + n2);
  }
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    for (int e = threadIdx.x; e < n2; e += blockDim.x) {
      double k = INFINITY;
      if (e < d) {
        if (pairs)
          k = static_cast<double>(X[pairs[2 * s] * d + e]) - static_cast<double>(X[pairs[2 * s + 1] * d + e]);
        else
          k = v[s * d + e];
      }
      key[e] = k;
      idx[e] = e;
    }
    __syncthreads();
    block_bitonic(key, idx, n2);
    for (int g = threadIdx.x; g < n2; g += blockDim.x) {
      if (idx[g] < d) ranks[s * d + idx[g]] = 0.5 * static_cast<double>(group_h(key, n2, g) + 1);
    }
    __syncthreads();
  }
}

// K2b: p > 1024.  CTA per pair; keys in shared memory or global scratch.
template <typename T, typename TO>
__global__ void gini_block_kernel(GiniTileArgs a, const T* __restrict__ X, TO* __restrict__ out, int n2,
                                  double* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* key = scratch ? scratch + static_cast<int64_t>(blockIdx.x) * n2 : reinterpret_cast<double*>(smem_raw);
  __shared__ double red[32];
  const int d = a.d;
  const double half_p = 0.5 * static_cast<double>(d);
  const int64_t npairs_total = a.n * (a.n - 1) / 2;
  // pair enumeration: row-major upper triangle of rows, split by [pair_begin, pair_end)
  for (int64_t pr = a.tile_begin + blockIdx.x; pr < a.tile_end && pr < npairs_total; pr += gridDim.x) {
    int64_t i, jj;
    decode_tile(pr, a.n - 1, i, jj);  // rows of the strict upper triangle: (i, j = jj + 1)
    const int64_t j = jj + 1;
    if (!tile_in_blocks(a, i, j)) continue;
    for (int e = threadIdx.x; e < n2; e += blockDim.x)
      key[e] = (e < d) ? static_cast<double>(X[i * d + e]) - static_cast<double>(X[j * d + e]) : INFINITY;
    __syncthreads();
    block_bitonic(key, nullptr, n2);
    for (int v = 0; v < a.nnu; ++v) {
      const double* L = a.lut + static_cast<size_t>(v) * 2 * d;
      double acc = 0.0;
      for (int g = threadIdx.x; g < d; g += blockDim.x) acc = fma(key[g], L[group_h(key, n2, g)], acc);
      acc = warp_sum(acc);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        const double val = clamp_nonneg(half_p * s);
        if (isinf(val)) atomicOr(a.flag, 1);
        TO* o = out + static_cast<size_t>(v) * a.out_stride;
        if (a.packed) {
          o[packed_offset(i, j, a.nb_packed)] = static_cast<TO>(val);
        } else {
          o[i * a.n + j] = static_cast<TO>(val);
          o[j * a.n + i] = static_cast<TO>(val);
        }
      }
      __syncthreads();
    }
  }
}

// Euclidean branch (metrics.cpp:220-235): sequential fp64 sum of squares,
// no FMA contraction, so entries are bit-identical to the reference.
template <typename T>
__global__ void euclid_kernel(const T* __restrict__ X, int64_t n, int d, double* __restrict__ out) {
  const int64_t npairs = n * (n - 1) / 2;
  for (int64_t pr = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; pr < npairs;
       pr += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t i, jj;
    decode_tile(pr, n - 1, i, jj);
    const int64_t j = jj + 1;
    double sq = 0.0;
    for (int c = 0; c < d; ++c) {
      const double delta = __dsub_rn(static_cast<double>(X[i * d + c]), static_cast<double>(X[j * d + c]));
      sq = __dadd_rn(sq, __dmul_rn(delta, delta));
    }
    const double v = sqrt(sq);
    out[i * n + j] = v;
    out[j * n + i] = v;
  }
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t rows, int64_t cols, T* __restrict__ out) {
  // in: column-major rows x cols  ->  out: row-major rows x cols
  __shared__ T tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[c * rows + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) out[r * cols + c] = tile[threadIdx.x][k];
  }
}

// ---------------------------------------------------------------------------
// Host launchers.

namespace {

int pick_k(int d) {
  int n2 = 32;
  while (n2 < d) n2 <<= 1;
  return n2 / 32;
}

template <typename T>
void launch_midrank_t(const double* dv, const T* dX, const int64_t* dpairs, int64_t nseg, int d, double* dranks,
                      cudaStream_t st) {
  if (nseg == 0) return;
  if (d <= 1024) {
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(nseg, threads / 32), 148 * 16);
    const dim3 g(static_cast<unsigned>(blocks));
    const gmds_dtype xt = sizeof(T) == 4 ? GMDS_F32 : GMDS_F64;
    switch (pick_k(d)) {
      case 1: launch_midrank_warp<1>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      case 2: launch_midrank_warp<2>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      case 4: launch_midrank_warp<4>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      case 8: launch_midrank_warp<8>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      case 16: launch_midrank_warp<16>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      case 32: launch_midrank_warp<32>(dv, dX, xt, dpairs, nseg, d, dranks, g, threads, st); break;
      default: fail(GMDS_ERROR, "midrank: bad K");
    }
    count_launch();
    check_launch("midrank_warp_kernel");
    return;
  }
  int n2 = 1;
  while (n2 < d) n2 <<= 1;
  const size_t smem = static_cast<size_t>(n2) * (sizeof(double) + sizeof(int));
  const int64_t blocks = std::min<int64_t>(nseg, 296);
  DevBuf<double> sk;
  DevBuf<int> si;
  size_t dyn = smem;
  if (smem > 200 * 1024) {
    sk.alloc(static_cast<size_t>(blocks) * n2);
    si.alloc(static_cast<size_t>(blocks) * n2);
    dyn = 0;
  } else {
    GMDS_CUDA(cudaFuncSetAttribute(midrank_block_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  }
  midrank_block_kernel<T><<<static_cast<unsigned>(blocks), 256, dyn, st>>>(dv, dX, dpairs, nseg, d, n2, sk.get(),
                                                                           si.get(), dranks);
  count_launch();
  check_launch("midrank_block_kernel");
  if (sk.get()) GMDS_CUDA(cudaStreamSynchronize(st));  // scratch freed on return
}

template <typename T, typename TO>
void launch_gini_t(GiniTileArgs a, const T* dX, TO* dout, cudaStream_t st, int64_t max_blocks) {
  if (a.d <= 1024) {
    if (a.tile_end <= a.tile_begin) return;
    const size_t panel = (2 * static_cast<size_t>(a.tile) * a.d * sizeof(T) + 15) & ~static_cast<size_t>(15);
    const size_t smem = panel + static_cast<size_t>(a.nnu) * a.tile * (a.tile + 1) * sizeof(double);
    const int64_t ntiles = a.tile_end - a.tile_begin;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ntiles, max_blocks > 0 ? max_blocks : 1 << 30));
    const gmds_dtype xt = sizeof(T) == 4 ? GMDS_F32 : GMDS_F64;
    const gmds_dtype ot = sizeof(TO) == 4 ? GMDS_F32 : GMDS_F64;
    switch (pick_k(a.d)) {
      case 1: launch_gini_tile<1>(a, dX, xt, dout, ot, smem, blocks, st); break;
      case 2: launch_gini_tile<2>(a, dX, xt, dout, ot, smem, blocks, st); break;
      case 4: launch_gini_tile<4>(a, dX, xt, dout, ot, smem, blocks, st); break;
      case 8: launch_gini_tile<8>(a, dX, xt, dout, ot, smem, blocks, st); break;
      case 16: launch_gini_tile<16>(a, dX, xt, dout, ot, smem, blocks, st); break;
      case 32: launch_gini_tile<32>(a, dX, xt, dout, ot, smem, blocks, st); break;
      default: fail(GMDS_ERROR, "gini: bad K");
    }
    count_launch();
    check_launch("gini_tile_kernel");
    return;
  }
  int n2 = 1;
  while (n2 < a.d) n2 <<= 1;
  const size_t smem = static_cast<size_t>(n2) * sizeof(double);
  const int64_t npairs = a.tile_end - a.tile_begin;
  if (npairs <= 0) return;
  const int64_t blocks = std::min<int64_t>(npairs, 148 * 4);
  DevBuf<double> sk;
  size_t dyn = smem;
  if (smem > 200 * 1024) {
    sk.alloc(static_cast<size_t>(blocks) * n2);
    dyn = 0;
  } else {
    GMDS_CUDA(cudaFuncSetAttribute(gini_block_kernel<T, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  }
  gini_block_kernel<T, TO><<<static_cast<unsigned>(blocks), 256, dyn, st>>>(a, dX, dout, n2, sk.get());
  count_launch();
  check_launch("gini_block_kernel");
  if (sk.get()) GMDS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void launch_midrank(const double* dv, const void* dX, gmds_dtype xt, const int64_t* dpairs, int64_t nseg, int d,
                    double* dranks, cudaStream_t st) {
  if (xt == GMDS_F32)
    launch_midrank_t<float>(dv, static_cast<const float*>(dX), dpairs, nseg, d, dranks, st);
  else
    launch_midrank_t<double>(dv, static_cast<const double*>(dX), dpairs, nseg, d, dranks, st);
}

int gini_tile_size(int d, gmds_dtype xt, int nnu) {
  const size_t sz = dtype_size(xt);
  int tile = 16;
  while (tile > 1 && 2 * static_cast<size_t>(tile) * d * sz + static_cast<size_t>(nnu) * tile * (tile + 1) * 8 >
                         static_cast<size_t>(110) * 1024)
    tile >>= 1;
  return tile;
}

void launch_gini(GiniTileArgs a, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, cudaStream_t st,
                 int64_t max_blocks) {
  if (xt == GMDS_F32 && ot == GMDS_F32)
    launch_gini_t<float, float>(a, static_cast<const float*>(dX), static_cast<float*>(dout), st, max_blocks);
  else if (xt == GMDS_F32)
    launch_gini_t<float, double>(a, static_cast<const float*>(dX), static_cast<double*>(dout), st, max_blocks);
  else if (ot == GMDS_F32)
    launch_gini_t<double, float>(a, static_cast<const double*>(dX), static_cast<float*>(dout), st, max_blocks);
  else
    launch_gini_t<double, double>(a, static_cast<const double*>(dX), static_cast<double*>(dout), st, max_blocks);
}

void launch_euclid(const void* dX, gmds_dtype xt, int64_t n, int d, double* dout, cudaStream_t st) {
  const int64_t npairs = n * (n - 1) / 2;
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(npairs, 256), 148 * 32)));
  if (xt == GMDS_F32)
    euclid_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dX), n, d, dout);
  else
    euclid_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dX), n, d, dout);
  count_launch();
  check_launch("euclid_kernel");
}

void launch_transpose(const void* din, gmds_dtype t, int64_t rows, int64_t cols, void* dout, cudaStream_t st) {
  const dim3 g(static_cast<unsigned>(ceil_div(cols, 32)), static_cast<unsigned>(ceil_div(rows, 32)));
  const dim3 b(32, 8);
  if (t == GMDS_F32)
    transpose_kernel<float><<<g, b, 0, st>>>(static_cast<const float*>(din), rows, cols, static_cast<float*>(dout));
  else
    transpose_kernel<double><<<g, b, 0, st>>>(static_cast<const double*>(din), rows, cols, static_cast<double*>(dout));
  count_launch();
  check_launch("transpose_kernel");
}

}  // namespace gmds
