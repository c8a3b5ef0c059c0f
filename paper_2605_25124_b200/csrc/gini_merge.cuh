// K2 v3: merge-based Gini distance for sparse, non-negative X (images,
// counts, tf-idf -- BASELINE configs 3/5 and the metric config).
//
// Every row's nonzeros are sorted by value once (row store `sidx`).  For a
// pair (i, j) with all x >= 0 the difference vector splits into
//   S_a  = {k : a_k > 0, b_k = 0}   z = a_k  > 0, already ascending in row i's order
//   S_b  = {k : a_k = 0, b_k > 0}   z = -b_k < 0, ascending in row j's REVERSE order
//   S_ab = {k : a_k > 0, b_k > 0}   z = a_k - b_k, any sign -- the only part to sort
//   the rest                        z = 0 (one tie group; only its size matters)
// so the negatives are merge(S_b, sort(S_ab^-)) and the positives
// merge(S_a, sort(S_ab^+)).  Ordered stream compaction (ballot + popc)
// extracts S_a / S_b in order; the small S_ab set is sorted with the split
// network; each half is then ONE bitonic merge (log2 H half-cleaner stages)
// instead of a full sort (log2 H (log2 H + 1) / 2 stages).  Ties and
// midranks are then exactly those of the sorted difference vector, as in
// gini_split.cuh.  Pairs whose halves exceed 256 keys fall back to the
// split path on the same panels.
#pragma once

#include "gini_split.cuh"

namespace gmds {

struct MergeArgs {
  SplitArgs s;
  const uint16_t* sidx;  // per row, its nonzero features sorted by value (rowptr layout)
};

namespace merge_detail {

constexpr int kHalfCap = 256;  // max keys per sign half on the merge path
constexpr int kMCap = 128;     // max |S_ab| on the merge path
constexpr int kAB = kHalfCap + kHalfCap / 16;  // skewed half buffer (doubles)
constexpr int kMB = kMCap + kMCap / 16;
constexpr int kWarpScratch = 2 * kAB + kMB;  // doubles per warp (>= kSplitCap for the fallback)
static_assert(kWarpScratch >= kSplitCap, "fallback scratch");

// skewed index: blocked reads of K consecutive doubles per lane hit distinct banks
__device__ __forceinline__ int sk(int e) { return e + (e >> 4); }

template <typename T>
__device__ __forceinline__ T feat_val(const T* vals, const uint32_t* mask, const uint16_t* pre, int f) {
  const int w = f >> 5, b = f & 31;
  return vals[pre[w] + __popc(mask[w] & ((1u << b) - 1u))];
}

// Sort the unsorted S_ab values (negatives M[0..mneg), positives M[kMCap-1-q])
// with the split network and write them descending into the tails of A / B.
template <int KM>
__device__ __forceinline__ void sort_mids(double* M, int mneg, int mpos, int H, double* A, double* B, int lane) {
  constexpr int Hm = 16 * KM;
  double key[KM];
  const bool hiB = lane >= 16;
  const int l16 = lane & 15;
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int e = r * 16 + l16;
    double v = INFINITY;
    if (!hiB) {
      if (e < mneg) v = M[sk(e)];
    } else {
      if (e < mpos) v = M[sk(kMCap - 1 - e)];
    }
    key[r] = v;
  }
  split_detail::warp_bitonic_upto<KM>(key, lane, Hm);
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int g = lane * KM + r;
    if (g < mneg) A[sk(H - 1 - g)] = key[r];
    else if (g >= Hm && g - Hm < mpos) B[sk(H - 1 - (g - Hm))] = key[r];
  }
}

template <int K>
__device__ __forceinline__ void merge_and_finish(const double* A, const double* B, int cn, int mneg, int cp, int mpos,
                                                 int zeros, int lane, const double* __restrict__ lut, int d, int nnu,
                                                 double half_p, bool store, double* out, size_t ostride, int* flag) {
  constexpr int H = 16 * K;
  double key[K];
  const bool hiB = lane >= 16;
  const int l16 = lane & 15;
  const double* src = hiB ? B : A;
  const int head = hiB ? cp : cn;
  const int tail = H - (hiB ? mpos : mneg);
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int g = l16 * K + r;  // slot within the half
    key[r] = (g < head || g >= tail) ? src[sk(g)] : INFINITY;
  }
  __syncwarp();
  split_detail::warp_bitonic_merge<K>(key, lane);
  split_detail::finish_split<K>(key, cn + mneg, cp + mpos, zeros, lane, lut, d, nnu, half_p, store, out, ostride,
                                flag);
}

}  // namespace merge_detail

// 16 warps per CTA on a tile x tile block of pairs (sparse panels + sorted-order index).
template <typename T, typename TO>
__global__ void __launch_bounds__(512, 1) gini_merge_kernel(MergeArgs ma, const T* __restrict__ X, TO* __restrict__ out) {
  using namespace merge_detail;
  using namespace split_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SplitArgs& sa = ma.s;
  const GiniTileArgs& a = sa.g;
  const int tile = a.tile;
  const int d = a.d;
  const int W = sa.W;
  const int stride = sa.maxnnz;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  double* scratch = reinterpret_cast<double*>(smem_raw) + warp * kWarpScratch;
  double* A = scratch;
  double* B = scratch + kAB;
  double* M = scratch + 2 * kAB;
  double* otile = reinterpret_cast<double*>(smem_raw) + nwarps * kWarpScratch;
  const int tstride = tile + 1;
  unsigned char* pbase = reinterpret_cast<unsigned char*>(otile + static_cast<size_t>(a.nnu) * tile * tstride);
  uint32_t* smask = reinterpret_cast<uint32_t*>(pbase);                       // [2 tile][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + 2 * tile * W);          // [2 tile][W]
  int* scnt = reinterpret_cast<int*>(pbase + ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)));
  T* svals = reinterpret_cast<T*>(scnt + 2 * tile + 4);                        // [2 tile][stride]
  uint16_t* ssidx = reinterpret_cast<uint16_t*>(svals + 2 * static_cast<size_t>(tile) * stride);  // [2 tile][stride]
  const T* gv = static_cast<const T*>(sa.vals);
  const double half_p = 0.5 * static_cast<double>(d);
  const unsigned lt = (1u << lane) - 1u;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    const int64_t i0 = I * tile, j0 = J * tile;
    for (int e = threadIdx.x; e < 2 * tile * W; e += blockDim.x) {
      const int r = e / W, w = e % W;
      const int64_t row = (r < tile) ? i0 + r : j0 + (r - tile);
      smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
      spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
    }
    for (int r = warp; r < 2 * tile; r += nwarps) {
      const int64_t row = (r < tile) ? i0 + r : j0 + (r - tile);
      int cnt = 0;
      if (row < a.n) {
        const int64_t b = sa.rowptr[row], e1 = sa.rowptr[row + 1];
        cnt = static_cast<int>(e1 - b);
        for (int64_t k = b + lane; k < e1; k += 32) {
          svals[static_cast<size_t>(r) * stride + (k - b)] = gv[k];
          ssidx[static_cast<size_t>(r) * stride + (k - b)] = ma.sidx[k];
        }
      }
      if (lane == 0) scnt[r] = cnt;
    }
    __syncthreads();

    const int per_warp = (tile * tile + nwarps - 1) / nwarps;
    for (int it = 0; it < per_warp; ++it) {
      const int k0 = warp + it * nwarps;
      const int kk = (k0 < tile * tile) ? k0 : 0;
      const int r = kk / tile, c = kk % tile;
      const int64_t i = i0 + r, j = j0 + c;
      const bool valid = (k0 < tile * tile) && (j < a.n) && (i < j);
      const int ri = r, rj = valid ? tile + c : r;
      const uint32_t* mi = smask + ri * W;
      const uint32_t* mj = smask + rj * W;
      const uint16_t* pi = spre + ri * W;
      const uint16_t* pj = spre + rj * W;
      const T* vi = svals + static_cast<size_t>(ri) * stride;
      const T* vj = svals + static_cast<size_t>(rj) * stride;
      const uint16_t* si = ssidx + static_cast<size_t>(ri) * stride;
      const uint16_t* sj = ssidx + static_cast<size_t>(rj) * stride;
      const int ci = scnt[ri], cj = scnt[rj];
      double* ot = otile + static_cast<size_t>(r) * tstride + c;
      const size_t ostride = static_cast<size_t>(tile) * tstride;

      // ---- row i in ascending value order: S_a -> B head (ordered), S_ab -> M (unordered)
      int cp = 0, mneg = 0, mpos = 0;
      for (int base = 0; base < ci; base += 32) {
        const int k = base + lane;
        const bool in = k < ci;
        const int f = in ? si[k] : 0;
        const int w = f >> 5, b = f & 31;
        const uint32_t mjw = mj[w];
        const bool inj = in && ((mjw >> b) & 1u);
        const double av = in ? static_cast<double>(vi[pi[w] + __popc(mi[w] & ((1u << b) - 1u))]) : 0.0;
        const unsigned bp = __ballot_sync(kFull, in && !inj);
        if (in && !inj) {
          const int pos = cp + __popc(bp & lt);
          if (pos < kHalfCap) B[sk(pos)] = av;
        }
        cp += __popc(bp);
        double z = 0.0;
        if (inj) z = av - static_cast<double>(vj[pj[w] + __popc(mjw & ((1u << b) - 1u))]);
        const unsigned bn = __ballot_sync(kFull, z < 0.0);
        const unsigned bq = __ballot_sync(kFull, z > 0.0);
        if (z < 0.0) {
          const int pos = mneg + __popc(bn & lt);
          if (pos < kMCap) M[sk(pos)] = z;
        } else if (z > 0.0) {
          const int pos = kMCap - 1 - (mpos + __popc(bq & lt));
          if (pos >= 0) M[sk(pos)] = z;
        }
        mneg += __popc(bn);
        mpos += __popc(bq);
      }
      // ---- row j in descending value order: S_b -> A head as -b (ascending)
      int cn = 0;
      for (int base = 0; base < cj; base += 32) {
        const int q = base + lane;
        const bool in = q < cj;
        const int f = in ? sj[cj - 1 - q] : 0;
        const int w = f >> 5, b = f & 31;
        const bool ini = in && ((mi[w] >> b) & 1u);
        const unsigned bn = __ballot_sync(kFull, in && !ini);
        if (in && !ini) {
          const int pos = cn + __popc(bn & lt);
          if (pos < kHalfCap) A[sk(pos)] = -static_cast<double>(vj[pj[w] + __popc(mj[w] & ((1u << b) - 1u))]);
        }
        cn += __popc(bn);
      }
      const int n_neg = cn + mneg, n_pos = cp + mpos;
      const int zeros = d - n_neg - n_pos;
      const bool fits = n_neg <= kHalfCap && n_pos <= kHalfCap && mneg + mpos <= kMCap;
      __syncwarp();
      if (fits) {
        if (n_neg + n_pos == 0) {
          if (valid && lane == 0)
            for (int v = 0; v < a.nnu; ++v) ot[v * ostride] = 0.0;
        } else {
          const int H = max(16, npow2(max(n_neg, n_pos)));
          if (mneg + mpos > 0) {
            const int Hm = max(16, npow2(max(mneg, mpos)));
            switch (Hm / 16) {
              case 1: sort_mids<1>(M, mneg, mpos, H, A, B, lane); break;
              case 2: sort_mids<2>(M, mneg, mpos, H, A, B, lane); break;
              case 4: sort_mids<4>(M, mneg, mpos, H, A, B, lane); break;
              default: sort_mids<8>(M, mneg, mpos, H, A, B, lane); break;
            }
            __syncwarp();
          }
          switch (H / 16) {
            case 1: merge_and_finish<1>(A, B, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 2: merge_and_finish<2>(A, B, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 4: merge_and_finish<4>(A, B, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 8: merge_and_finish<8>(A, B, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            default: merge_and_finish<16>(A, B, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
          }
        }
      } else {
        // ---- fallback: full split path (z in feature order, compaction, network) on the same panels
        double* scr = scratch;  // kSplitCap doubles
        int nn = 0, np = 0;
        for (int w = 0; w < W; ++w) {
          const uint32_t miw = mi[w], mjw = mj[w];
          double z = 0.0;
          if ((miw >> lane) & 1u) z += static_cast<double>(vi[pi[w] + __popc(miw & lt)]);
          if ((mjw >> lane) & 1u) z -= static_cast<double>(vj[pj[w] + __popc(mjw & lt)]);
          const unsigned bn = __ballot_sync(kFull, z < 0.0);
          const unsigned bq = __ballot_sync(kFull, z > 0.0);
          if (z < 0.0) {
            const int slot = nn + __popc(bn & lt);
            if (slot < kSplitCap) scr[slot] = z;
          } else if (z > 0.0) {
            const int slot = kSplitCap - 1 - (np + __popc(bq & lt));
            if (slot >= 0) scr[slot] = z;
          }
          nn += __popc(bn);
          np += __popc(bq);
        }
        __syncwarp();
        const int nnz = nn + np;
        const int Nf = max(32, npow2(nnz));
        const int Hs = max(16, npow2(max(nn, np)));
        const bool split = net_cost(2 * Hs, Hs) <= net_cost(Nf, Nf);
        const int Nsel = split ? 2 * Hs : Nf;
        if (nnz > kSplitCap || Nsel > 512) {
          if (valid && lane == 0) {
            const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
            if (static_cast<int64_t>(slot) < sa.ovf_cap) {
              sa.ovf_pairs[2 * slot] = i;
              sa.ovf_pairs[2 * slot + 1] = j;
            }
            for (int v = 0; v < a.nnu; ++v) ot[v * ostride] = -1.0;
          }
        } else {
          switch (Nsel / 32) {
            case 1: sort_and_sum<1>(scr, nn, np, d - nnz, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 2: sort_and_sum<2>(scr, nn, np, d - nnz, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 4: sort_and_sum<4>(scr, nn, np, d - nnz, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            case 8: sort_and_sum<8>(scr, nn, np, d - nnz, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            default: sort_and_sum<16>(scr, nn, np, d - nnz, split, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();
    for (int v = 0; v < a.nnu; ++v) {
      const double* otv = otile + static_cast<size_t>(v) * tile * tstride;
      TO* o = out + static_cast<size_t>(v) * a.out_stride;
      if (a.packed) {
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int r = e / tile, c = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = otv[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[packed_offset(i, j, a.nb_packed)] = static_cast<TO>(val);
        }
      } else {
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int r = e / tile, c = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = otv[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[i * a.n + j] = static_cast<TO>(val);
        }
        for (int e = threadIdx.x; e < tile * tile; e += blockDim.x) {
          const int c = e / tile, r = e % tile;
          const int64_t i = i0 + r, j = j0 + c;
          const double val = otv[r * tstride + c];
          if (j < a.n && i < j && val >= 0.0) o[j * a.n + i] = static_cast<TO>(val);
        }
      }
    }
    __syncthreads();
  }
}

inline size_t merge_smem(int tile, int W, int maxnnz, size_t sz, int nnu) {
  return static_cast<size_t>(16) * merge_detail::kWarpScratch * 8 + static_cast<size_t>(nnu) * tile * (tile + 1) * 8 +
         ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)) + (2 * tile + 4) * 4 +
         2 * static_cast<size_t>(tile) * maxnnz * (sz + 2) + 16;
}

void launch_gini_merge(const MergeArgs& ma, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st);

}  // namespace gmds
