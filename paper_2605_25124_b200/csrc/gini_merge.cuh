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
  const void* svs;       // per row, its nonzero values sorted ascending (rowptr layout)
};

namespace merge_detail {

#ifndef GMDS_MERGE_THREADS
#define GMDS_MERGE_THREADS 640
#endif
// 20 warps per CTA, one CTA per SM (96 registers): measured 724 ms per metric
// matrix vs 779 ms at 16 warps (126 registers), 773 / 742 / 761 ms at 18 / 24 / 22
constexpr int kMergeThreads = GMDS_MERGE_THREADS;
constexpr int kHalfCap = 256;  // max keys per sign half on the merge path
constexpr int kMCap = 128;     // max |S_ab| on the merge path
constexpr int kAB32 = 272;     // u32 half buffer (256 keys; 16-byte aligned halves)
constexpr int kMB = kMCap + kMCap / 16;
// per-warp scratch in doubles: A32 | B32 (u32 keys) | M (fp64 S_ab) | RA | RB (residuals)
constexpr int kOffB = kAB32 / 2, kOffM = kAB32, kOffRA = kOffM + kMB, kOffRB = kOffRA + kMCap;
constexpr int kWarpScratch = kOffRB + kMCap;
static_assert(kWarpScratch >= kSplitCap, "fallback scratch");

// skewed indices: blocked reads of K consecutive elements per lane hit distinct banks
__device__ __forceinline__ int sk(int e) { return e + (e >> 4); }  // 8-byte elements
// The u32 key halves are NOT skewed: they are read as 16-byte vectors.
__device__ __forceinline__ int sk32(int e) { return e; }

// Exact 32-bit keys of one sign half.  With f = z rounded toward zero to fp32
// and x = 1 when that rounding was inexact, the magnitude code 2*bits(f) + x
// orders |z| exactly (an inexact |z| lies strictly between f and the next
// float, i.e. between the codes 2*bits(f) and 2*bits(f) + 2).  Positives use
// the code, negatives its complement, so ascending keys = ascending z within
// the half.  Two DIFFERENT inexact values in the same float interval would
// share a key: sort_mids detects that and the pair takes the fp64 path.
__device__ __forceinline__ uint32_t pos_key(float f, bool inexact) { return 2u * __float_as_uint(f) + (inexact ? 1u : 0u); }
__device__ __forceinline__ uint32_t neg_key(float f, bool inexact) { return 0xFFFFFFFFu - pos_key(f, inexact); }

template <typename T>
__device__ __forceinline__ T feat_val(const T* vals, const uint32_t* mask, const uint16_t* pre, int f) {
  const int w = f >> 5, b = f & 31;
  return vals[pre[w] + __popc(mask[w] & ((1u << b) - 1u))];
}

// Sort the unsorted S_ab values (negatives M[0..mneg), positives M[kMCap-1-q])
// exactly in fp64 with the split network, turn them into 32-bit keys written
// descending into the tails of A32 / B32, and store the residual z - (+-f) of
// each inexact one, in ascending-z order, in RA / RB.  Returns true when two
// different values share a key (the pair then takes the fp64 path).
template <int KM>
__device__ __forceinline__ bool sort_mids(const double* M, int mneg, int mpos, int H, uint32_t* A32, uint32_t* B32,
                                          double* RA, double* RB, int lane) {
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
  const int cnt = hiB ? mpos : mneg;
  uint32_t k32[KM];
  bool inex[KM];
  int ninex = 0;
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;  // slot within the half (ascending z)
    const double z = key[r];
    const double mag = fabs(z);
    const float f = __double2float_rz(mag);
    inex[r] = (q < cnt) && (static_cast<double>(f) != mag);
    k32[r] = hiB ? pos_key(f, inex[r]) : neg_key(f, inex[r]);
    ninex += inex[r] ? 1 : 0;
  }
  // collisions: equal key, different value, between adjacent real slots of the half
  bool coll = false;
  const double znext0 = __shfl_down_sync(kFull, key[0], 1);
  const uint32_t knext0 = __shfl_down_sync(kFull, k32[0], 1);
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;
    const double zn = (r + 1 < KM) ? key[r + 1 < KM ? r + 1 : 0] : znext0;
    const uint32_t kn = (r + 1 < KM) ? k32[r + 1 < KM ? r + 1 : 0] : knext0;
    if (q + 1 < cnt && kn == k32[r] && zn != key[r]) coll = true;
  }
  if (__any_sync(kFull, coll)) return true;
  // exclusive prefix of inexact counts within each 16-lane half
  int incl = ninex;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const int o = __shfl_up_sync(kFull, incl, d, 16);
    if (l16 >= d) incl += o;
  }
  int t = incl - ninex;
  double* R = hiB ? RB : RA;
  uint32_t* T32 = hiB ? B32 : A32;
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;
    if (q < cnt) {
      T32[sk32(H - 1 - q)] = k32[r];
      if (inex[r]) {
        const double z = key[r];
        const double f = static_cast<double>(__double2float_rz(fabs(z)));
        R[t++] = hiB ? z - f : z + f;  // exact (Sterbenz)
      }
    }
  }
  return false;
}

// Bitonic merge of 2H = 32K blocked u32 keys (two independent bitonic halves).
template <int K>
__device__ __forceinline__ void warp_merge_u32(uint32_t (&v)[K], int lane) {
  constexpr int H = 16 * K;
#pragma unroll
  for (int t = H / 2; t > 0; t >>= 1) {
    if (t < K) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (!(r & t)) {
          const uint32_t a = v[r], b = v[r + t];
          v[r] = min(a, b);
          v[r + t] = max(a, b);
        }
    } else {
      const int m = t / K;
      const bool keep_lo = !(lane & m);
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const uint32_t o = __shfl_xor_sync(kFull, v[r], m);
        v[r] = keep_lo ? min(v[r], o) : max(v[r], o);
      }
    }
  }
}

// Tie groups of the merged halves (lanes 0-15 negatives, 16-31 positives),
// as warp_tie_groups but with a group start forced at slot H: a negative can
// never tie a positive, even when a full negative half's last code equals the
// positive half's first code numerically.  (A "no ties in this pair" fast
// path was measured slower on the metric data, whose clipped values tie often.)
template <int K>
__device__ __forceinline__ void merge_tie_groups(const uint32_t (&v)[K], int (&h)[K], int lane) {
  const int l16 = lane & 15;
  const uint32_t prev_last = __shfl_up_sync(kFull, v[K - 1], 1);
  int start_pos[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t prev = (r == 0) ? prev_last : v[r - 1];
    const bool st = (r == 0 && l16 == 0) ? true : (v[r] != prev);
    start_pos[r] = st ? (lane * K + r) : -1;
  }
  int run = -1;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    run = max(run, start_pos[r]);
    h[r] = run;
  }
  int carry = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(kFull, carry, d);
    if (lane >= d) carry = max(carry, o);
  }
  int excl = __shfl_up_sync(kFull, carry, 1);
  if (lane == 0) excl = -1;
#pragma unroll
  for (int r = 0; r < K; ++r) h[r] = max(h[r], excl);
  constexpr int N = 32 * K;
  int runb = N;
  int bpos[K];
#pragma unroll
  for (int r = K - 1; r >= 0; --r) {
    bpos[r] = runb;
    runb = min(runb, (start_pos[r] >= 0) ? start_pos[r] : N);
  }
  int carryb = runb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_down_sync(kFull, carryb, d);
    if (lane + d < 32) carryb = min(carryb, o);
  }
  int exclb = __shfl_down_sync(kFull, carryb, 1);
  if (lane == 31) exclb = N;
#pragma unroll
  for (int r = 0; r < K; ++r) h[r] += min(bpos[r], exclb);
}

template <int K>
__device__ __forceinline__ void merge_and_finish(const uint32_t* A32, const uint32_t* B32, const double* RA,
                                                 const double* RB, int cn, int mneg, int cp, int mpos, int zeros,
                                                 int lane, const double* __restrict__ lut, int d, int nnu,
                                                 double half_p, bool store, double* out, size_t ostride, int* flag) {
  constexpr int H = 16 * K;
  uint32_t key[K];
  const bool hiB = lane >= 16;
  const int l16 = lane & 15;
  const uint32_t* src = hiB ? B32 : A32;
  const int head = hiB ? cp : cn;
  const int tail = H - (hiB ? mpos : mneg);
  if constexpr (K >= 4) {
    // blocked 16-byte reads; the gap between the head (compacted row-only
    // keys) and the tail (sorted S_ab keys) is replaced by the pad key through
    // a per-lane slot mask
    const int lo = min(max(head - l16 * K, 0), K), hi = min(max(tail - l16 * K, 0), K);
    const uint32_t gapm = (hi > lo) ? (((K >= 32 ? 0u : (1u << hi)) - 1u) & ~((1u << lo) - 1u)) : 0u;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + l16 * K);
#pragma unroll
    for (int m = 0; m < K / 4; ++m) {
      const uint4 v = s4[m];
      key[4 * m] = ((gapm >> (4 * m)) & 1u) ? 0xFFFFFFFFu : v.x;
      key[4 * m + 1] = ((gapm >> (4 * m + 1)) & 1u) ? 0xFFFFFFFFu : v.y;
      key[4 * m + 2] = ((gapm >> (4 * m + 2)) & 1u) ? 0xFFFFFFFFu : v.z;
      key[4 * m + 3] = ((gapm >> (4 * m + 3)) & 1u) ? 0xFFFFFFFFu : v.w;
    }
  } else {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int g = l16 * K + r;  // slot within the half
      key[r] = (g < head || g >= tail) ? src[g] : 0xFFFFFFFFu;
    }
  }
  __syncwarp();
  warp_merge_u32<K>(key, lane);
  int h[K];
  const int n_neg = cn + mneg, n_pos = cp + mpos;
  merge_tie_groups<K>(key, h, lane);
  // values: +-f from the key (negatives: complemented code, sign bit set), plus
  // the residual of inexact (odd-code) S_ab keys; per-lane constants hoisted
  const uint32_t flip = hiB ? 0u : 0xFFFFFFFFu;
  const uint32_t sgn = hiB ? 0u : 0x80000000u;
  const int lim = (hiB ? n_pos : n_neg) - l16 * K;  // slot r is real iff r < lim
  const int hadd = hiB ? 2 * (n_neg + zeros) - 2 * H : 0;
  uint32_t oddm = 0;  // bit r: real slot with an inexact (odd) code
  double z[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t code = key[r] ^ flip;
    z[r] = static_cast<double>(__uint_as_float((code >> 1) | sgn));
    const bool real = r < lim;
    h[r] = real ? h[r] + hadd : -1;
    oddm |= (real ? (code & 1u) : 0u) << r;
  }
  const int nodd = __popc(oddm);
  int incl = nodd;
#pragma unroll
  for (int dd = 1; dd < 16; dd <<= 1) {
    const int o = __shfl_up_sync(kFull, incl, dd, 16);
    if (l16 >= dd) incl += o;
  }
  const int t0 = incl - nodd;
  const double* R = hiB ? RB : RA;
#pragma unroll
  for (int r = 0; r < K; ++r)
    if ((oddm >> r) & 1u) z[r] += R[t0 + __popc(oddm & ((1u << r) - 1u))];
  for (int v = 0; v < nnu; ++v) {
    const double* L = lut + static_cast<size_t>(v) * 2 * d;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (h[r] >= 0) acc = fma(z[r], __ldg(L + h[r]), acc);
    acc = warp_sum(acc);
    const double val = clamp_nonneg(half_p * acc);
    if (lane == 0 && store) {
      out[v * ostride] = val;
      if (isinf(val)) atomicOr(flag, 1);
    }
  }
}

}  // namespace merge_detail

// 16 warps per CTA on a tile x tile block of pairs (sparse panels + sorted-order index).
template <typename T, typename TO>
__global__ void __launch_bounds__(merge_detail::kMergeThreads, 1) gini_merge_kernel(MergeArgs ma, const T* __restrict__ X, TO* __restrict__ out) {
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
  uint32_t* A32 = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* B32 = reinterpret_cast<uint32_t*>(scratch + kOffB);
  double* M = scratch + kOffM;
  double* RA = scratch + kOffRA;
  double* RB = scratch + kOffRB;
  double* otile = reinterpret_cast<double*>(smem_raw) + nwarps * kWarpScratch;
  const int tstride = tile + 1;
  unsigned char* pbase = reinterpret_cast<unsigned char*>(otile + static_cast<size_t>(a.nnu) * tile * tstride);
  uint32_t* smask = reinterpret_cast<uint32_t*>(pbase);                       // [2 tile][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + 2 * tile * W);          // [2 tile][W]
  int* scnt = reinterpret_cast<int*>(pbase + ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)));
  T* svals = reinterpret_cast<T*>(scnt + 2 * tile + 4);                        // [2 tile][stride]
  T* ssv = svals + 2 * static_cast<size_t>(tile) * stride;                        // [2 tile][stride] sorted values
  uint16_t* ssidx = reinterpret_cast<uint16_t*>(ssv + 2 * static_cast<size_t>(tile) * stride);  // [2 tile][stride]
  const T* gsv = static_cast<const T*>(ma.svs);
  const T* gv = static_cast<const T*>(sa.vals);
  const double half_p = 0.5 * static_cast<double>(d);
  const unsigned lt = (1u << lane) - 1u;
  __shared__ double s_score[2 * kMaxScoreNu];
  __shared__ double s_red[32 * 8];
  for (int e = threadIdx.x; e < 2 * kMaxScoreNu; e += blockDim.x) s_score[e] = 0.0;

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
          ssv[static_cast<size_t>(r) * stride + (k - b)] = gsv[k];
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
      const T* svi = ssv + static_cast<size_t>(ri) * stride;
      const T* svj = ssv + static_cast<size_t>(rj) * stride;
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
        const T avt = in ? svi[k] : T(0);  // row i's k-th smallest nonzero (no feature-order gather)
        const double av = static_cast<double>(avt);
        const unsigned bp = __ballot_sync(kFull, in && !inj);
        if (in && !inj) {
          const int pos = cp + __popc(bp & lt);
          if (pos < kHalfCap) B32[sk32(pos)] = pos_key(static_cast<float>(avt), false);
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
          if (pos < kHalfCap)
            A32[sk32(pos)] = neg_key(static_cast<float>(svj[cj - 1 - q]), false);
        }
        cn += __popc(bn);
      }
      const int n_neg = cn + mneg, n_pos = cp + mpos;
      const int zeros = d - n_neg - n_pos;
      const bool fits = n_neg <= kHalfCap && n_pos <= kHalfCap && mneg + mpos <= kMCap;
      __syncwarp();
      bool done = false;
      if (fits) {
        if (n_neg + n_pos == 0) {
          if (valid && lane == 0)
            for (int v = 0; v < a.nnu; ++v) ot[v * ostride] = 0.0;
          done = true;
        } else {
          const int H = max(16, npow2(max(n_neg, n_pos)));
          bool coll = false;
          if (mneg + mpos > 0) {
            const int Hm = max(16, npow2(max(mneg, mpos)));
            switch (Hm / 16) {
              case 1: coll = sort_mids<1>(M, mneg, mpos, H, A32, B32, RA, RB, lane); break;
              case 2: coll = sort_mids<2>(M, mneg, mpos, H, A32, B32, RA, RB, lane); break;
              case 4: coll = sort_mids<4>(M, mneg, mpos, H, A32, B32, RA, RB, lane); break;
              default: coll = sort_mids<8>(M, mneg, mpos, H, A32, B32, RA, RB, lane); break;
            }
            __syncwarp();
          }
          if (!coll) {
            switch (H / 16) {
              case 1: merge_and_finish<1>(A32, B32, RA, RB, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
              case 2: merge_and_finish<2>(A32, B32, RA, RB, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
              case 4: merge_and_finish<4>(A32, B32, RA, RB, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
              case 8: merge_and_finish<8>(A32, B32, RA, RB, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
              default: merge_and_finish<16>(A32, B32, RA, RB, cn, mneg, cp, mpos, zeros, lane, a.lut, d, a.nnu, half_p, valid, ot, ostride, a.flag); break;
            }
            done = true;
          }
        }
      }
      if (!done) {
        __syncwarp();
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
    tile_epilogue<TO>(a, otile, tile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}

inline size_t merge_smem(int tile, int W, int maxnnz, size_t sz, int nnu) {
  return static_cast<size_t>(merge_detail::kMergeThreads / 32) * merge_detail::kWarpScratch * 8 + static_cast<size_t>(nnu) * tile * (tile + 1) * 8 +
         ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)) + (2 * tile + 4) * 4 +
         2 * static_cast<size_t>(tile) * maxnnz * (2 * sz + 2) + 16;
}

void launch_gini_merge(const MergeArgs& ma, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st);

}  // namespace gmds
