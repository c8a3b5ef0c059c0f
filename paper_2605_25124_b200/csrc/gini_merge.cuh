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
  int fast;              // try the rank-by-counting path first (GMDS_MERGE_FAST=1 enables)
  unsigned long long* fast_miss;  // optional: pairs the fast path handed to the merge path
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

// ---------------------------------------------------------------------------
// Rank-by-counting fast path (no merged array at all).
//
// With P = S_a u S_ab+ (the positives) and N = S_b u S_ab- (the negatives),
// the midrank of every element is a COUNT that the pre-sorted rows give
// directly:
//   x in S_a  at position k of row i's sorted list (tie group [g0, g1)):
//     #less  = n_neg + zeros + (g0 - removed_i(g0)) + #{m in S_ab+ : m < x}
//     #equal = (g1 - g0) - (removed_i(g1) - removed_i(g0))
//   -x in S_b at position k of row j's sorted list (tie group [g0, g1)):
//     #less  = #{non-removed row-j entries > x} + #{m in S_ab- : m < -x}
//   m in S_ab+ (index q in sorted S_ab+):
//     #less  = n_neg + zeros + q + #{x in S_a : x < m}
//   m in S_ab- likewise against row j.
// "removed" = the feature is nonzero in both rows (its z is in S_ab);
// removed_i(pos) is a popc prefix over the ballot words of the row-i scan.
// #{m in S_ab+ : m < x_k} = #{q : lb_q <= k} with lb_q = #{row-i values < m_q}
// (no S_ab value equals a row value on this path), so each S_ab element adds
// one count at its row position (a per-warp histogram) and the row pass reads
// it back with a warp scan.  The LUT index of a midrank is 2 #less + #equal
// (gini_tile.cuh).  Only S_ab is sorted (fp64, exact); all counts are exact
// integers, so the ranks are those of the sorted difference vector
// (metrics.cpp:42-56).  The path gives up (returns false, warp-uniform,
// before touching the histogram) -- and the caller runs the merge path --
// when an S_ab value equals another S_ab value or any value of its row, two
// inexact S_ab values share a 32-bit key, or a half of S_ab exceeds kFastCap.
constexpr int kFastCap = 64;   // max |S_ab+|, |S_ab-| on the fast path (16 * KM, KM <= 4)
constexpr int kFastNu = 4;     // nu values per launch on the fast path
constexpr int kRowWords = 8;   // ballot words per row (rows of <= 256 nonzeros)
constexpr int kOffH = kOffRB + kMCap;  // per-warp histograms: 2 rows x 256 u16 counters (128 u32 each)
constexpr int kHistWords = 128;
constexpr int kWarpScratchAll = kOffH + kHistWords;  // doubles per warp, fast path included

struct FastRows {
  const uint32_t* mi;
  const uint32_t* mj;
  const uint16_t* pj;
  const float* vj;
  const uint16_t* si;
  const float* svi;
  const uint16_t* sj;
  const float* svj;
  int ci, cj;
};

__device__ __forceinline__ uint32_t fkey(float v) { return 2u * __float_as_uint(v); }  // exact code of v >= 0

// # of entries of the sorted row (n <= 256) whose code is < t (LE: <= t); branch-free
template <bool LE>
__device__ __forceinline__ int row_bound(const float* sv, int n, uint32_t t) {
  int pos = 0;
#pragma unroll
  for (int step = 256; step > 0; step >>= 1) {
    const int np = pos + step;
    if (np <= n) {
      const uint32_t c = fkey(sv[np - 1]);
      if (LE ? (c <= t) : (c < t)) pos = np;
    }
  }
  return pos;
}
// removed entries before sorted position pos (words rm[], per-word exclusive prefix pre[])
__device__ __forceinline__ int removed_before(const uint32_t* rm, const uint32_t* pre, int pos, int cnt, int total) {
  if (pos >= cnt) return total;
  const int w = pos >> 5;
  return static_cast<int>(pre[w]) + __popc(rm[w] & ((1u << (pos & 31)) - 1u));
}
__device__ __forceinline__ void hist_add(uint32_t* H, int pos) { atomicAdd(H + (pos >> 1), 1u << ((pos & 1) << 4)); }
__device__ __forceinline__ int hist_get(const uint32_t* H, int pos) { return (H[pos >> 1] >> ((pos & 1) << 4)) & 0xFFFF; }

template <int NNU>
struct FastAcc {
  double v[NNU];
  const double* L;  // LUT of nu 0 (nu v at L + v * 2d)
  int stride;       // 2d
  int nnu;
  __device__ __forceinline__ void add(double z, int idx) {
#pragma unroll
    for (int t = 0; t < NNU; ++t)
      if (NNU == 1 || t < nnu) v[t] = fma(z, __ldg(L + t * stride + idx), v[t]);
  }
};

// Sort S_ab (negatives in lanes 0-15, positives in lanes 16-31, KM slots
// each), locate every element in the other row's sorted list, add its term,
// and count it into the histogram at that position.  hpos: the positions
// counted (-1: none), for the clean-up.
template <int KM, int NNU>
__device__ __forceinline__ bool fast_mids(const double* M, int mneg, int mpos, const FastRows& R, const uint32_t* RW,
                                          uint32_t* HI, uint32_t* HJ, int sab, int n_neg, int zeros, int lane,
                                          FastAcc<NNU>& acc, int (&hpos)[4]) {
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
  split_detail::warp_bitonic_upto<KM>(key, lane, 16 * KM);
  const int cnt = hiB ? mpos : mneg;
  uint32_t mag[KM];  // magnitude codes 2 bits(rz|z|) + inexact
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const double a = fabs(key[r]);
    const float f = __double2float_rz(a);
    mag[r] = fkey(f) + ((static_cast<double>(f) != a) ? 1u : 0u);
  }
  bool bad = false;
  const uint32_t mnext0 = __shfl_down_sync(kFull, mag[0], 1);
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;
    const uint32_t mn = (r + 1 < KM) ? mag[r + 1 < KM ? r + 1 : 0] : mnext0;
    if (q + 1 < cnt && mn == mag[r]) bad = true;  // tie or shared key inside the half
  }
  int pos[KM];
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;
    pos[r] = -1;
    if (q >= cnt) continue;
    if (hiB) {  // lb: row i's values below m
      const int lb = row_bound<false>(R.svi, R.ci, mag[r]);
      if (lb < R.ci && fkey(R.svi[lb]) == mag[r]) bad = true;
      pos[r] = lb;
    } else {  // ub: row j's values <= |m|
      const int ub = row_bound<true>(R.svj, R.cj, mag[r]);
      if (ub > 0 && fkey(R.svj[ub - 1]) == mag[r]) bad = true;
      pos[r] = ub;
    }
  }
  if (__any_sync(kFull, bad)) return false;
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    const int q = l16 * KM + r;
    hpos[r] = -1;
    if (q >= cnt) continue;
    int less;
    if (hiB) {
      less = n_neg + zeros + q + pos[r] - removed_before(RW, RW + kRowWords, pos[r], R.ci, sab);
      if (pos[r] < R.ci) {
        hist_add(HI, pos[r]);
        hpos[r] = pos[r];
      }
    } else {
      less = q + (R.cj - pos[r]) - (sab - removed_before(RW + 2 * kRowWords, RW + 3 * kRowWords, pos[r], R.cj, sab));
      if (pos[r] < R.cj) {
        hist_add(HJ, pos[r]);
        hpos[r] = pos[r];
      }
    }
    acc.add(key[r], 2 * less + 1);
  }
  return true;
}

// Terms of the row-only elements of one row: S_a of row i (z = x, base
// n_neg + zeros, S_ab+ below from the histogram) or S_b of row j (z = -x, the
// row's larger entries and S_ab- below).
template <bool ROW_I, int NNU>
__device__ __forceinline__ void fast_row_terms(const float* sv, int c, const uint32_t* rm, const uint32_t* pre,
                                               const uint32_t* H, int sab, int mcnt, int base_less, int lane,
                                               FastAcc<NNU>& acc) {
  const unsigned lt = (1u << lane) - 1u;
  int carry = 0;
  float lastx = -1.f;  // values are >= 0
  for (int base = 0; base < c; base += 32) {
    const int k = base + lane;
    const bool in = k < c;
    const uint32_t rw = rm[base >> 5];
    const int removed = (rw >> lane) & 1u;
    const bool live = in && !removed;
    const float x = in ? sv[k] : -2.f;
    // S_ab below: inclusive scan of the histogram over positions <= k
    int s = in ? hist_get(H, k) : 0;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int o = __shfl_up_sync(kFull, s, dd);
      if (lane >= dd) s += o;
    }
    s += carry;
    carry = __shfl_sync(kFull, s, 31);
    // tie group in the row (neighbours through shuffles; lane 31 reads the next chunk's first)
    float xp = __shfl_up_sync(kFull, x, 1);
    float xn = __shfl_down_sync(kFull, x, 1);
    if (lane == 0) xp = lastx;
    if (lane == 31) xn = (k + 1 < c) ? sv[k + 1] : -3.f;
    lastx = __shfl_sync(kFull, x, 31);
    int g0 = k, g1 = k + 1;
    int rb0 = static_cast<int>(pre[base >> 5]) + __popc(rw & lt);
    int rb1 = rb0 + removed;
    if (live && (xp == x || xn == x)) {
      while (g0 > 0 && sv[g0 - 1] == x) --g0;
      while (g1 < c && sv[g1] == x) ++g1;
      rb0 = removed_before(rm, pre, g0, c, sab);
      rb1 = removed_before(rm, pre, g1, c, sab);
    }
    if (live) {
      const int eq = (g1 - g0) - (rb1 - rb0);
      const int less = ROW_I ? base_less + (g0 - rb0) + s : (c - g1) - (sab - rb1) + (mcnt - s);
      acc.add(ROW_I ? static_cast<double>(x) : -static_cast<double>(x), 2 * less + eq);
    }
  }
}

// The whole pair on the fast path; false (warp-uniform) = not handled.
template <int NNU>
__device__ __forceinline__ bool fast_pair(const FastRows& R, double* scratch, int d, int lane,
                                          const double* __restrict__ lut, int nnu, double half_p, bool store,
                                          double* ot, size_t ostride, int* flag) {
  uint32_t* RW = reinterpret_cast<uint32_t*>(scratch + kOffB);  // rm_i | pre_i | rm_j | pre_j
  uint32_t* HI = reinterpret_cast<uint32_t*>(scratch + kOffH);
  uint32_t* HJ = HI + kHistWords;
  double* M = scratch + kOffM;
  const unsigned lt = (1u << lane) - 1u;
  // ---- row i (ascending): removal words; S_ab values (unordered) into M
  int mneg = 0, mpos = 0, sab = 0;
  for (int base = 0; base < R.ci; base += 32) {
    const int k = base + lane;
    const bool in = k < R.ci;
    const int f = in ? R.si[k] : 0;
    const int w = f >> 5, b = f & 31;
    const uint32_t mjw = R.mj[w];
    const bool inj = in && ((mjw >> b) & 1u);
    const unsigned rm = __ballot_sync(kFull, inj);
    if (lane == 0) {
      RW[base >> 5] = rm;
      RW[kRowWords + (base >> 5)] = static_cast<uint32_t>(sab);
    }
    sab += __popc(rm);
    double z = 0.0;
    if (inj) z = static_cast<double>(R.svi[k]) - static_cast<double>(R.vj[R.pj[w] + __popc(mjw & ((1u << b) - 1u))]);
    const unsigned bn = __ballot_sync(kFull, z < 0.0);
    const unsigned bq = __ballot_sync(kFull, z > 0.0);
    if (z < 0.0) {
      const int p = mneg + __popc(bn & lt);
      if (p < kFastCap) M[sk(p)] = z;
    } else if (z > 0.0) {
      const int p = mpos + __popc(bq & lt);
      if (p < kFastCap) M[sk(kMCap - 1 - p)] = z;
    }
    mneg += __popc(bn);
    mpos += __popc(bq);
  }
  if (mneg > kFastCap || mpos > kFastCap) return false;
  // ---- row j (ascending): removal words only
  int sabj = 0;
  for (int base = 0; base < R.cj; base += 32) {
    const int k = base + lane;
    const bool in = k < R.cj;
    const int f = in ? R.sj[k] : 0;
    const bool ini = in && ((R.mi[f >> 5] >> (f & 31)) & 1u);
    const unsigned rm = __ballot_sync(kFull, ini);
    if (lane == 0) {
      RW[2 * kRowWords + (base >> 5)] = rm;
      RW[3 * kRowWords + (base >> 5)] = static_cast<uint32_t>(sabj);
    }
    sabj += __popc(rm);
  }
  __syncwarp();
  const int n_neg = (R.cj - sab) + mneg, n_pos = (R.ci - sab) + mpos;
  const int zeros = d - n_neg - n_pos;
  FastAcc<NNU> acc;
#pragma unroll
  for (int t = 0; t < NNU; ++t) acc.v[t] = 0.0;
  acc.L = lut;
  acc.stride = 2 * d;
  acc.nnu = nnu;
  int hpos[4] = {-1, -1, -1, -1};
  if (mneg + mpos > 0) {
    const int Hm = max(16, split_detail::npow2(max(mneg, mpos)));
    bool ok;
    switch (Hm / 16) {
      case 1: ok = fast_mids<1, NNU>(M, mneg, mpos, R, RW, HI, HJ, sab, n_neg, zeros, lane, acc, hpos); break;
      case 2: ok = fast_mids<2, NNU>(M, mneg, mpos, R, RW, HI, HJ, sab, n_neg, zeros, lane, acc, hpos); break;
      default: ok = fast_mids<4, NNU>(M, mneg, mpos, R, RW, HI, HJ, sab, n_neg, zeros, lane, acc, hpos); break;
    }
    if (!ok) return false;
    __syncwarp();
  }
  fast_row_terms<true, NNU>(R.svi, R.ci, RW, RW + kRowWords, HI, sab, mpos, n_neg + zeros, lane, acc);
  fast_row_terms<false, NNU>(R.svj, R.cj, RW + 2 * kRowWords, RW + 3 * kRowWords, HJ, sab, mneg, 0, lane, acc);
  __syncwarp();
  const bool hiB = lane >= 16;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (hpos[r] >= 0) (hiB ? HI : HJ)[hpos[r] >> 1] = 0u;  // leave the histograms zero
#pragma unroll
  for (int t = 0; t < NNU; ++t) {
    if (NNU > 1 && t >= nnu) break;
    const double sum = warp_sum(acc.v[t]);
    const double val = clamp_nonneg(half_p * sum);
    if (lane == 0 && store) {
      ot[t * ostride] = val;
      if (isinf(val)) atomicOr(flag, 1);
    }
  }
  return true;
}

}  // namespace merge_detail

// 16 warps per CTA on a tile x tile block of pairs (sparse panels + sorted-order index).
template <typename T, typename TO, bool FAST>
__global__ void __launch_bounds__(merge_detail::kMergeThreads, 1) gini_merge_kernel(MergeArgs ma, const T* __restrict__ X, TO* __restrict__ out) {
  // FAST: the rank-by-counting path is compiled in (its registers would otherwise spill the merge path)
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
  double* scratch = reinterpret_cast<double*>(smem_raw) + warp * kWarpScratchAll;
  uint32_t* A32 = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* B32 = reinterpret_cast<uint32_t*>(scratch + kOffB);
  double* M = scratch + kOffM;
  double* RA = scratch + kOffRA;
  double* RB = scratch + kOffRB;
  double* otile = reinterpret_cast<double*>(smem_raw) + nwarps * kWarpScratchAll;
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
  {  // fast-path histograms start (and are left) zero
    uint32_t* H = reinterpret_cast<uint32_t*>(scratch + kOffH);
    for (int e = lane; e < 2 * kHistWords; e += 32) H[e] = 0u;
  }

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
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

      bool fastdone = false;
      if constexpr (FAST && std::is_same<T, float>::value) {
        if (ma.fast && a.nnu <= kFastNu && ci <= 32 * kRowWords && cj <= 32 * kRowWords) {
          const FastRows R{mi, mj, pj, vj, si, svi, sj, svj, ci, cj};
          fastdone = (a.nnu == 1)
                         ? fast_pair<1>(R, scratch, d, lane, a.lut, 1, half_p, valid, ot, ostride, a.flag)
                         : fast_pair<kFastNu>(R, scratch, d, lane, a.lut, a.nnu, half_p, valid, ot, ostride, a.flag);
          if (!fastdone && ma.fast_miss && valid && lane == 0) atomicAdd(ma.fast_miss, 1ull);
          __syncwarp();
        }
      }
      if (!fastdone) {
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
      }  // !fastdone
      __syncwarp();
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, tile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}

inline size_t merge_smem(int tile, int W, int maxnnz, size_t sz, int nnu) {
  return static_cast<size_t>(merge_detail::kMergeThreads / 32) * merge_detail::kWarpScratchAll * 8 + static_cast<size_t>(nnu) * tile * (tile + 1) * 8 +
         ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)) + (2 * tile + 4) * 4 +
         2 * static_cast<size_t>(tile) * maxnnz * (2 * sz + 2) + 16;
}

void launch_gini_merge(const MergeArgs& ma, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st);

}  // namespace gmds
