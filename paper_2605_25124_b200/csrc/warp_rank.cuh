// Warp-level exact midrank machinery (sm_100a).
//
// One warp owns one segment of length p <= N = 32*K (a pair's difference
// vector z = x_i - x_j, or a caller vector for the public midrank API).
// Keys live in registers: lane L holds slots g = L*K + r, r < K ("blocked").
// The segment is loaded "striped" (slot (L, r) <- element r*32 + L) so the
// shared-memory loads are conflict-free; a sort does not care where keys
// start.  Padding slots hold +inf, which sorts after every finite key and
// forms its own tie group, so real groups are unaffected.
//
// Sort: bitonic network in its direction-free form (first stage of every
// merge compares g with g ^ (s-1), the rest compare g with g ^ t), so every
// compare-exchange is "ascending".  Intra-lane stages are register CEs;
// stages whose partner lives in another lane use __shfl_xor_sync.
//
// Ties follow midrank_into (metrics.cpp:42-56) exactly: keys are the fp64
// values themselves compared with '<' / '==', so -0.0 and +0.0 form one
// group, and a tie group occupying sorted 0-based slots [a, b) has midrank
// (a + 1 + b) / 2, i.e. 2R - 1 = a + b.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gmds {

constexpr unsigned kFull = 0xffffffffu;

// c ? a : b as two 32-bit selects.  (ptxas compiled the fp64 `?:` of the cross-lane sort steps
// into BRA / MOV / BSYNC triples -- 36% of gini_split_kernel's warp instructions at the C4 shape,
// profiles/r2b_split_c4_lines_n4000.txt; the halves select as SEL.)
__device__ __forceinline__ double sel64(bool c, double a, double b) {
  return __hiloint2double(c ? __double2hiint(a) : __double2hiint(b), c ? __double2loint(a) : __double2loint(b));
}

// Compare-exchange, ascending (lower slot keeps the smaller key).
__device__ __forceinline__ void ce_asc(double& a, double& b) {
  const bool sw = b < a;
  const double lo = sel64(sw, b, a);
  const double hi = sel64(sw, a, b);
  a = lo;
  b = hi;
}

template <bool kPayload>
struct Payload;
template <>
struct Payload<false> {
  template <int K>
  struct Arr {
    __device__ __forceinline__ int& operator[](int) { return dummy; }
    int dummy;
  };
};
template <>
struct Payload<true> {
  template <int K>
  struct Arr {
    __device__ __forceinline__ int& operator[](int r) { return v[r]; }
    int v[K];
  };
};

template <int K, bool kPayload>
__device__ __forceinline__ void ce_asc_p(double (&v)[K], typename Payload<kPayload>::template Arr<K>& idx, int r1,
                                         int r2) {
  const bool sw = v[r2] < v[r1];
  const double a = v[r1], b = v[r2];
  v[r1] = sel64(sw, b, a);
  v[r2] = sel64(sw, a, b);
  if constexpr (kPayload) {
    const int ia = idx[r1], ib = idx[r2];
    idx[r1] = sw ? ib : ia;
    idx[r2] = sw ? ia : ib;
  }
}

// Cross-lane exchange step: this lane's slot holds `a`, the partner's `o`;
// keep the min if `keep_lo`, else the max.
template <bool kPayload>
__device__ __forceinline__ void xchg(double& a, double o, int& ia, int io, bool keep_lo) {
  const bool lt = o < a, gt = a < o;
  const bool take = keep_lo ? lt : gt;
  a = sel64(take, o, a);
  if constexpr (kPayload) ia = take ? io : ia;
}

// Full bitonic sort of N = 32*K keys held blocked across the warp.
template <int K, bool kPayload>
__device__ __forceinline__ void warp_bitonic_sort(double (&v)[K], typename Payload<kPayload>::template Arr<K>& idx,
                                                  int lane) {
  constexpr int N = 32 * K;
#pragma unroll
  for (int s = 2; s <= N; s <<= 1) {
    // --- mirror stage: partner g ^ (s-1)
    if (s <= K) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const int r2 = r ^ (s - 1);
        if (r < r2) ce_asc_p<K, kPayload>(v, idx, r, r2);
      }
    } else {
      const int m = s / K - 1;               // partner lane mask
      const bool keep_lo = !(lane & (s / (2 * K)));
#pragma unroll
      for (int r = 0; r < (K + 1) / 2; ++r) {
        const int r2 = K - 1 - r;
        const double o1 = __shfl_xor_sync(kFull, v[r2], m);
        int i1 = 0, i2 = 0;
        if constexpr (kPayload) i1 = __shfl_xor_sync(kFull, idx[r2], m);
        if (r2 != r) {
          const double o2 = __shfl_xor_sync(kFull, v[r], m);
          if constexpr (kPayload) i2 = __shfl_xor_sync(kFull, idx[r], m);
          xchg<kPayload>(v[r2], o2, idx[r2], i2, keep_lo);
        }
        xchg<kPayload>(v[r], o1, idx[r], i1, keep_lo);
      }
    }
    // --- half-cleaners: partner g ^ t
#pragma unroll
    for (int t = s / 4; t > 0; t >>= 1) {
      if (t < K) {
#pragma unroll
        for (int r = 0; r < K; ++r)
          if (!(r & t)) ce_asc_p<K, kPayload>(v, idx, r, r + t);
      } else {
        const int m = t / K;
        const bool keep_lo = !(lane & m);
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const double o = __shfl_xor_sync(kFull, v[r], m);
          int io = 0;
          if constexpr (kPayload) io = __shfl_xor_sync(kFull, idx[r], m);
          xchg<kPayload>(v[r], o, idx[r], io, keep_lo);
        }
      }
    }
  }
}

// After a sort: for every slot, h = a + b where [a, b) is its tie group
// (0-based, b exclusive).  Midrank R = (h + 1) / 2.
template <int K, typename KT>
__device__ __forceinline__ void warp_tie_groups(const KT (&v)[K], int (&h)[K], int lane) {
  // group starts: slot g starts a group iff g == 0 or v[g] != v[g-1]
  const KT prev_last = __shfl_up_sync(kFull, v[K - 1], 1);
  int start_pos[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const KT prev = (r == 0) ? prev_last : v[r - 1];
    const bool st = (r == 0 && lane == 0) ? true : (v[r] != prev);
    start_pos[r] = st ? (lane * K + r) : -1;
  }
  // a(g): inclusive max-scan of start positions (forward)
  int run = -1;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    run = max(run, start_pos[r]);
    h[r] = run;
  }
  int carry = run;  // lane total
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(kFull, carry, d);
    if (lane >= d) carry = max(carry, o);
  }
  int excl = __shfl_up_sync(kFull, carry, 1);
  if (lane == 0) excl = -1;
#pragma unroll
  for (int r = 0; r < K; ++r) h[r] = max(h[r], excl);
  // b(g): min over g' > g of start positions (suffix), default 32*K
  constexpr int N = 32 * K;
  int nxt[K];
#pragma unroll
  for (int r = 0; r < K; ++r) nxt[r] = (start_pos[r] >= 0) ? start_pos[r] : N;
  int runb = N;
  int bpos[K];
#pragma unroll
  for (int r = K - 1; r >= 0; --r) {
    bpos[r] = runb;  // min over slots strictly after r within the lane
    runb = min(runb, nxt[r]);
  }
  int carryb = runb;  // lane's min start position
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

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}

}  // namespace gmds
