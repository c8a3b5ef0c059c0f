// K2 linear-weight kernel: the Gini distance matrix at nu = 2 / nu = 3 for
// sparse non-negative fp32 X (the metric config, C3, C5) without ranking any
// element individually.
//
// For e = nu - 1 in {1, 2} the weight is affine in the midrank:
//   G(R) = ((R-1/2)/p)^e - (1-(R-1/2)/p)^e = (2R - 1 - p)/p,
// so D = (p/2) sum_k z_k G(R_k) (metrics.cpp:69-82, 157-163) becomes
//   D = sum_k z_k R_k - h sum_k z_k,   h = (p+1)/2,
// and for any multiset S with midranks r, sum_S z r = sum_S z + PM(S), where
// PM(S) = sum over unordered pairs of their maximum (exact with ties).  With
// z split into negatives N = S_b u S_ab-, zeros, and positives P = S_a u S_ab+
// (gini_merge.cuh for the sets):
//   D = (1 - h) sum_N z + (1 + |N| + zeros - h) sum_P z + PM(N) + PM(P).
// PM(P) = PM(row i) - [pairs touching F] + PM(S_ab+) + X(S_a, S_ab+), where F
// = the features nonzero in both rows (|F| = s ~ 31 at the metric shape) --
// and likewise for N with minima of row j.  Every term is a per-row constant
// (s1 = sum of values, tm = PM of the row, suffix sums of its sorted values,
// from row_sort_kernel) corrected by O(s) quantities:
//   * F's values and sorted positions in both rows (pmap),
//   * F's position-order ranks in each row (popc prefix of a position mask)
//     and prefix sums of F's values in that order,
//   * per S_ab value: its lower bound in the other row's sorted values
//     (branch-free binary search), and
//   * PM(S_ab+) + PM(S_ab-) = PM(Z) - (|S_ab-| + |Z0|) sum(S_ab+), with Z the
//     s values of z on F and PM(Z) = (s-1)/2 sum z + 1/2 sum_{f<g} |z_f - z_g|
//     (each lane sums its values against the next half of F, circularly).
// Nothing is O(nnz) per pair.  All sums are fp64 from exact fp32 inputs; the
// reference's pow-based weights agree to round-off (tests: <= 1e-12
// max-normalised vs the compiled reference).  Pairs with s > 64 or a row with
// more nonzeros than the panel stride (<= 256, sized to shared memory) go to
// the overflow list (exact full-sort kernel).
#pragma once

#include <cstdio>

#include "gini_split.cuh"

namespace gmds {

struct GmdArgs {
  SplitArgs s;           // tile args, row store (masks, prefix, rowptr, vals), overflow list
  const uint16_t* pmap;  // sorted position of each nonzero (feature order)
  const float* svs;      // sorted values per row
  const double* suf;     // suffix sums of the sorted values per row
  const double* s1;      // per row: sum of values
  const double* tm;      // per row: sum_k v_(k) k
  const uint32_t* tiew;  // per row, 8 words: bit g = (v_(g) == v_(g+1)) (general kernel's tie groups)
  const uint8_t* bkt;    // per row, 256 bytes: bkt[b] = #{sorted values in a bucket below b} (gini_gmd2_kernel)
  const float* bscale;   // per row: bucket(v) = min(255, int(v * bscale)), bscale = 256 / (the row's largest value)
};

namespace gmd_detail {

constexpr int kTile = 32;
constexpr int kRows = 2 * kTile;
constexpr int kCap = 64;      // max |F| per pair
constexpr int kMaxC = 256;    // max nonzeros per row
// per-warp scratch (8-byte words): F[64] ints (32) | QM[32] u32 (16) | PQi[72] | PQj[72] | BL[2][64]
constexpr int kOffQM = 32, kOffPQi = 48, kOffPQj = 120, kOffBL = 192;
constexpr int kWarpWords = kOffBL + 2 * kCap;

__device__ __forceinline__ uint32_t fkey(float v) { return 2u * __float_as_uint(v); }

// #{entries of the sorted row (n <= 256) with code < t}; branch-free
__device__ __forceinline__ int lower_count(const float* sv, int n, uint32_t t) {
  int pos = 0;
#pragma unroll
  for (int step = 128; step > 0; step >>= 1) {
    const int idx = pos + step - 1;
    const bool go = (idx < n) && (fkey(sv[idx]) < t);  // idx <= 254: inside shared memory even past n
    pos += go ? step : 0;
  }
  // the ninth probe (n = 256): position 255
  if (pos == 255 && n == 256 && fkey(sv[255]) < t) pos = 256;
  return pos;
}

// the same on a row of precomputed codes (the linear kernel stages codes, not values)
__device__ __forceinline__ int lower_count_codes(const uint32_t* sc, int n, uint32_t t) {
  int pos = 0;
#pragma unroll
  for (int step = 128; step > 0; step >>= 1) {
    const int idx = pos + step - 1;
    pos += ((idx < n) && (sc[idx] < t)) ? step : 0;  // idx <= 254: inside shared memory even past n
  }
  if (pos == 255 && n == 256 && sc[255] < t) pos = 256;
  return pos;
}

// #{F positions < pos} from a position mask QM[8] and its word prefix QP[8]
__device__ __forceinline__ int qcount(const uint32_t* QM, const uint32_t* QP, int pos, int s) {
  if (pos >= kMaxC) return s;
  const int w = pos >> 5;
  return static_cast<int>(QP[w]) + __popc(QM[w] & ((1u << (pos & 31)) - 1u));
}

// the same without the sentinel test, for callers whose positions are < kMaxC whenever the result
// is used (gini_gmd2_kernel: rows of <= 255 nonzeros; dead lanes pass kMaxC and ignore the result)
__device__ __forceinline__ int qcount2(const uint32_t* QM, const uint32_t* QP, int pos) {
  const int w = (pos >> 5) & 7;
  return static_cast<int>(QP[w]) + __popc(QM[w] & ((1u << (pos & 31)) - 1u));
}

// per-warp histograms of u16 counters packed two per u32 word
__device__ __forceinline__ void hist_add(uint32_t* H, int pos) { atomicAdd(H + (pos >> 1), 1u << ((pos & 1) << 4)); }
__device__ __forceinline__ int hist_get(const uint32_t* H, int pos) { return (H[pos >> 1] >> ((pos & 1) << 4)) & 0xFFFF; }

__device__ __forceinline__ double warp_incl(double v, int lane) {
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const double o = __shfl_up_sync(0xffffffffu, v, dd);
    if (lane >= dd) v += o;
  }
  return v;
}

}  // namespace gmd_detail

template <typename TO, int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) gini_gmd_kernel(GmdArgs ga, TO* __restrict__ out) {
  using namespace gmd_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SplitArgs& sa = ga.s;
  const GiniTileArgs& a = sa.g;
  const int d = a.d;
  const int W = sa.W;
  const int stride = sa.maxnnz;  // panel stride (<= kMaxC): rows with more nonzeros overflow
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // ---- shared memory
  double* wscr = reinterpret_cast<double*>(smem_raw) + warp * kWarpWords;
  int* F = reinterpret_cast<int*>(wscr);
  uint32_t* QM = reinterpret_cast<uint32_t*>(wscr + kOffQM);  // qm_i[8] qm_j[8] qp_i[8] qp_j[8]
  double* PQi = wscr + kOffPQi;
  double* PQj = wscr + kOffPQj;
  double* ZL = wscr + kOffBL;  // z on F, stored twice (F order): circular reads without a wrap
  double* otile = reinterpret_cast<double*>(smem_raw) + kWarps * kWarpWords;  // [nnu][32][33]
  double* rs1 = otile + static_cast<size_t>(a.nnu) * kTile * (kTile + 1);
  double* rtm = rs1 + kRows;
  int64_t* rbase = reinterpret_cast<int64_t*>(rtm + kRows);
  int* rcnt = reinterpret_cast<int*>(rbase + kRows);
  uint32_t* smask = reinterpret_cast<uint32_t*>(rcnt + kRows);  // [64][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + kRows * W);
  float* svals = reinterpret_cast<float*>(spre + ((kRows * W + 1) & ~1));  // [64][stride]
  uint32_t* ssc = reinterpret_cast<uint32_t*>(svals + kRows * stride);     // [64][stride] sorted value codes
  uint16_t* spm = reinterpret_cast<uint16_t*>(ssc + kRows * stride);         // [64][stride]
  const float* gv = static_cast<const float*>(sa.vals);
  const double h = 0.5 * static_cast<double>(d + 1);
  const int tstride = kTile + 1;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * kTile, j0 = J * kTile;
    for (int e = threadIdx.x; e < kRows * W; e += blockDim.x) {
      const int r = e / W, w = e - (e / W) * W;
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
      spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
    }
    for (int r = warp; r < kRows; r += kWarps) {
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      int cnt = 0;
      int64_t b = 0;
      if (row < a.n) {
        b = sa.rowptr[row];
        cnt = static_cast<int>(sa.rowptr[row + 1] - b);
        for (int k = lane; k < cnt && k < stride; k += 32) {
          svals[r * stride + k] = gv[b + k];
          ssc[r * stride + k] = fkey(ga.svs[b + k]);
          spm[r * stride + k] = ga.pmap[b + k];
        }
      }
      if (lane == 0) {
        rcnt[r] = cnt;
        rbase[r] = b;
        rs1[r] = (row < a.n) ? ga.s1[row] : 0.0;
        rtm[r] = (row < a.n) ? ga.tm[row] : 0.0;
      }
    }
    __syncthreads();

    for (int k0 = warp; k0 < kTile * kTile; k0 += kWarps) {
      const int r = k0 >> 5, c = k0 & 31;
      const int64_t gi = i0 + r, gj = j0 + c;
      if (!(gj < a.n && gi < gj)) continue;
      const int ri = r, rj = kTile + c;
      const int ci = rcnt[ri], cj = rcnt[rj];
      const uint32_t* mi = smask + ri * W;
      const uint32_t* mj = smask + rj * W;
      double* ot = otile + r * tstride + c;
      // ---- F = features nonzero in both rows, in feature order
      if (lane < 16) QM[lane] = 0u;
      uint32_t m = (lane < W) ? (mi[lane] & mj[lane]) : 0u;
      const int cm = __popc(m);
      int incl = cm;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, dd);
        if (lane >= dd) incl += o;
      }
      const int s = __shfl_sync(0xffffffffu, incl, 31);
      if (s > kCap || ci > stride || cj > stride) {  // overflow list: the exact full-sort kernel
        if (lane == 0) {
          const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
          if (static_cast<int64_t>(slot) < sa.ovf_cap) {
            sa.ovf_pairs[2 * slot] = gi;
            sa.ovf_pairs[2 * slot + 1] = gj;
          }
          for (int v = 0; v < a.nnu; ++v) ot[v * kTile * tstride] = -1.0;
        }
        continue;
      }
      {
        int off = incl - cm;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1u;
          F[off++] = (lane << 5) | b;
        }
      }
      __syncwarp();
      const uint16_t* pim = spre + ri * W;
      const uint16_t* pjm = spre + rj * W;
      const float* vi = svals + ri * stride;
      const float* vj = svals + rj * stride;
      const uint16_t* pmi = spm + ri * stride;
      const uint16_t* pmj = spm + rj * stride;
      // ---- F's values and sorted positions in both rows; position masks
      float al[2], be[2];
      int pI[2], pJ[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = lane + 32 * u;
        al[u] = be[u] = 0.f;
        pI[u] = pJ[u] = kMaxC;  // sentinel: qcount -> s, never stored
        if (u == 1 && s <= 32) break;  // warp-uniform: the second element slot is empty
        if (e < s) {
          const int f = F[e];
          const int w = f >> 5;
          const uint32_t lo = (1u << (f & 31)) - 1u;
          const int ii = pim[w] + __popc(mi[w] & lo);
          const int jj = pjm[w] + __popc(mj[w] & lo);
          al[u] = vi[ii];
          be[u] = vj[jj];
          pI[u] = pmi[ii];
          pJ[u] = pmj[jj];
          atomicOr(QM + (pI[u] >> 5), 1u << (pI[u] & 31));
          atomicOr(QM + 8 + (pJ[u] >> 5), 1u << (pJ[u] & 31));
        }
      }
      __syncwarp();
      {  // word prefixes of the two masks (groups of 8 lanes)
        const uint32_t wv = (lane < 16) ? QM[lane] : 0u;
        const int pc = __popc(wv);
        int x = pc;
#pragma unroll
        for (int dd = 1; dd < 8; dd <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, x, dd, 8);
          if ((lane & 7) >= dd) x += o;
        }
        if (lane < 16) QM[16 + lane] = static_cast<uint32_t>(x - pc);
      }
      __syncwarp();
      // ---- position-order ranks; F's values scattered in that order
      int rI[2], rJ[2];
      double z[2];
      int mneg = 0, mpos = 0;
      z[1] = 0.0;
      rI[1] = rJ[1] = s;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && s <= 32) break;  // warp-uniform
        rI[u] = qcount(QM, QM + 16, pI[u], s);
        rJ[u] = qcount(QM + 8, QM + 24, pJ[u], s);
        const bool live = lane + 32 * u < s;
        if (live) {
          PQi[1 + rI[u]] = static_cast<double>(al[u]);
          PQj[1 + rJ[u]] = static_cast<double>(be[u]);
        }
        z[u] = static_cast<double>(al[u]) - static_cast<double>(be[u]);
        if (live) {
          ZL[lane + 32 * u] = z[u];
          ZL[lane + 32 * u + s] = z[u];
        }
        mneg += __popc(__ballot_sync(0xffffffffu, z[u] < 0.0));
        mpos += __popc(__ballot_sync(0xffffffffu, z[u] > 0.0));
      }
      __syncwarp();
      {  // prefix sums PQ[k] = sum of the first k values in position order
        const int t0 = 1 + 2 * lane, t1 = t0 + 1;
        const double a0 = (t0 <= s) ? PQi[t0] : 0.0, a1 = (t1 <= s) ? PQi[t1] : 0.0;
        const double b0 = (t0 <= s) ? PQj[t0] : 0.0, b1 = (t1 <= s) ? PQj[t1] : 0.0;
        const double ea = warp_incl(a0 + a1, lane) - (a0 + a1);
        const double eb = warp_incl(b0 + b1, lane) - (b0 + b1);
        __syncwarp();
        if (t0 <= s) {
          PQi[t0] = ea + a0;
          PQj[t0] = eb + b0;
        }
        if (t1 <= s) {
          PQi[t1] = ea + a0 + a1;
          PQj[t1] = eb + b0 + b1;
        }
        if (lane == 0) {
          PQi[0] = 0.0;
          PQj[0] = 0.0;
        }
      }
      __syncwarp();
      const int nP = ci - s + mpos, nN = cj - s + mneg;
      const double kp = static_cast<double>(1 + nN + (d - nP - nN)) - h, kn = 1.0 - h;
      const double* sufi = ga.suf + rbase[ri];
      const double* sufj = ga.suf + rbase[rj];
      const double s1j = rs1[rj];
      double acc = 0.0;
      if (lane == 0) acc = kp * rs1[ri] - kn * s1j + rtm[ri] - (static_cast<double>(cj - 1) * s1j - rtm[rj]);
      const double sumQi = PQi[s];
      // PM(S_ab+) + PM(S_ab-) = PM(Z) - (|S_ab-| + |Z0|) sum(S_ab+), Z = all s values of
      // z on F; PM(Z) = (s-1)/2 sum z + 1/2 sum over unordered pairs |z_f - z_g|
      // (each lane: its values against the next floor((s-1)/2) in circular order,
      // plus half of the opposite one when s is even: every pair exactly once)
      const double wneg = static_cast<double>(s - mpos);  // |S_ab-| + |Z0|
      const int half = (s - 1) >> 1;
      const bool even = (s & 1) == 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && s <= 32) break;  // warp-uniform
        const int e = lane + 32 * u;
        if (e >= s) continue;
        const double av = al[u], bv = be[u];
        // pairs of row i touching F (PM(S_a)) and of row j (minima, PM(S_b))
        const double si1 = (pI[u] + 1 < ci) ? __ldg(sufi + pI[u] + 1) : 0.0;
        const double sj0 = __ldg(sufj + pJ[u]);
        acc += av * static_cast<double>(rI[u] - pI[u]) - si1 - kp * av;
        acc += (s1j - sj0) + bv * static_cast<double>((cj - 1 - pJ[u]) - (s - 1 - rJ[u])) + kn * bv;
        const double zz = z[u];
        // PM(Z) pieces
        double g0 = 0.0, g1 = 0.0;  // two chains: DADD latency
        const double* zr = ZL + e + 1;
        int t = 0;
        for (; t + 1 < half; t += 2) {
          g0 += fabs(zz - zr[t]);
          g1 += fabs(zz - zr[t + 1]);
        }
        if (t < half) g0 += fabs(zz - zr[t]);
        if (even) g1 += 0.5 * fabs(zz - zr[half]);
        const double gsum = g0 + g1;
        acc += 0.5 * gsum + 0.5 * static_cast<double>(s - 1) * zz;
        if (zz == 0.0) continue;
        // zz's pairs with the other row's row-only values (one search, sign-selected row)
        const bool pos = zz > 0.0;
        const double mg = fabs(zz);
        const float f = __double2float_rz(mg);
        const uint32_t code = fkey(f) + ((static_cast<double>(f) != mg) ? 1u : 0u);
        const int n = pos ? ci : cj;
        const int lb = lower_count_codes(ssc + (pos ? ri : rj) * stride, n, code);  // #{row values < |zz|}
        const int ql = qcount(QM + (pos ? 0 : 8), QM + (pos ? 16 : 24), lb, s);
        const double sl = (lb < n) ? __ldg((pos ? sufi : sufj) + lb) : 0.0;
        if (pos)
          acc += (kp - wneg) * zz + zz * static_cast<double>(lb - ql) + sl - sumQi + PQi[ql];
        else
          acc += kn * zz - ((s1j - sl) - PQj[ql] + mg * static_cast<double>((cj - lb) - (s - ql)));
      }
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, dd);
      if (lane == 0) {
        const double val = clamp_nonneg(acc);
        ot[0] = val;
        for (int v = 1; v < a.nnu; ++v) ot[v * kTile * tstride] = val;
        if (isinf(val)) atomicOr(a.flag, 1);
      }
      __syncwarp();
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, kTile, tstride, i0, j0, out, nullptr, nullptr);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// gini_gmd2_kernel: the same arithmetic as gini_gmd_kernel (every fp64 term is unchanged;
// the terms are added in list order instead of feature order, so results agree to round-off,
// ~1e-15 max-normalised), with three
// changes to the work around it (round 2, profiles/r1_gini_gmd_lines_n4000.txt:
// F extraction 13%, the 8-probe search 11% of the warp instructions):
//   * F lists are built for 8 pairs at a time by 4 lanes per pair (each lane walks
//     every fourth mask word and writes the (row-i index, row-j index) byte pairs of
//     its common features at its group-prefix offset), instead of one warp-wide scan
//     and compaction per pair; the element phase reads its list entry directly;
//   * the lower bound of |z| in a sorted row comes from a 256-bucket table per row
//     (bkt/bscale, built once per matrix by row_bucket_kernel) and a short scan inside
//     the bucket, instead of an 8-probe binary search;
//   * the panel keeps the sorted values and the position map only (feature-order
//     values are sv[pmap[k]]), which pays for the lists and the tables in shared memory.
// Rows with more than 255 nonzeros take the overflow list (bucket counters are bytes).
// -DGMDS_BOUNDS_CHECK: every index the round-2b kernels form is checked and a violation traps (the
// stand-in for compute-sanitizer memcheck, which is closed on the GPU pool: tools/gpu/bounds_check.sh)
#ifdef GMDS_BOUNDS_CHECK
#define GMDS_CHK(cond)                                                                  \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("GMDS_BOUNDS_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);      \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define GMDS_CHK(cond) ((void)0)
#endif

namespace gmd2_detail {
constexpr int kBatch = 8;      // pairs per extraction batch (4 lanes each)
constexpr int kFLStride = 66;  // u16 per list: 64 entries + pad (33 words: lists start on distinct banks)
constexpr int kMaxC2 = 255;    // max nonzeros per staged row
// per-warp scratch (8-byte words): QM[32] u32 (16) | PQi[72] | PQj[72] | ZL[2][64] | lists (8 x 66 u16 = 132)
constexpr int kOffPQi2 = 16, kOffPQj2 = 88, kOffZL2 = 160, kOffFL2 = 288;
constexpr int kWarpWords2 = kOffFL2 + (kBatch * kFLStride * 2 + 7) / 8;
// gini_gen2_kernel: QM[32] u32 (16) | BL[2][64] (128) | HI, HJ: 2 x 256 u16 counters (128) | lists (132)
constexpr int kGenOffBL = 16, kGenOffH = 144, kGenOffFL = 272;
constexpr int kGenWords2 = kGenOffFL + (kBatch * kFLStride * 2 + 7) / 8;
}  // namespace gmd2_detail

template <typename TO, int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) gini_gmd2_kernel(GmdArgs ga, TO* __restrict__ out) {
  using namespace gmd_detail;
  using namespace gmd2_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SplitArgs& sa = ga.s;
  const GiniTileArgs& a = sa.g;
  const int d = a.d;
  const int W = sa.W;
  const int stride = sa.maxnnz;  // panel stride (<= kMaxC2): rows with more nonzeros overflow
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // ---- shared memory
  double* wscr = reinterpret_cast<double*>(smem_raw) + warp * kWarpWords2;
  uint32_t* QM = reinterpret_cast<uint32_t*>(wscr);  // qm_i[8] qm_j[8] qp_i[8] qp_j[8]
  double* PQi = wscr + kOffPQi2;
  double* PQj = wscr + kOffPQj2;
  double* ZL = wscr + kOffZL2;  // z on F, stored twice (list order): circular reads without a wrap
  uint16_t* FL = reinterpret_cast<uint16_t*>(wscr + kOffFL2);  // [kBatch][kFLStride]: ii | jj << 8
  double* otile = reinterpret_cast<double*>(smem_raw) + kWarps * kWarpWords2;  // [nnu][32][33]
  double* rs1 = otile + static_cast<size_t>(a.nnu) * kTile * (kTile + 1);
  double* rtm = rs1 + kRows;
  int64_t* rbase = reinterpret_cast<int64_t*>(rtm + kRows);
  int* rcnt = reinterpret_cast<int*>(rbase + kRows);
  float* rscale = reinterpret_cast<float*>(rcnt + kRows);
  uint32_t* smask = reinterpret_cast<uint32_t*>(rscale + kRows);  // [64][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + kRows * W);
  uint32_t* ssv = reinterpret_cast<uint32_t*>(spre + ((kRows * W + 1) & ~1));  // [64][stride] sorted value bits
  uint16_t* spm = reinterpret_cast<uint16_t*>(ssv + kRows * stride);            // [64][stride] sorted position
  uint8_t* sbk = reinterpret_cast<uint8_t*>(spm + ((kRows * stride + 1) & ~1));  // [64][256] bucket starts
  const uint32_t* gsv = reinterpret_cast<const uint32_t*>(ga.svs);
  const double h = 0.5 * static_cast<double>(d + 1);
  const int tstride = kTile + 1;
  const int g4 = lane >> 2, sub = lane & 3;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * kTile, j0 = J * kTile;
    for (int e = threadIdx.x; e < kRows * W; e += blockDim.x) {
      const int r = e / W, w = e - (e / W) * W;
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
      spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
    }
    for (int r = warp; r < kRows; r += kWarps) {
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      int cnt = 0;
      int64_t b = 0;
      if (row < a.n) {
        b = sa.rowptr[row];
        cnt = static_cast<int>(sa.rowptr[row + 1] - b);
        for (int k = lane; k < cnt && k < stride; k += 32) {
          ssv[r * stride + k] = gsv[b + k];
          spm[r * stride + k] = ga.pmap[b + k];
        }
        const uint32_t* gb = reinterpret_cast<const uint32_t*>(ga.bkt) + row * 64;
        uint32_t* sb = reinterpret_cast<uint32_t*>(sbk) + r * 64;
        sb[lane] = gb[lane];
        sb[lane + 32] = gb[lane + 32];
      }
      if (lane == 0) {
        rcnt[r] = cnt;
        rbase[r] = b;
        rs1[r] = (row < a.n) ? ga.s1[row] : 0.0;
        rtm[r] = (row < a.n) ? ga.tm[row] : 0.0;
        rscale[r] = (row < a.n) ? ga.bscale[row] : 0.f;
      }
    }
    __syncthreads();

    for (int t0 = 0; warp + kWarps * t0 < kTile * kTile; t0 += kBatch) {
      // ---- F lists of this batch: 4 lanes per pair, every fourth mask word each
      int stat;  // the pair's |F|, or 0x100: overflow list, 0x200: not a pair of this tile
      {
        const int kg = warp + kWarps * (t0 + g4);
        bool valid = kg < kTile * kTile;
        const int rg = valid ? (kg >> 5) : 0, cg = valid ? (kg & 31) : 0;
        valid = valid && (j0 + cg < a.n) && (i0 + rg < j0 + cg);
        const uint32_t* mi = smask + rg * W;
        const uint32_t* mj = smask + (kTile + cg) * W;
        int cnt = 0;
        if (valid)
          for (int w = sub; w < W; w += 4) cnt += __popc(mi[w] & mj[w]);
        int incl = cnt;
        int o = __shfl_up_sync(0xffffffffu, incl, 1, 4);
        if (sub >= 1) incl += o;
        o = __shfl_up_sync(0xffffffffu, incl, 2, 4);
        if (sub >= 2) incl += o;
        const int sg = __shfl_sync(0xffffffffu, incl, 3, 4);
        const bool ok = valid && sg <= kCap && rcnt[rg] <= stride && rcnt[kTile + cg] <= stride;
        if (ok) {
          int off = incl - cnt;
          uint16_t* fl = FL + g4 * kFLStride;
          const uint16_t* pim = spre + rg * W;
          const uint16_t* pjm = spre + (kTile + cg) * W;
          for (int w = sub; w < W; w += 4) {
            const uint32_t wa = mi[w], wb = mj[w];
            uint32_t m = wa & wb;
            const int bi = pim[w], bj = pjm[w];
            while (m) {
              const int bit = __ffs(m) - 1;
              m &= m - 1u;
              const uint32_t lo = (1u << bit) - 1u;
              GMDS_CHK(off >= 0 && off < kCap && bi + __popc(wa & lo) < 256 && bj + __popc(wb & lo) < 256);
              fl[off++] = static_cast<uint16_t>((bi + __popc(wa & lo)) | ((bj + __popc(wb & lo)) << 8));
            }
          }
        }
        stat = !valid ? 0x200 : (ok ? sg : 0x100);
      }
      __syncwarp();

      for (int gg = 0; gg < kBatch; ++gg) {
        const int st = __shfl_sync(0xffffffffu, stat, gg * 4);
        if (st & 0x200) continue;  // warp-uniform
        const int k0 = warp + kWarps * (t0 + gg);
        const int r = k0 >> 5, c = k0 & 31;
        const int64_t gi = i0 + r, gj = j0 + c;
        const int ri = r, rj = kTile + c;
        const int ci = rcnt[ri], cj = rcnt[rj];
        double* ot = otile + r * tstride + c;
        if (st & 0x100) {  // overflow list: the exact full-sort kernel
          if (lane == 0) {
            const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
            if (static_cast<int64_t>(slot) < sa.ovf_cap) {
              sa.ovf_pairs[2 * slot] = gi;
              sa.ovf_pairs[2 * slot + 1] = gj;
            }
            for (int v = 0; v < a.nnu; ++v) ot[v * kTile * tstride] = -1.0;
          }
          continue;
        }
        const int s = st;
        const uint16_t* fl = FL + gg * kFLStride;
        if (lane < 16) QM[lane] = 0u;
        __syncwarp();
        const uint32_t* svi = ssv + ri * stride;
        const uint32_t* svj = ssv + rj * stride;
        const uint16_t* pmi = spm + ri * stride;
        const uint16_t* pmj = spm + rj * stride;
        // ---- F's values and sorted positions in both rows; position masks
        float al[2], be[2];
        int pI[2], pJ[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = lane + 32 * u;
          al[u] = be[u] = 0.f;
          pI[u] = pJ[u] = kMaxC;  // sentinel: qcount -> s, never stored
          if (u == 1 && s <= 32) break;  // warp-uniform: the second element slot is empty
          if (e < s) {
            const uint32_t pk = fl[e];
            GMDS_CHK(static_cast<int>(pk & 255u) < ci && static_cast<int>(pk >> 8) < cj && ci <= stride && cj <= stride);
            pI[u] = pmi[pk & 255u];
            pJ[u] = pmj[pk >> 8];
            GMDS_CHK(pI[u] < ci && pJ[u] < cj);
            al[u] = __uint_as_float(svi[pI[u]]);
            be[u] = __uint_as_float(svj[pJ[u]]);
            atomicOr(QM + (pI[u] >> 5), 1u << (pI[u] & 31));
            atomicOr(QM + 8 + (pJ[u] >> 5), 1u << (pJ[u] & 31));
          }
        }
        __syncwarp();
        {  // word prefixes of the two masks (groups of 8 lanes)
          const uint32_t wv = (lane < 16) ? QM[lane] : 0u;
          const int pc = __popc(wv);
          int x = pc;
#pragma unroll
          for (int dd = 1; dd < 8; dd <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, x, dd, 8);
            if ((lane & 7) >= dd) x += o;
          }
          if (lane < 16) QM[16 + lane] = static_cast<uint32_t>(x - pc);
        }
        __syncwarp();
        // ---- position-order ranks; F's values scattered in that order
        int rI[2], rJ[2];
        double z[2];
        int mneg = 0, mpos = 0;
        z[1] = 0.0;
        rI[1] = rJ[1] = s;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && s <= 32) break;  // warp-uniform
          rI[u] = qcount2(QM, QM + 16, pI[u]);
          rJ[u] = qcount2(QM + 8, QM + 24, pJ[u]);
          const bool live = lane + 32 * u < s;
          if (live) {
            GMDS_CHK(rI[u] >= 0 && rI[u] < s && rJ[u] >= 0 && rJ[u] < s && s <= kCap);
            PQi[1 + rI[u]] = static_cast<double>(al[u]);
            PQj[1 + rJ[u]] = static_cast<double>(be[u]);
          }
          z[u] = static_cast<double>(al[u]) - static_cast<double>(be[u]);
          if (live) {
            ZL[lane + 32 * u] = z[u];
            ZL[lane + 32 * u + s] = z[u];
          }
          mneg += __popc(__ballot_sync(0xffffffffu, z[u] < 0.0));
          mpos += __popc(__ballot_sync(0xffffffffu, z[u] > 0.0));
        }
        __syncwarp();
        {  // prefix sums PQ[k] = sum of the first k values in position order
          const int t1a = 1 + 2 * lane, t1b = t1a + 1;
          const double a0 = (t1a <= s) ? PQi[t1a] : 0.0, a1 = (t1b <= s) ? PQi[t1b] : 0.0;
          const double b0 = (t1a <= s) ? PQj[t1a] : 0.0, b1 = (t1b <= s) ? PQj[t1b] : 0.0;
          const double ea = warp_incl(a0 + a1, lane) - (a0 + a1);
          const double eb = warp_incl(b0 + b1, lane) - (b0 + b1);
          __syncwarp();
          if (t1a <= s) {
            PQi[t1a] = ea + a0;
            PQj[t1a] = eb + b0;
          }
          if (t1b <= s) {
            PQi[t1b] = ea + a0 + a1;
            PQj[t1b] = eb + b0 + b1;
          }
          if (lane == 0) {
            PQi[0] = 0.0;
            PQj[0] = 0.0;
          }
        }
        __syncwarp();
        const int nP = ci - s + mpos, nN = cj - s + mneg;
        const double kp = static_cast<double>(1 + nN + (d - nP - nN)) - h, kn = 1.0 - h;
        const double* sufi = ga.suf + rbase[ri];
        const double* sufj = ga.suf + rbase[rj];
        const double s1j = rs1[rj];
        double acc = 0.0;
        if (lane == 0) acc = kp * rs1[ri] - kn * s1j + rtm[ri] - (static_cast<double>(cj - 1) * s1j - rtm[rj]);
        const double sumQi = PQi[s];
        const double wneg = static_cast<double>(s - mpos);  // |S_ab-| + |Z0|
        const int half = (s - 1) >> 1;
        const bool even = (s & 1) == 0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && s <= 32) break;  // warp-uniform
          const int e = lane + 32 * u;
          if (e >= s) continue;
          const double av = al[u], bv = be[u];
          // pairs of row i touching F (PM(S_a)) and of row j (minima, PM(S_b))
          const double si1v = __ldg(sufi + min(pI[u] + 1, ci - 1));  // clamped: no branch around the load
          const double si1 = (pI[u] + 1 < ci) ? si1v : 0.0;
          const double sj0 = __ldg(sufj + pJ[u]);
          acc += av * static_cast<double>(rI[u] - pI[u]) - si1 - kp * av;
          acc += (s1j - sj0) + bv * static_cast<double>((cj - 1 - pJ[u]) - (s - 1 - rJ[u])) + kn * bv;
          const double zz = z[u];
          // PM(Z) pieces
          double g0 = 0.0, g1 = 0.0;  // two chains: DADD latency
          const double* zr = ZL + e + 1;
          int tq = 0;
          for (; tq + 1 < half; tq += 2) {
            g0 += fabs(zz - zr[tq]);
            g1 += fabs(zz - zr[tq + 1]);
          }
          if (tq < half) g0 += fabs(zz - zr[tq]);
          if (even) g1 += 0.5 * fabs(zz - zr[half]);
          const double gsum = g0 + g1;
          acc += 0.5 * gsum + 0.5 * static_cast<double>(s - 1) * zz;
          if (zz == 0.0) continue;
          // zz's pairs with the other row's row-only values: #{row values < |zz|} from the
          // row's bucket table and a scan inside the bucket (sign-selected row)
          const bool pos = zz > 0.0;
          const double mg = fabs(zz);
          const float f = __double2float_rz(mg);
          const uint32_t tt = __float_as_uint(f) + ((static_cast<double>(f) != mg) ? 1u : 0u);
          const int prow = pos ? ri : rj;
          const int n = pos ? ci : cj;
          const uint32_t* sb = ssv + prow * stride;
          const uint8_t* tb = sbk + prow * 256;
          const int bk = min(255, __float2int_rz(f * rscale[prow]));
          GMDS_CHK(bk >= 0 && n >= 1 && n <= stride);
          int lb = tb[bk];
          const int end = (bk < 255) ? static_cast<int>(tb[bk + 1]) : n;
          GMDS_CHK(lb <= end && end <= n);
          while (lb < end && sb[lb] < tt) ++lb;
          GMDS_CHK(lb == n || sb[lb] >= tt);
          GMDS_CHK(lb == 0 || sb[lb - 1] < tt);  // the bucket scan found the exact lower bound
          const int ql = qcount2(QM + (pos ? 0 : 8), QM + (pos ? 16 : 24), lb);
          const double slv = __ldg((pos ? sufi : sufj) + min(lb, n - 1));
          const double sl = (lb < n) ? slv : 0.0;
          if (pos)
            acc += (kp - wneg) * zz + zz * static_cast<double>(lb - ql) + sl - sumQi + PQi[ql];
          else
            acc += kn * zz - ((s1j - sl) - PQj[ql] + mg * static_cast<double>((cj - lb) - (s - ql)));
        }
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, dd);
        if (lane == 0) {
          const double val = clamp_nonneg(acc);
          ot[0] = val;
          for (int v = 1; v < a.nnu; ++v) ot[v * kTile * tstride] = val;
          if (isinf(val)) atomicOr(a.flag, 1);
        }
        __syncwarp();
      }
      __syncwarp();
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, kTile, tstride, i0, j0, out, nullptr, nullptr);
    __syncthreads();
  }
}

inline size_t gmd2_smem(int W, int maxnnz, int nnu, int nwarps) {
  using namespace gmd_detail;
  using namespace gmd2_detail;
  return static_cast<size_t>(nwarps) * kWarpWords2 * 8 + static_cast<size_t>(nnu) * kTile * (kTile + 1) * 8 +
         kRows * (8 + 8 + 8 + 4 + 4) + kRows * W * 4 + ((kRows * W + 1) & ~1) * 2 +
         static_cast<size_t>(kRows) * maxnnz * 4 + ((static_cast<size_t>(kRows) * maxnnz + 1) & ~size_t(1)) * 2 +
         kRows * 256 + 16;
}

// per-row bucket tables of the sorted values (gini_gmd2_kernel's search)
void launch_row_buckets(const float* svs, const int64_t* rowptr, int64_t n, uint8_t* bkt, float* bscale,
                        cudaStream_t st);
void launch_gini_gmd2(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                      cudaStream_t st);

// ---------------------------------------------------------------------------
// General-nu kernel on the same panels (nu not in {2, 3}, nnu <= 4): every
// element's midrank is a count, and the weight comes from the LUT
// (gini_tile.cuh: L[2 #less + #equal], p/2 sum z L).  With F, its sorted
// positions and the position masks as in the linear kernel:
//   x in S_a at row-i position k (tie group [g0, g1)):
//     #less  = n_neg + zeros + (g0 - f_i(g0)) + #{b in S_ab+ : lb_b <= k}
//     #equal = (g1 - g0) - (f_i(g1) - f_i(g0))
//   -x in S_b at row-j position k:
//     #less  = (cj - g1) - (s - f_j(g1)) + |S_ab-| - #{b in S_ab- : lb_b <= k}
//   b in S_ab+- : #less from its rank in its sign group (counting loop over
//     the group, fp64) and its lower bound lb_b in the other row,
// where f_r(pos) = #{F positions < pos} (popc prefix of the position mask)
// and the S_ab counts come from a per-warp histogram over row positions read
// back with a warp scan per 32-element chunk.  One pass over each row's
// nonzeros, no sort and no merge network.  Pairs whose S_ab values tie
// anything (each other, or a value of the other row) go to the exact
// overflow list, as do s > 64 and rows longer than the panel stride.
template <typename TO, int kWarps, int NNU>
__global__ void __launch_bounds__(kWarps * 32, 1) gini_gen_kernel(GmdArgs ga, TO* __restrict__ out) {
  using namespace gmd_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SplitArgs& sa = ga.s;
  const GiniTileArgs& a = sa.g;
  const int d = a.d;
  const int W = sa.W;
  const int stride = sa.maxnnz;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  double* wscr = reinterpret_cast<double*>(smem_raw) + warp * kWarpWords;
  int* F = reinterpret_cast<int*>(wscr);
  uint32_t* QM = reinterpret_cast<uint32_t*>(wscr + kOffQM);  // qm_i[8] qm_j[8] qp_i[8] qp_j[8]
  double* BL = wscr + kOffPQi;                                // [0, 64): S_ab- values, [64, 128): S_ab+
  uint32_t* HI = reinterpret_cast<uint32_t*>(wscr + kOffPQi + 2 * kCap);  // 256 u16 counters
  uint32_t* HJ = HI + 128;
  double* otile = reinterpret_cast<double*>(smem_raw) + kWarps * kWarpWords;  // [nnu][32][33]
  double* rs1 = otile + static_cast<size_t>(a.nnu) * kTile * (kTile + 1);
  double* rtm = rs1 + kRows;
  int64_t* rbase = reinterpret_cast<int64_t*>(rtm + kRows);
  int* rcnt = reinterpret_cast<int*>(rbase + kRows);
  uint32_t* smask = reinterpret_cast<uint32_t*>(rcnt + kRows);  // [64][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + kRows * W);
  float* svals = reinterpret_cast<float*>(spre + ((kRows * W + 1) & ~1));  // [64][stride]
  float* ssv = svals + kRows * stride;                                       // [64][stride]
  uint16_t* spm = reinterpret_cast<uint16_t*>(ssv + kRows * stride);         // [64][stride]
  uint32_t* stie = reinterpret_cast<uint32_t*>(spm + ((kRows * stride + 1) & ~1));  // [64][8]
  const float* gv = static_cast<const float*>(sa.vals);
  const double half_p = 0.5 * static_cast<double>(d);
  const int tstride = kTile + 1;
  const int nnu = (NNU == 1) ? 1 : a.nnu;
  const int lstride = 2 * d;
  __shared__ double s_score[2 * kMaxScoreNu];
  __shared__ double s_red[32 * 8];
  for (int e = threadIdx.x; e < 2 * kMaxScoreNu; e += blockDim.x) s_score[e] = 0.0;
  for (int e = lane; e < 256; e += 32) HI[e] = 0u;  // HI and HJ: left zero after every pair

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * kTile, j0 = J * kTile;
    for (int e = threadIdx.x; e < kRows * W; e += blockDim.x) {
      const int r = e / W, w = e - (e / W) * W;
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
      spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
    }
    for (int r = warp; r < kRows; r += kWarps) {
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      int cnt = 0;
      if (row < a.n) {
        const int64_t b = sa.rowptr[row];
        cnt = static_cast<int>(sa.rowptr[row + 1] - b);
        for (int k = lane; k < cnt && k < stride; k += 32) {
          svals[r * stride + k] = gv[b + k];
          ssv[r * stride + k] = ga.svs[b + k];
          spm[r * stride + k] = ga.pmap[b + k];
        }
      }
      if (lane == 0) rcnt[r] = cnt;
      if (lane < 8) stie[r * 8 + lane] = (row < a.n) ? ga.tiew[row * 8 + lane] : 0u;
    }
    __syncthreads();

    for (int k0 = warp; k0 < kTile * kTile; k0 += kWarps) {
      const int r = k0 >> 5, c = k0 & 31;
      const int64_t gi = i0 + r, gj = j0 + c;
      if (!(gj < a.n && gi < gj)) continue;
      const int ri = r, rj = kTile + c;
      const int ci = rcnt[ri], cj = rcnt[rj];
      const uint32_t* mi = smask + ri * W;
      const uint32_t* mj = smask + rj * W;
      double* ot = otile + r * tstride + c;
      auto overflow = [&]() {
        if (lane == 0) {
          const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
          if (static_cast<int64_t>(slot) < sa.ovf_cap) {
            sa.ovf_pairs[2 * slot] = gi;
            sa.ovf_pairs[2 * slot + 1] = gj;
          }
          for (int v = 0; v < nnu; ++v) ot[v * kTile * tstride] = -1.0;
        }
      };
      // ---- F = features nonzero in both rows
      if (lane < 16) QM[lane] = 0u;
      uint32_t m = (lane < W) ? (mi[lane] & mj[lane]) : 0u;
      const int cm = __popc(m);
      int incl = cm;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, dd);
        if (lane >= dd) incl += o;
      }
      const int s = __shfl_sync(0xffffffffu, incl, 31);
      if (s > kCap || ci > stride || cj > stride) {
        overflow();
        continue;
      }
      {
        int off = incl - cm;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1u;
          F[off++] = (lane << 5) | b;
        }
      }
      __syncwarp();
      const uint16_t* pim = spre + ri * W;
      const uint16_t* pjm = spre + rj * W;
      const float* vi = svals + ri * stride;
      const float* vj = svals + rj * stride;
      const float* svi = ssv + ri * stride;
      const float* svj = ssv + rj * stride;
      // ---- F's values and sorted positions in both rows; position masks
      double z[2];
      int lbp[2];  // histogram position of this lane's S_ab values (-1: none)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = lane + 32 * u;
        z[u] = 0.0;
        lbp[u] = -1;
        if (e < s) {
          const int f = F[e];
          const int w = f >> 5;
          const uint32_t lo = (1u << (f & 31)) - 1u;
          const int ii = pim[w] + __popc(mi[w] & lo);
          const int jj = pjm[w] + __popc(mj[w] & lo);
          z[u] = static_cast<double>(vi[ii]) - static_cast<double>(vj[jj]);
          const int pI = spm[ri * stride + ii], pJ = spm[rj * stride + jj];
          atomicOr(QM + (pI >> 5), 1u << (pI & 31));
          atomicOr(QM + 8 + (pJ >> 5), 1u << (pJ & 31));
        }
      }
      int mneg = 0, mpos = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const unsigned bn = __ballot_sync(0xffffffffu, z[u] < 0.0);
        const unsigned bq = __ballot_sync(0xffffffffu, z[u] > 0.0);
        if (z[u] < 0.0) BL[mneg + __popc(bn & lt)] = z[u];
        if (z[u] > 0.0) BL[kCap + mpos + __popc(bq & lt)] = z[u];
        mneg += __popc(bn);
        mpos += __popc(bq);
      }
      __syncwarp();
      {  // word prefixes of the two masks (groups of 8 lanes)
        const uint32_t wv = (lane < 16) ? QM[lane] : 0u;
        const int pc = __popc(wv);
        int x = pc;
#pragma unroll
        for (int dd = 1; dd < 8; dd <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, x, dd, 8);
          if ((lane & 7) >= dd) x += o;
        }
        if (lane < 16) QM[16 + lane] = static_cast<uint32_t>(x - pc);
      }
      __syncwarp();
      const int n_neg = (cj - s) + mneg, n_pos = (ci - s) + mpos;
      const int zeros = d - n_neg - n_pos;
      // ---- S_ab values: rank in their sign group, lower bound in the other row
      bool bad = false;
      int bidx[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        bidx[u] = -1;
        const double zz = z[u];
        if (zz == 0.0) continue;
        const bool pos = zz > 0.0;
        const double* L = BL + (pos ? kCap : 0);
        const int len = pos ? mpos : mneg;
        int cl = 0, ce = 0;
        for (int q = 0; q < len; ++q) {
          const double o = L[q];
          cl += (o < zz) ? 1 : 0;
          ce += (o == zz) ? 1 : 0;
        }
        if (ce != 1) bad = true;  // two equal S_ab values
        const double mg = fabs(zz);
        const float f = __double2float_rz(mg);
        const uint32_t code = fkey(f) + ((static_cast<double>(f) != mg) ? 1u : 0u);
        const int n = pos ? ci : cj;
        const float* sv = pos ? svi : svj;
        const int lb = lower_count(sv, n, code);
        if (lb < n && fkey(sv[lb]) == code) bad = true;  // equal to a value of the other row
        const int ql = qcount(QM + (pos ? 0 : 8), QM + (pos ? 16 : 24), lb, s);
        const int less = pos ? n_neg + zeros + cl + (lb - ql) : cl + (cj - lb) - (s - ql);
        bidx[u] = 2 * less + 1;
        lbp[u] = (lb < n) ? (pos ? lb : 256 + lb) : -1;
      }
      if (__any_sync(0xffffffffu, bad)) {
        overflow();
        continue;
      }
      double acc[NNU];
#pragma unroll
      for (int v = 0; v < NNU; ++v) acc[v] = 0.0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (lbp[u] >= 0) hist_add(HI, lbp[u]);  // HJ == HI + 128: position 256 + lb
        if (bidx[u] >= 0) {
#pragma unroll
          for (int v = 0; v < NNU; ++v)
            if (NNU == 1 || v < nnu) acc[v] = fma(z[u], __ldg(a.lut + v * lstride + bidx[u]), acc[v]);
        }
      }
      __syncwarp();
      // ---- one pass over each row's nonzeros (S_a of row i, S_b of row j)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const bool RI = side == 0;
        const int cnt = RI ? ci : cj;
        const float* sv = RI ? svi : svj;
        const uint32_t* qm = QM + (RI ? 0 : 8);
        const uint32_t* qp = QM + (RI ? 16 : 24);
        const uint32_t* H = RI ? HI : HJ;
        int carry = 0;
        for (int base = 0; base < cnt; base += 32) {
          const int k = base + lane;
          const bool in = k < cnt;
          const uint32_t qw = qm[base >> 5];
          const int rem = (qw >> lane) & 1u;
          const bool live = in && !rem;
          const float x = in ? sv[k] : -2.f;
          // S_ab values counted at positions <= k: a popc of the chunk's occupied
          // positions, or a warp scan when a position holds more than one
          const int hc = in ? hist_get(H, k) : 0;
          const unsigned occ = __ballot_sync(0xffffffffu, hc > 0);
          int hs;
          if (__any_sync(0xffffffffu, hc > 1)) {
            hs = hc;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
              const int o = __shfl_up_sync(0xffffffffu, hs, dd);
              if (lane >= dd) hs += o;
            }
            hs += carry;
            carry = __shfl_sync(0xffffffffu, hs, 31);
          } else {
            hs = carry + __popc(occ & (lt | (1u << lane)));
            carry += __popc(occ);
          }
          int g0 = k, g1 = k + 1;
          int rb0 = static_cast<int>(qp[base >> 5]) + __popc(qw & lt);
          int rb1 = rb0 + rem;
          // tie groups in the row (clipped values, repeats) from the row's tie bits:
          // group bounds by bit scans; only a group crossing a 32-entry chunk walks the row
          const int prow = RI ? ri : rj;
          const uint32_t tw = stie[prow * 8 + (base >> 5)];
          const uint32_t pbit = (base > 0) ? (stie[prow * 8 + (base >> 5) - 1] >> 31) : 0u;
          const bool tied = live && ((lane > 0 ? (tw >> (lane - 1)) & 1u : pbit) || ((tw >> lane) & 1u));
          if (tied) {
            const uint32_t below = ~tw & lt;                    // positions t < lane with v_t != v_(t+1)
            const uint32_t above = ~tw & (0xffffffffu << lane);  // positions t >= lane with v_t != v_(t+1)
            bool cross = false;
            if (below) {
              g0 = base + 32 - __clz(below);
            } else {
              g0 = base;
              cross = pbit != 0;
            }
            if (above) {
              g1 = base + __ffs(above);
            } else {
              g1 = base + 32;
              cross = true;
            }
            if (cross) {
              while (g0 > 0 && sv[g0 - 1] == x) --g0;
              while (g1 < cnt && sv[g1] == x) ++g1;
            }
            rb0 = qcount(qm, qp, g0, s);
            rb1 = qcount(qm, qp, g1, s);
          }
          if (live) {
            const int eq = (g1 - g0) - (rb1 - rb0);
            const int less = RI ? n_neg + zeros + (g0 - rb0) + hs : (cnt - g1) - (s - rb1) + (mneg - hs);
            const int idx = 2 * less + eq;
            const double zv = RI ? static_cast<double>(x) : -static_cast<double>(x);
#pragma unroll
            for (int v = 0; v < NNU; ++v)
              if (NNU == 1 || v < nnu) acc[v] = fma(zv, __ldg(a.lut + v * lstride + idx), acc[v]);
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (lbp[u] >= 0) HI[lbp[u] >> 1] = 0u;  // leave the histograms zero
#pragma unroll
      for (int v = 0; v < NNU; ++v) {
        if (NNU > 1 && v >= nnu) break;
        double sum = acc[v];
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, dd);
        if (lane == 0) {
          const double val = clamp_nonneg(half_p * sum);
          ot[v * kTile * tstride] = val;
          if (isinf(val)) atomicOr(a.flag, 1);
        }
      }
      __syncwarp();
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, kTile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}

// gini_gen2_kernel: gini_gen_kernel with gini_gmd2_kernel's batched F lists, bucket-table lower
// bounds and the (sorted values, position map) panel; same counts, LUT indices and sums.
template <typename TO, int kWarps, int NNU>
__global__ void __launch_bounds__(kWarps * 32, 1) gini_gen2_kernel(GmdArgs ga, TO* __restrict__ out) {
  using namespace gmd_detail;
  using namespace gmd2_detail;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SplitArgs& sa = ga.s;
  const GiniTileArgs& a = sa.g;
  const int d = a.d;
  const int W = sa.W;
  const int stride = sa.maxnnz;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  double* wscr = reinterpret_cast<double*>(smem_raw) + warp * kGenWords2;
  uint32_t* QM = reinterpret_cast<uint32_t*>(wscr);  // qm_i[8] qm_j[8] qp_i[8] qp_j[8]
  double* BL = wscr + kGenOffBL;                     // [0, 64): S_ab- values, [64, 128): S_ab+
  uint32_t* HI = reinterpret_cast<uint32_t*>(wscr + kGenOffH);  // 256 u16 counters
  uint32_t* HJ = HI + 128;
  uint16_t* FL = reinterpret_cast<uint16_t*>(wscr + kGenOffFL);  // [kBatch][kFLStride]: ii | jj << 8
  double* otile = reinterpret_cast<double*>(smem_raw) + kWarps * kGenWords2;  // [nnu][32][33]
  double* rs1 = otile + static_cast<size_t>(a.nnu) * kTile * (kTile + 1);
  double* rtm = rs1 + kRows;
  int64_t* rbase = reinterpret_cast<int64_t*>(rtm + kRows);
  int* rcnt = reinterpret_cast<int*>(rbase + kRows);
  float* rscale = reinterpret_cast<float*>(rcnt + kRows);
  uint32_t* smask = reinterpret_cast<uint32_t*>(rscale + kRows);  // [64][W]
  uint16_t* spre = reinterpret_cast<uint16_t*>(smask + kRows * W);
  float* ssv = reinterpret_cast<float*>(spre + ((kRows * W + 1) & ~1));      // [64][stride] sorted values
  uint16_t* spm = reinterpret_cast<uint16_t*>(ssv + kRows * stride);         // [64][stride] sorted position
  uint32_t* stie = reinterpret_cast<uint32_t*>(spm + ((kRows * stride + 1) & ~1));  // [64][8]
  uint8_t* sbk = reinterpret_cast<uint8_t*>(stie + kRows * 8);               // [64][256] bucket starts
  const int g4 = lane >> 2, sub = lane & 3;
  const double half_p = 0.5 * static_cast<double>(d);
  const int tstride = kTile + 1;
  const int nnu = (NNU == 1) ? 1 : a.nnu;
  const int lstride = 2 * d;
  __shared__ double s_score[2 * kMaxScoreNu];
  __shared__ double s_red[32 * 8];
  for (int e = threadIdx.x; e < 2 * kMaxScoreNu; e += blockDim.x) s_score[e] = 0.0;
  for (int e = lane; e < 256; e += 32) HI[e] = 0u;  // HI and HJ: left zero after every pair

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
    if (!tile_in_blocks(a, I, J)) continue;
    const int64_t i0 = I * kTile, j0 = J * kTile;
    for (int e = threadIdx.x; e < kRows * W; e += blockDim.x) {
      const int r = e / W, w = e - (e / W) * W;
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      smask[e] = (row < a.n) ? sa.masks[row * W + w] : 0u;
      spre[e] = (row < a.n) ? sa.prefix[row * W + w] : uint16_t(0);
    }
    for (int r = warp; r < kRows; r += kWarps) {
      const int64_t row = (r < kTile) ? i0 + r : j0 + (r - kTile);
      int cnt = 0;
      if (row < a.n) {
        const int64_t b = sa.rowptr[row];
        cnt = static_cast<int>(sa.rowptr[row + 1] - b);
        for (int k = lane; k < cnt && k < stride; k += 32) {
          ssv[r * stride + k] = ga.svs[b + k];
          spm[r * stride + k] = ga.pmap[b + k];
        }
        const uint32_t* gb = reinterpret_cast<const uint32_t*>(ga.bkt) + row * 64;
        uint32_t* sb = reinterpret_cast<uint32_t*>(sbk) + r * 64;
        sb[lane] = gb[lane];
        sb[lane + 32] = gb[lane + 32];
      }
      if (lane == 0) {
        rcnt[r] = cnt;
        rscale[r] = (row < a.n) ? ga.bscale[row] : 0.f;
      }
      if (lane < 8) stie[r * 8 + lane] = (row < a.n) ? ga.tiew[row * 8 + lane] : 0u;
    }
    __syncthreads();

    for (int t0 = 0; warp + kWarps * t0 < kTile * kTile; t0 += kBatch) {
      // ---- F lists of this batch: 4 lanes per pair, every fourth mask word each (gini_gmd2_kernel)
      int stat;  // the pair's |F|, or 0x100: overflow list, 0x200: not a pair of this tile
      {
        const int kg = warp + kWarps * (t0 + g4);
        bool valid = kg < kTile * kTile;
        const int rg = valid ? (kg >> 5) : 0, cg = valid ? (kg & 31) : 0;
        valid = valid && (j0 + cg < a.n) && (i0 + rg < j0 + cg);
        const uint32_t* mi = smask + rg * W;
        const uint32_t* mj = smask + (kTile + cg) * W;
        int cnt = 0;
        if (valid)
          for (int w = sub; w < W; w += 4) cnt += __popc(mi[w] & mj[w]);
        int incl = cnt;
        int o = __shfl_up_sync(0xffffffffu, incl, 1, 4);
        if (sub >= 1) incl += o;
        o = __shfl_up_sync(0xffffffffu, incl, 2, 4);
        if (sub >= 2) incl += o;
        const int sg = __shfl_sync(0xffffffffu, incl, 3, 4);
        const bool ok = valid && sg <= kCap && rcnt[rg] <= stride && rcnt[kTile + cg] <= stride;
        if (ok) {
          int off = incl - cnt;
          uint16_t* fl = FL + g4 * kFLStride;
          const uint16_t* pim = spre + rg * W;
          const uint16_t* pjm = spre + (kTile + cg) * W;
          for (int w = sub; w < W; w += 4) {
            const uint32_t wa = mi[w], wb = mj[w];
            uint32_t m = wa & wb;
            const int bi = pim[w], bj = pjm[w];
            while (m) {
              const int bit = __ffs(m) - 1;
              m &= m - 1u;
              const uint32_t lo = (1u << bit) - 1u;
              GMDS_CHK(off >= 0 && off < kCap && bi + __popc(wa & lo) < 256 && bj + __popc(wb & lo) < 256);
              fl[off++] = static_cast<uint16_t>((bi + __popc(wa & lo)) | ((bj + __popc(wb & lo)) << 8));
            }
          }
        }
        stat = !valid ? 0x200 : (ok ? sg : 0x100);
      }
      __syncwarp();
      for (int gg = 0; gg < kBatch; ++gg) {
      const int st = __shfl_sync(0xffffffffu, stat, gg * 4);
      if (st & 0x200) continue;  // warp-uniform
      const int k0 = warp + kWarps * (t0 + gg);
      const int r = k0 >> 5, c = k0 & 31;
      const int64_t gi = i0 + r, gj = j0 + c;
      const int ri = r, rj = kTile + c;
      const int ci = rcnt[ri], cj = rcnt[rj];
      double* ot = otile + r * tstride + c;
      auto overflow = [&]() {
        if (lane == 0) {
          const unsigned long long slot = atomicAdd(sa.ovf_count, 1ull);
          if (static_cast<int64_t>(slot) < sa.ovf_cap) {
            sa.ovf_pairs[2 * slot] = gi;
            sa.ovf_pairs[2 * slot + 1] = gj;
          }
          for (int v = 0; v < nnu; ++v) ot[v * kTile * tstride] = -1.0;
        }
      };
      if (st & 0x100) {
        overflow();
        continue;
      }
      const int s = st;
      const uint16_t* fl = FL + gg * kFLStride;
      if (lane < 16) QM[lane] = 0u;
      __syncwarp();
      const float* svi = ssv + ri * stride;
      const float* svj = ssv + rj * stride;
      // ---- F's values and sorted positions in both rows; position masks
      double z[2];
      int lbp[2];  // histogram position of this lane's S_ab values (-1: none)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = lane + 32 * u;
        z[u] = 0.0;
        lbp[u] = -1;
        if (e < s) {
          const uint32_t pk = fl[e];
          GMDS_CHK(static_cast<int>(pk & 255u) < ci && static_cast<int>(pk >> 8) < cj && ci <= stride && cj <= stride);
          const int pI = spm[ri * stride + (pk & 255u)], pJ = spm[rj * stride + (pk >> 8)];
          GMDS_CHK(pI < ci && pJ < cj);
          z[u] = static_cast<double>(svi[pI]) - static_cast<double>(svj[pJ]);
          atomicOr(QM + (pI >> 5), 1u << (pI & 31));
          atomicOr(QM + 8 + (pJ >> 5), 1u << (pJ & 31));
        }
      }
      int mneg = 0, mpos = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const unsigned bn = __ballot_sync(0xffffffffu, z[u] < 0.0);
        const unsigned bq = __ballot_sync(0xffffffffu, z[u] > 0.0);
        if (z[u] < 0.0) BL[mneg + __popc(bn & lt)] = z[u];
        if (z[u] > 0.0) BL[kCap + mpos + __popc(bq & lt)] = z[u];
        mneg += __popc(bn);
        mpos += __popc(bq);
      }
      __syncwarp();
      {  // word prefixes of the two masks (groups of 8 lanes)
        const uint32_t wv = (lane < 16) ? QM[lane] : 0u;
        const int pc = __popc(wv);
        int x = pc;
#pragma unroll
        for (int dd = 1; dd < 8; dd <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, x, dd, 8);
          if ((lane & 7) >= dd) x += o;
        }
        if (lane < 16) QM[16 + lane] = static_cast<uint32_t>(x - pc);
      }
      __syncwarp();
      const int n_neg = (cj - s) + mneg, n_pos = (ci - s) + mpos;
      const int zeros = d - n_neg - n_pos;
      // ---- S_ab values: rank in their sign group, lower bound in the other row
      bool bad = false;
      int bidx[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        bidx[u] = -1;
        const double zz = z[u];
        if (zz == 0.0) continue;
        const bool pos = zz > 0.0;
        const double* L = BL + (pos ? kCap : 0);
        const int len = pos ? mpos : mneg;
        int cl = 0, ce = 0;
        for (int q = 0; q < len; ++q) {
          const double o = L[q];
          cl += (o < zz) ? 1 : 0;
          ce += (o == zz) ? 1 : 0;
        }
        if (ce != 1) bad = true;  // two equal S_ab values
        const double mg = fabs(zz);
        const float f = __double2float_rz(mg);
        const bool inexact = static_cast<double>(f) != mg;
        const uint32_t tt = __float_as_uint(f) + (inexact ? 1u : 0u);
        const int n = pos ? ci : cj;
        const int prow = pos ? ri : rj;
        const uint32_t* sb = reinterpret_cast<const uint32_t*>(ssv) + prow * stride;
        const uint8_t* tb = sbk + prow * 256;
        const int bk = min(255, __float2int_rz(f * rscale[prow]));
        GMDS_CHK(bk >= 0 && n >= 1 && n <= stride);
        int lb = tb[bk];
        const int end = (bk < 255) ? static_cast<int>(tb[bk + 1]) : n;
        GMDS_CHK(lb <= end && end <= n);
        while (lb < end && sb[lb] < tt) ++lb;  // #{row values < |zz|}
        GMDS_CHK((lb == n || sb[lb] >= tt) && (lb == 0 || sb[lb - 1] < tt));
        if (!inexact && lb < n && sb[lb] == tt) bad = true;  // equal to a value of the other row
        const int ql = qcount(QM + (pos ? 0 : 8), QM + (pos ? 16 : 24), lb, s);
        const int less = pos ? n_neg + zeros + cl + (lb - ql) : cl + (cj - lb) - (s - ql);
        bidx[u] = 2 * less + 1;
        lbp[u] = (lb < n) ? (pos ? lb : 256 + lb) : -1;
      }
      if (__any_sync(0xffffffffu, bad)) {
        overflow();
        continue;
      }
      double acc[NNU];
#pragma unroll
      for (int v = 0; v < NNU; ++v) acc[v] = 0.0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (lbp[u] >= 0) hist_add(HI, lbp[u]);  // HJ == HI + 128: position 256 + lb
        if (bidx[u] >= 0) {
#pragma unroll
          for (int v = 0; v < NNU; ++v)
            if (NNU == 1 || v < nnu) acc[v] = fma(z[u], __ldg(a.lut + v * lstride + bidx[u]), acc[v]);
        }
      }
      __syncwarp();
      // ---- one pass over each row's nonzeros (S_a of row i, S_b of row j)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const bool RI = side == 0;
        const int cnt = RI ? ci : cj;
        const float* sv = RI ? svi : svj;
        const uint32_t* qm = QM + (RI ? 0 : 8);
        const uint32_t* qp = QM + (RI ? 16 : 24);
        const uint32_t* H = RI ? HI : HJ;
        int carry = 0;
        for (int base = 0; base < cnt; base += 32) {
          const int k = base + lane;
          const bool in = k < cnt;
          const uint32_t qw = qm[base >> 5];
          const int rem = (qw >> lane) & 1u;
          const bool live = in && !rem;
          const float x = in ? sv[k] : -2.f;
          // S_ab values counted at positions <= k: a popc of the chunk's occupied
          // positions, or a warp scan when a position holds more than one
          const int hc = in ? hist_get(H, k) : 0;
          const unsigned occ = __ballot_sync(0xffffffffu, hc > 0);
          int hs;
          if (__any_sync(0xffffffffu, hc > 1)) {
            hs = hc;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
              const int o = __shfl_up_sync(0xffffffffu, hs, dd);
              if (lane >= dd) hs += o;
            }
            hs += carry;
            carry = __shfl_sync(0xffffffffu, hs, 31);
          } else {
            hs = carry + __popc(occ & (lt | (1u << lane)));
            carry += __popc(occ);
          }
          int g0 = k, g1 = k + 1;
          int rb0 = static_cast<int>(qp[base >> 5]) + __popc(qw & lt);
          int rb1 = rb0 + rem;
          // tie groups in the row (clipped values, repeats) from the row's tie bits:
          // group bounds by bit scans; only a group crossing a 32-entry chunk walks the row
          const int prow = RI ? ri : rj;
          const uint32_t tw = stie[prow * 8 + (base >> 5)];
          const uint32_t pbit = (base > 0) ? (stie[prow * 8 + (base >> 5) - 1] >> 31) : 0u;
          const bool tied = live && ((lane > 0 ? (tw >> (lane - 1)) & 1u : pbit) || ((tw >> lane) & 1u));
          if (tied) {
            const uint32_t below = ~tw & lt;                    // positions t < lane with v_t != v_(t+1)
            const uint32_t above = ~tw & (0xffffffffu << lane);  // positions t >= lane with v_t != v_(t+1)
            bool cross = false;
            if (below) {
              g0 = base + 32 - __clz(below);
            } else {
              g0 = base;
              cross = pbit != 0;
            }
            if (above) {
              g1 = base + __ffs(above);
            } else {
              g1 = base + 32;
              cross = true;
            }
            if (cross) {
              while (g0 > 0 && sv[g0 - 1] == x) --g0;
              while (g1 < cnt && sv[g1] == x) ++g1;
            }
            rb0 = qcount(qm, qp, g0, s);
            rb1 = qcount(qm, qp, g1, s);
          }
          if (live) {
            const int eq = (g1 - g0) - (rb1 - rb0);
            const int less = RI ? n_neg + zeros + (g0 - rb0) + hs : (cnt - g1) - (s - rb1) + (mneg - hs);
            const int idx = 2 * less + eq;
            const double zv = RI ? static_cast<double>(x) : -static_cast<double>(x);
#pragma unroll
            for (int v = 0; v < NNU; ++v)
              if (NNU == 1 || v < nnu) acc[v] = fma(zv, __ldg(a.lut + v * lstride + idx), acc[v]);
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (lbp[u] >= 0) HI[lbp[u] >> 1] = 0u;  // leave the histograms zero
#pragma unroll
      for (int v = 0; v < NNU; ++v) {
        if (NNU > 1 && v >= nnu) break;
        double sum = acc[v];
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, dd);
        if (lane == 0) {
          const double val = clamp_nonneg(half_p * sum);
          ot[v * kTile * tstride] = val;
          if (isinf(val)) atomicOr(a.flag, 1);
        }
      }
      __syncwarp();
      }
      __syncwarp();
    }
    __syncthreads();
    tile_epilogue<TO>(a, otile, kTile, tstride, i0, j0, out, s_score, s_red);
    __syncthreads();
  }
  score_flush(a, s_score);
}

inline size_t gen2_smem(int W, int maxnnz, int nnu, int nwarps) {
  using namespace gmd_detail;
  using namespace gmd2_detail;
  return static_cast<size_t>(nwarps) * kGenWords2 * 8 + static_cast<size_t>(nnu) * kTile * (kTile + 1) * 8 +
         kRows * (8 + 8 + 8 + 4 + 4) + kRows * W * 4 + ((kRows * W + 1) & ~1) * 2 +
         static_cast<size_t>(kRows) * maxnnz * 4 + ((static_cast<size_t>(kRows) * maxnnz + 1) & ~size_t(1)) * 2 +
         kRows * 8 * 4 + kRows * 256 + 16;
}
void launch_gini_gen2(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                      cudaStream_t st);

inline size_t gmd_smem(int W, int maxnnz, int nnu, int nwarps) {
  using namespace gmd_detail;
  return static_cast<size_t>(nwarps) * kWarpWords * 8 + static_cast<size_t>(nnu) * kTile * (kTile + 1) * 8 +
         kRows * (8 + 8 + 8 + 4) + kRows * W * 4 + ((kRows * W + 1) & ~1) * 2 +
         static_cast<size_t>(kRows) * maxnnz * (4 + 4 + 2) + 4 + kRows * 8 * 4 + 16;  // + tie words
}

void launch_gini_gmd(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                     cudaStream_t st);
void launch_gini_gen(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                     cudaStream_t st);

}  // namespace gmds
