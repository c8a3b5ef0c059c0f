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

#include "gini_split.cuh"

namespace gmds {

struct GmdArgs {
  SplitArgs s;           // tile args, row store (masks, prefix, rowptr, vals), overflow list
  const uint16_t* pmap;  // sorted position of each nonzero (feature order)
  const float* svs;      // sorted values per row
  const double* suf;     // suffix sums of the sorted values per row
  const double* s1;      // per row: sum of values
  const double* tm;      // per row: sum_k v_(k) k
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

// #{F positions < pos} from a position mask QM[8] and its word prefix QP[8]
__device__ __forceinline__ int qcount(const uint32_t* QM, const uint32_t* QP, int pos, int s) {
  if (pos >= kMaxC) return s;
  const int w = pos >> 5;
  return static_cast<int>(QP[w]) + __popc(QM[w] & ((1u << (pos & 31)) - 1u));
}

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
  float* ssv = svals + kRows * stride;                                       // [64][stride]
  uint16_t* spm = reinterpret_cast<uint16_t*>(ssv + kRows * stride);         // [64][stride]
  const float* gv = static_cast<const float*>(sa.vals);
  const double h = 0.5 * static_cast<double>(d + 1);
  const int tstride = kTile + 1;

  for (int64_t t = a.tile_begin + blockIdx.x; t < a.tile_end; t += gridDim.x) {
    int64_t I, J;
    decode_tile(t, a.nbt, I, J);
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
          ssv[r * stride + k] = ga.svs[b + k];
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
#pragma unroll
      for (int u = 0; u < 2; ++u) {
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
        const int lb = lower_count(ssv + (pos ? ri : rj) * stride, n, code);  // #{row values < |zz|}
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

inline size_t gmd_smem(int W, int maxnnz, int nnu, int nwarps) {
  using namespace gmd_detail;
  return static_cast<size_t>(nwarps) * kWarpWords * 8 + static_cast<size_t>(nnu) * kTile * (kTile + 1) * 8 +
         kRows * (8 + 8 + 8 + 4) + kRows * W * 4 + ((kRows * W + 1) & ~1) * 2 +
         static_cast<size_t>(kRows) * maxnnz * (4 + 4 + 2) + 16;
}

void launch_gini_gmd(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                     cudaStream_t st);

}  // namespace gmds
