// K3 stress-pass kernel template (instantiated in stress_pass_*.cu).
// K3 stress passes over the packed upper-triangle D (sm_100a, HBM-bound).
//
// One pass streams every stored D_ij (i < j) exactly once and, at the same
// configuration Y, produces the loss partials of the chosen kind and (GRAD
// passes) the per-row sums  g_i = sum_j c_ij (y_i - y_j)  with the kind's
// weight c_ij (embed.cpp:164-212 gradient_value; embed.cpp:276-294
// guttman_transform):
//   kruskal  c = -e/dist             (x 1/(KS*den) after the reduction)
//   huber    c = -clamp(e,-d,d)/dist
//   sammon   c = -e/(D*dist)          (x 2/sum(D) after the reduction)
//   smacof   c = -2 w e/dist
//   guttman  c =  w D/dist            (X+ = (1/n) g, the uniform-weight transform)
// with e = D - dist, dist = |y_i - y_j|; pairs with dist <= 0 add no gradient
// (embed.cpp:187, 283).  LOSS passes evaluate up to 4 candidate
// configurations at once (the Armijo trial points step, step/2, ...).
//
// Work split: a CTA takes a chunk of up to kChunk consecutive 128x128 blocks
// of one block-row I; 256 threads, each an 8x8 micro-tile of pairs.  Row
// sums accumulate in registers across the chunk; column sums are reduced in
// shared memory per block.  Both leave as per-chunk / per-block partials
// that reduce_rows_kernel sums in a fixed order: results are bit-identical
// run to run (no floating-point atomics).
#pragma once

#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "stress.cuh"

namespace gmds {

namespace stress_detail {

template <typename TD>
struct MathOf {
  using type = double;
};
template <>
struct MathOf<float> {
  using type = float;
};

constexpr int kMT = 8;     // micro-tile edge
constexpr int kTG = 16;    // thread grid edge (kPT / kMT)
constexpr int kThreads = kTG * kTG;

__device__ __forceinline__ int64_t blk_index(int64_t I, int64_t J, int64_t nb) { return I * nb - (I * (I - 1)) / 2 + (J - I); }

template <typename M>
struct PairTerms {
  M term;  // loss contribution
  M c;     // gradient weight c_ij (already divided by dist; 0 when dist == 0)
};

// dist and 1/dist of a squared distance.  fp64 path: IEEE sqrt and division
// (parity mode).  fp32 path: one MUFU.RSQ (rsqrtf, <= 2 ulp) gives both, so a
// pair costs one XU op per configuration and no division.
__device__ __forceinline__ void dist_inv(double d2, double& dist, double& inv) {
  dist = sqrt(d2);
  inv = (dist > 0.0) ? 1.0 / dist : 0.0;
}
__device__ __forceinline__ void dist_inv(float d2, float& dist, float& inv) {
  const float r = rsqrtf(d2);
  inv = (d2 > 0.f) ? r : 0.f;
  dist = d2 * inv;
}

// invD = 1/D (Sammon only; computed once per pair, shared by all candidates).
template <int KIND, typename M>
__device__ __forceinline__ PairTerms<M> pair_terms(M Dv, M invD, M dist, M inv, M w, M delta) {
  const M e = Dv - dist;
  PairTerms<M> r;
  switch (KIND) {
    case kKruskal:
      r.term = e * e;
      r.c = -e * inv;
      break;
    case kHuber: {
      const M ae = fabs(e);
      r.term = (ae <= delta) ? M(0.5) * e * e : delta * (ae - M(0.5) * delta);
      r.c = -fmin(fmax(e, -delta), delta) * inv;
      break;
    }
    case kSammon:
      r.term = e * e * invD;
      r.c = -e * invD * inv;
      break;
    case kSmacof:
      r.term = w * e * e;
      r.c = M(-2) * w * e * inv;
      break;
    default:  // kGuttman: loss is the smacof loss at the same Z
      r.term = w * e * e;
      r.c = w * Dv * inv;
      break;
  }
  return r;
}

// Shared-memory slot of block row r (0..127): rows are stored [y][tj] so the
// 16 tj-threads of a half-warp read 16 different banks (r = tj * 8 + y).
__device__ __forceinline__ int yslot(int r) { return (r % kMT) * kTG + r / kMT; }

}  // namespace stress_detail
using namespace stress_detail;

// ---------------------------------------------------------------------------
// MT: arithmetic type (fp64 for fp64 storage; fp32 storage takes fp32 math in the
// TMA kernels and fp64 math in the "precise" loss pass that resolves tiny changes)
template <int Q, typename TD, bool GRAD, int KIND, typename MT = typename MathOf<TD>::type>
__global__ void __launch_bounds__(kThreads) stress_pass_kernel(PassArgs a) {
  using M = MT;
  constexpr int NCM = GRAD ? 1 : kMaxCand;
  __shared__ M sYi[NCM][kPT][Q];
  __shared__ M sYj[NCM][kPT][Q];  // [yslot(r)]
  __shared__ double sRed[GRAD ? kTG * kPT : 1];
  __shared__ double sLoss[kThreads / 32][kMaxCand];
  // row sums of the chunk (fixed order: x rows reduced across the half-warp, then += per block)
  __shared__ double sRowTot[GRAD ? kPT * Q : 1];

  const int tid = threadIdx.x;
  const int ti = tid / kTG, tj = tid % kTG;
  const int64_t chunk = blockIdx.x;
  const int64_t I = a.chunk_I[chunk];
  const int64_t J0 = a.chunk_J0[chunk];
  const int64_t J1 = min(J0 + a.chunk_len, a.nb);
  const int nc = GRAD ? 1 : a.ncand;
  const TD* __restrict__ D = static_cast<const TD*>(a.D);
  const TD* __restrict__ W = static_cast<const TD*>(a.W);
  const M delta = static_cast<M>(a.huber_delta);

  for (int e = tid; e < nc * kPT * Q; e += kThreads) {
    const int c = e / (kPT * Q), r = (e / Q) % kPT, k = e % Q;
    const int64_t i = I * kPT + r;
    sYi[c][r][k] = (i < a.n) ? static_cast<M>(a.Y[c][i * Q + k]) : M(0);
  }
  if constexpr (GRAD) {
    for (int e = tid; e < kPT * Q; e += kThreads) sRowTot[e] = 0.0;
  }
  double lossacc[NCM];
#pragma unroll
  for (int c = 0; c < NCM; ++c) lossacc[c] = 0.0;

  for (int64_t J = J0; J < J1; ++J) {
    __syncthreads();  // previous block's sYj / sRed consumers are done
    for (int e = tid; e < nc * kPT * Q; e += kThreads) {
      const int c = e / (kPT * Q), r = (e / Q) % kPT, k = e % Q;
      const int64_t j = J * kPT + r;
      sYj[c][yslot(r)][k] = (j < a.n) ? static_cast<M>(a.Y[c][j * Q + k]) : M(0);
    }
    __syncthreads();
    const int64_t blk = blk_index(I, J, a.nb);
    const TD* Db = D + blk * (kPT * kPT);
    const TD* Wb = W ? W + blk * (kPT * kPT) : nullptr;
    M colacc[GRAD ? kMT : 1][Q];
    if constexpr (GRAD) {
#pragma unroll
      for (int y = 0; y < kMT; ++y)
#pragma unroll
        for (int k = 0; k < Q; ++k) colacc[y][k] = M(0);
    }
    const bool diag = (I == J);
#pragma unroll 1
    for (int x = 0; x < kMT; ++x) {
      const int ri = ti * kMT + x;
      M rowacc[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) rowacc[k] = M(0);
      M lossrow[NCM];
#pragma unroll
      for (int c = 0; c < NCM; ++c) lossrow[c] = M(0);
      TD dv[kMT];
      const TD* drow = Db + ri * kPT + tj * kMT;
      if constexpr (sizeof(TD) == 4) {
        const float4 v0 = __ldcs(reinterpret_cast<const float4*>(drow));
        const float4 v1 = __ldcs(reinterpret_cast<const float4*>(drow + 4));
        dv[0] = v0.x, dv[1] = v0.y, dv[2] = v0.z, dv[3] = v0.w;
        dv[4] = v1.x, dv[5] = v1.y, dv[6] = v1.z, dv[7] = v1.w;
      } else {
#pragma unroll
        for (int y = 0; y < kMT; y += 2) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(drow + y));
          dv[y] = v.x, dv[y + 1] = v.y;
        }
      }
      TD wv[kMT];
#pragma unroll
      for (int y = 0; y < kMT; ++y) wv[y] = Wb ? Wb[ri * kPT + tj * kMT + y] : TD(1);
#pragma unroll
      for (int y = 0; y < kMT; ++y) {
        const int rj = tj * kMT + y;
        const int64_t j = J * kPT + rj;
        const bool valid = (j < a.n) && (!diag || ri < rj);
        const M Dv = static_cast<M>(dv[y]);
        const M invD = (KIND == kSammon && valid) ? M(1) / Dv : M(0);
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
          if (c >= nc) break;
          M dy[Q];
          M d2 = M(0);
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            dy[k] = sYi[c][ri][k] - sYj[c][y * kTG + tj][k];
            d2 = fma(dy[k], dy[k], d2);
          }
          M dist, inv;
          dist_inv(d2, dist, inv);
          const PairTerms<M> t = pair_terms<KIND, M>(Dv, invD, dist, inv, static_cast<M>(wv[y]), delta);
          lossrow[c] += valid ? t.term : M(0);
          if constexpr (GRAD) {
            const M cc = valid ? t.c : M(0);
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              const M g = cc * dy[k];
              rowacc[k] += g;
              colacc[y][k] -= g;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCM; ++c) lossacc[c] += static_cast<double>(lossrow[c]);
      if constexpr (GRAD) {
        // the 16 tj-threads of row ri share a half-warp: xor-tree in a fixed order
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          double v = static_cast<double>(rowacc[k]);
#pragma unroll
          for (int m = 8; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
          if (tj == 0) sRowTot[ri * Q + k] += v;
        }
      }
    }
    if constexpr (GRAD) {
      // column partials of this block: reduce the 16 ti-threads per column in a fixed order
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        if (k > 0) __syncthreads();
#pragma unroll
        for (int y = 0; y < kMT; ++y) sRed[ti * kPT + tj * kMT + y] = static_cast<double>(colacc[y][k]);
        __syncthreads();
        if (tid < kPT) {
          double s = 0.0;
          for (int t = 0; t < kTG; ++t) s += sRed[t * kPT + tid];
          a.colpart[(blk * kPT + tid) * Q + k] = s;
        }
      }
    }
  }
  if constexpr (GRAD) {
    __syncthreads();
    for (int e = tid; e < kPT * Q; e += kThreads) a.rowpart[chunk * (kPT * Q) + e] = sRowTot[e];
  }
  // loss partial of the chunk (fixed-order tree)
#pragma unroll
  for (int c = 0; c < NCM; ++c) {
    double v = lossacc[c];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((tid & 31) == 0) sLoss[tid >> 5][c] = v;
  }
  __syncthreads();
  if (tid < nc) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += sLoss[w][tid];
    a.losspart[chunk * kMaxCand + tid] = s;
  }
}

template <typename TD, bool GRAD>
void launch_pass_td(const PassArgs& a, int Q, cudaStream_t st);

#define GMDS_PASS_KIND(QQ, KK) \
  case KK: stress_pass_kernel<QQ, TD, GRAD, KK><<<g, kThreads, 0, st>>>(a); break;
#define GMDS_PASS_Q(QQ)                                                                     \
  case QQ:                                                                                  \
    switch (a.kind) {                                                                       \
      GMDS_PASS_KIND(QQ, kKruskal) GMDS_PASS_KIND(QQ, kHuber) GMDS_PASS_KIND(QQ, kSammon)   \
      GMDS_PASS_KIND(QQ, kSmacof) GMDS_PASS_KIND(QQ, kGuttman)                              \
      default: fail(GMDS_ERROR, "stress pass: bad kind");                                   \
    }                                                                                       \
    break;
#define GMDS_INSTANTIATE_PASS(TDT, GR)                                                      \
  template <>                                                                               \
  void launch_pass_td<TDT, GR>(const PassArgs& a, int Q, cudaStream_t st) {                  \
    using TD = TDT;                                                                         \
    constexpr bool GRAD = GR;                                                               \
    const unsigned g = static_cast<unsigned>(a.nchunks);                                    \
    switch (Q) {                                                                            \
      GMDS_PASS_Q(1) GMDS_PASS_Q(2) GMDS_PASS_Q(3) GMDS_PASS_Q(4)                           \
      default: fail(GMDS_ERROR, "stress pass: unsupported padded dimension");               \
    }                                                                                       \
  }

// fp32 storage, fp64 arithmetic, loss only (Engine::loss_raw_precise)
#define GMDS_PRECISE_KIND(QQ, KK) \
  case KK: stress_pass_kernel<QQ, float, false, KK, double><<<g, kThreads, 0, st>>>(a); break;
#define GMDS_PRECISE_Q(QQ)                                                                      \
  case QQ:                                                                                      \
    switch (a.kind) {                                                                           \
      GMDS_PRECISE_KIND(QQ, kKruskal) GMDS_PRECISE_KIND(QQ, kHuber) GMDS_PRECISE_KIND(QQ, kSammon) \
      GMDS_PRECISE_KIND(QQ, kSmacof) GMDS_PRECISE_KIND(QQ, kGuttman)                            \
      default: fail(GMDS_ERROR, "stress pass: bad kind");                                       \
    }                                                                                           \
    break;

}  // namespace gmds
