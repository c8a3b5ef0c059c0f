// Support kernels of the stress path (generic rows pass, reductions, trial
// points) and the pass dispatcher.  The fused pass itself is in
// stress_pass.cuh.
#include "stress_pass.cuh"

namespace gmds {

// Generic (any q <= 64) loss / gradient pass: thread per row i, sequential
// over j.  Used for q > 4 (embedding dimensions the fused pass does not
// instantiate).  Row i's gradient is the full sum over j != i.
template <typename TD>
__global__ void stress_rows_kernel(PassArgs a, int q, int grad) {
  using M = typename MathOf<TD>::type;
  const TD* __restrict__ D = static_cast<const TD*>(a.D);
  const TD* __restrict__ W = static_cast<const TD*>(a.W);
  const M delta = static_cast<M>(a.huber_delta);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double loss[kMaxCand] = {0, 0, 0, 0};
    double g[64];
    for (int k = 0; k < (grad ? q : 0); ++k) g[k] = 0.0;
    const int nc = grad ? 1 : a.ncand;
    for (int64_t j = 0; j < a.n; ++j) {
      if (j == i) continue;
      const int64_t lo = min(i, j), hi = max(i, j);
      const int64_t off = packed_offset(lo, hi, a.nb);
      const M Dv = static_cast<M>(D[off]);
      const M wv = W ? static_cast<M>(W[off]) : M(1);
      for (int c = 0; c < nc; ++c) {
        M d2 = 0;
        for (int k = 0; k < q; ++k) {
          const M dy = static_cast<M>(a.Y[c][i * q + k]) - static_cast<M>(a.Y[c][j * q + k]);
          d2 = fma(dy, dy, d2);
        }
        M dist, inv;
        dist_inv(d2, dist, inv);
        const M invD = (a.kind == kSammon) ? M(1) / Dv : M(0);
        PairTerms<M> t;
        switch (a.kind) {
          case kKruskal: t = pair_terms<kKruskal, M>(Dv, invD, dist, inv, wv, delta); break;
          case kHuber: t = pair_terms<kHuber, M>(Dv, invD, dist, inv, wv, delta); break;
          case kSammon: t = pair_terms<kSammon, M>(Dv, invD, dist, inv, wv, delta); break;
          case kSmacof: t = pair_terms<kSmacof, M>(Dv, invD, dist, inv, wv, delta); break;
          default: t = pair_terms<kGuttman, M>(Dv, invD, dist, inv, wv, delta); break;
        }
        if (j > i) loss[c] += static_cast<double>(t.term);  // each pair once
        if (grad)
          for (int k = 0; k < q; ++k)
            g[k] += static_cast<double>(t.c * (static_cast<M>(a.Y[0][i * q + k]) - static_cast<M>(a.Y[0][j * q + k])));
      }
    }
    if (grad)
      for (int k = 0; k < q; ++k) a.rowpart[i * q + k] = g[k];
    for (int c = 0; c < nc; ++c) a.losspart[i * kMaxCand + c] = loss[c];
  }
}

// Stage 2: out[r][k] = sum over strip-R chunks of rowpart + sum over I <= R of colpart(I, R).
// Eight lanes per output (strided over the partial list), combined by a fixed
// xor-tree: deterministic, and eight times the loads in flight.
// Strided partial sums over VT virtual threads then a pairwise tree -- the
// exact order of a VT-thread CTA doing `for k = t; k < count; k += VT`
// followed by `red[t] += red[t + w]` (VT = 256: finish_grad_kernel; VT =
// 1024: sum_parts_kernel), computed by a 256-thread CTA: every caller of
// the same (part, count, stride, slot, VT) gets the same bits.
// (Any blockDim >= 256: threads beyond 256 only take part in the barriers.)
template <int VT>
__device__ double tree_sum(const double* __restrict__ part, int64_t count, int stride, int slot, double* red) {
  constexpr int per = VT / 256;
  const bool act = threadIdx.x < 256;
  if (act) {
#pragma unroll
    for (int u = 0; u < per; ++u) {
      const int t = threadIdx.x + 256 * u;
      double r = 0.0;
      for (int64_t k = t; k < count; k += VT) r += part[k * stride + slot];
      red[t] = r;
    }
  }
  __syncthreads();
  for (int w = VT / 2; w > 0; w >>= 1) {
    if (act) {
#pragma unroll
      for (int u = 0; u < per; ++u) {
        const int t = threadIdx.x + 256 * u;
        if (t < w) red[t] += red[t + w];
      }
    }
    __syncthreads();
  }
  const double v = red[0];
  __syncthreads();
  return v;
}

// The device loop's three loss sums of a fused pass (trial slots 0 and 1 as
// sum_parts_kernel, slot 0 as finish_grad_kernel), by one extra CTA of the
// reduction launch that follows the pass: out[0..2].
__device__ void gd_pass_sums(const double* __restrict__ losspart, int64_t nparts, int stride, double* out,
                             int which) {  // one sum per CTA: 0, 1 = trial slots, 2 = slot 0 (finish order)
  __shared__ double red[1024];
  const double v = (which == 2) ? tree_sum<256>(losspart, nparts, stride, 0, red)
                                : tree_sum<1024>(losspart, nparts, stride, which, red);
  if (threadIdx.x == 0) out[which] = v;
}

template <typename TP>
__global__ void reduce_rows_kernel(const TP* __restrict__ rowpart, const TP* __restrict__ colpart,
                                   const int64_t* __restrict__ strip_first, int64_t n, int64_t nb, int Q,
                                   double* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int sub = static_cast<int>(t & 7);
  const int64_t e = t >> 3;
  const bool live = e < n * Q;
  double s = 0.0;
  if (live) {
    const int64_t r = e / Q;
    const int k = static_cast<int>(e % Q);
    const int64_t R = r / kPT, rr = r % kPT;
    const int64_t c0 = strip_first[R], c1 = strip_first[R + 1];
    for (int64_t c = c0 + sub; c < c1; c += 8) s += static_cast<double>(rowpart[(c * kPT + rr) * Q + k]);
    for (int64_t I = sub; I <= R; I += 8) s += static_cast<double>(colpart[(blk_index(I, R, nb) * kPT + rr) * Q + k]);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  if (live && sub == 0) out[e] = s;
}

// Two-level version of the same sums, bandwidth-friendly: CTA (R, s) adds
// group s of strip R's terms (its chunks' row partials, then the column
// partials of blocks (I, R), I <= R) for all 128 x Q entries at once -- every
// term is a contiguous 128 x Q run, read coalesced -- and combine_kernel adds
// the kRedGroups group sums of each entry in order.  Fixed order throughout.
// TP: the partials' type (fp32 from the TMA passes, fp64 from the fp64 pass).
#ifndef GMDS_RED_GROUPS
#define GMDS_RED_GROUPS 8
#endif
#ifndef GMDS_RED_UNROLL
#define GMDS_RED_UNROLL 4
#endif
constexpr int kRedGroups = GMDS_RED_GROUPS;
constexpr int kRedUnroll = GMDS_RED_UNROLL;
template <typename TP>
__global__ void reduce_groups_kernel(const TP* __restrict__ rowpart, const TP* __restrict__ colpart,
                                     const int64_t* __restrict__ strip_first, int64_t nb, int Q,
                                     double* __restrict__ gpart, const int* __restrict__ halt,
                                     const double* __restrict__ losspart, int64_t nparts, int lstride,
                                     double* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  if (halt && *halt) return;
  if (blockIdx.x >= nb * kRedGroups) {  // the extra CTAs (device loop): the pass's loss sums
    gd_pass_sums(losspart, nparts, lstride, sums, static_cast<int>(blockIdx.x - nb * kRedGroups));
    return;
  }
  const int64_t R = blockIdx.x / kRedGroups;
  const int s = blockIdx.x % kRedGroups;
  const int64_t c0 = strip_first[R], nrow = strip_first[R + 1] - c0;
  const int64_t T = nrow + R + 1;
  const int64_t t0 = T * s / kRedGroups, t1 = T * (s + 1) / kRedGroups;
  const int e = threadIdx.x;  // (rr, k), < 128 Q
  const int64_t run = static_cast<int64_t>(kPT) * Q;
  double acc = 0.0;
  int64_t t = t0;
  for (; t + kRedUnroll <= t1; t += kRedUnroll) {  // kRedUnroll loads in flight, added in order
    TP v[kRedUnroll];
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) {
      const int64_t tt = t + u;
      v[u] = ((tt < nrow) ? rowpart + (c0 + tt) * run : colpart + blk_index(tt - nrow, R, nb) * run)[e];
    }
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) acc += static_cast<double>(v[u]);
  }
  for (; t < t1; ++t) {
    const TP* src = (t < nrow) ? rowpart + (c0 + t) * run : colpart + blk_index(t - nrow, R, nb) * run;
    acc += static_cast<double>(src[e]);
  }
  gpart[(R * kRedGroups + s) * run + e] = acc;
}
__global__ void combine_kernel(const double* __restrict__ gpart, int64_t n, int Q, double* __restrict__ out,
                               const int* __restrict__ halt) {
  pdl_wait();
  pdl_trigger();
  if (halt && *halt) return;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * Q) return;
  const int64_t r = idx / Q, R = r / kPT;
  const int64_t e = (r % kPT) * Q + idx % Q, run = static_cast<int64_t>(kPT) * Q;
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < kRedGroups; ++s) acc += gpart[(R * kRedGroups + s) * run + e];
  out[idx] = acc;
}

// Row-sharded device loop (gmds_minimize_stress_sharded): this rank's gradient groups
// summed into xred[0, nQ) (combine_kernel's order) and its pass's loss-slot sums 0-2
// into xred[nQ, nQ + 3) (tree_sum<1024>, gd_pass_sums' order) -- the payload of the
// all-reduce that follows.  Once the loop has stopped the payload is zeros, so that
// all-reduce (enqueued ahead with the batch) cannot re-add a stale buffer.
__global__ void shard_collect_kernel(const double* __restrict__ gpart, int64_t n, int Q,
                                     const double* __restrict__ losspart, int64_t nparts, int stride,
                                     double* __restrict__ xred, const int* __restrict__ halt) {
  pdl_wait();
  pdl_trigger();
  const bool stopped = halt && *halt;
  const int64_t m = n * Q;
  if (blockIdx.x == gridDim.x - 1) {
    __shared__ double red[1024];
    for (int c = 0; c < 3; ++c) {  // trial slots (or, after a tiny-phase pass, difference slots 0-2)
      const double v = stopped ? 0.0 : tree_sum<1024>(losspart, nparts, stride, c, red);
      if (threadIdx.x == 0) xred[m + c] = v;
    }
    return;
  }
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= m) return;
  if (stopped) {
    xred[idx] = 0.0;
    return;
  }
  const int64_t r = idx / Q, R = r / kPT;
  const int64_t e = (r % kPT) * Q + idx % Q, run = static_cast<int64_t>(kPT) * Q;
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < kRedGroups; ++s) acc += gpart[(R * kRedGroups + s) * run + e];
  xred[idx] = acc;
}

// Deterministic single-CTA sums: out[c] = sum_k part[k*stride + c] for c < m.
__global__ void sum_parts_kernel(const double* __restrict__ part, int64_t count, int stride, int m,
                                 double* __restrict__ out) {
  __shared__ double red[1024];
  for (int c = 0; c < m; ++c) {
    double s = 0.0;
    for (int64_t k = threadIdx.x; k < count; k += blockDim.x) s += part[k * stride + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = red[0];
    __syncthreads();
  }
}

// g *= scale (in place); per-block partial sums of g^2 (fixed order), then
// sum_parts_kernel adds the block partials: deterministic.
__global__ void scale_sqnorm_kernel(double* __restrict__ g, int64_t m, double scale, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = g[k] * scale;
    g[k] = v;
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// One kernel between the gradient pass and the first trial pass: every block
// sums the pass's loss partials (same fixed order in every block) to the raw
// loss at Y, derives the kind's gradient scale exactly as the host would
// (embed.cpp:179-181 for Kruskal; 2/sum(D) for Sammon; 1 otherwise), scales
// its slice of g, writes the two trial points Y - s0 g and Y - s1 g, and leaves
// a per-block partial of |g|^2 (summed in order on the host).
// the kind's gradient scale at a raw loss (embed.cpp:179-181 Kruskal, 2/sum(D) Sammon, 1 otherwise)
__device__ __forceinline__ double grad_scale(int kind, double raw, double sum_sq, double sum) {
  if (kind == kKruskal) {
    const double ks = sqrt(raw / sum_sq);
    return (ks <= 0.0) ? 0.0 : 1.0 / (ks * sum_sq);
  }
  if (kind == kSammon) return 2.0 * (1.0 / sum);
  return 1.0;
}

// g *= scale over this grid's slice, trial points T0/T1 = Y - s g, |g|^2 block partial.
// Y and T0 may alias (the device loop's accepted point): each element is read then written
// by one thread.
__device__ void finish_body(double scale, double* __restrict__ g, const double* Y, int64_t m, double s0,
                            double s1, double* T0, double* __restrict__ T1, double* __restrict__ sqpart,
                            double* red, double* Ycopy = nullptr, const double* gsrc = nullptr) {
  double sq = 0.0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = (gsrc ? gsrc[k] : g[k]) * scale;
    g[k] = v;
    sq += v * v;
    const double y = Y[k];
    if (Ycopy) Ycopy[k] = y;
    T0[k] = y - s0 * v;
    T1[k] = y - s1 * v;
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) sqpart[blockIdx.x] = red[0];
}

__global__ void finish_grad_kernel(const double* __restrict__ losspart, int64_t nparts, int stride, int kind,
                                   double sum_sq, double sum, double* __restrict__ g, const double* __restrict__ Y,
                                   int64_t m, double s0, double s1, double* __restrict__ T0, double* __restrict__ T1,
                                   double* __restrict__ sqpart, double* __restrict__ raw_out,
                                   const double* __restrict__ raw_in) {
  __shared__ double red[256];
  // the raw loss at Y: this device's pass partials, or (row-sharded) the all-reduced value
  const double raw = raw_in ? *raw_in : tree_sum<256>(losspart, nparts, stride, 0, red);
  const double scale = grad_scale(kind, raw, sum_sq, sum);
  if (blockIdx.x == 0 && threadIdx.x == 0) *raw_out = raw;
  finish_body(scale, g, Y, m, s0, s1, T0, T1, sqpart, red);
}

// Device-resident gradient descent (fp32 storage, fused passes): one launch
// per iteration decides the previous fused pass exactly as the host loop
// (fit.cu gradient_descent: Armijo in the reference's order, embed.cpp:236-
// 262) and, in the common case -- the trial in slot 0 accepted, so its
// gradient is already in gnext -- moves Y to it, records the history, and
// forms the next trial pair.  Every CTA evaluates the same decision on the
// same bits (no grid sync); the state is double-buffered by iteration
// parity.  Anything else (slot 1 accepted, no trial accepted, |g|^2 <= 0)
// hands the iteration back to the host (stop = 2) untouched.
__global__ void gd_step_kernel(GdState* st, int par, const double* __restrict__ losspart, int64_t nparts,
                               int stride, const double* __restrict__ sqprev, int nsq, double* __restrict__ sqnext,
                               int kind, double sum_sq, double sum, double* __restrict__ Y, double* cand0,
                               double* __restrict__ cand1, double* __restrict__ gnext,
                               const double* __restrict__ gpart, int Q,
                               double* __restrict__ graw, int64_t m, double* __restrict__ history, int max_iters,
                               double rel_tol, const double* __restrict__ pre, double precise_rel, int phase,
                               const double* __restrict__ xred, const double* __restrict__ dsum, int tiny_ok,
                               int solo_ok, int ondev) {
  // xred (row-sharded loop): the all-reduced [gradient at cand0 (n Q) | trial loss sums (2)]
  // of the last pass; dsum: the all-reduced sums of a difference pass (slots 0, 1, 2)
  pdl_wait();
  pdl_trigger();
  __shared__ double red[1024];
  __shared__ double sgsq;
  const GdState S = st[par];
  GdState* N = st + (par ^ 1);
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  auto publish = [&](GdState R) {  // the next passes' halt flags follow stop / tiny
    R.halt_fused = (R.stop != 0 || R.tiny != 0) ? 1 : 0;
    R.halt_grad = (R.stop != 0 || R.tiny == 0) ? 1 : 0;
    *N = R;
  };
  if (S.stop || (phase == 1 && !S.pending)) {
    if (lead) publish(S);
    return;
  }
  if (S.fix) {
    // The last pass was the gradient pass at Y (the accepted slot-1 point): what the host's
    // next iteration does first (grad_raw, then finish_grad): scale from the raw loss at Y,
    // the scaled gradient, the trial pair of iteration S.it, |g|^2 partials.  No decision.
    GdState R = S;
    R.fix = 0;
    if (S.init) {  // the loss before the loop (embed.cpp:226): the host's order of the same sums (sum_parts_kernel)
      const double raw0 = xred ? xred[m] : (pre ? pre[0] : tree_sum<1024>(losspart, nparts, stride, 0, red));
      R.f = (kind == kKruskal) ? sqrt(__ddiv_rn(raw0, sum_sq))
                               : ((kind == kSammon) ? __dmul_rn(__ddiv_rn(1.0, sum), raw0) : raw0);
      R.init = 0;
      if (lead) history[S.it] = R.f;
    }
    if (lead) publish(R);
    const double raw = xred ? xred[m] : (pre ? pre[2] : tree_sum<256>(losspart, nparts, stride, 0, red));
    const double scale = grad_scale(kind, raw, sum_sq, sum);
    const double s0 = (S.pred == 0) ? S.step : __dmul_rn(S.step, 0.5);
    const double s1 = (S.pred == 0) ? __dmul_rn(S.step, 0.5) : S.step;
    if (xred) {
      for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
           k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        gnext[k] = xred[k];
    } else {
      const int64_t run = static_cast<int64_t>(kPT) * Q;
      for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
           k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = k / Q, Rr = r / kPT;
        const int64_t e = (r % kPT) * Q + k % Q;
        double a = 0.0;
#pragma unroll
        for (int g = 0; g < kRedGroups; ++g) a += gpart[(Rr * kRedGroups + g) * run + e];
        gnext[k] = a;
      }
    }
    finish_body(scale, graw, Y, m, s0, s1, cand0, cand1, sqnext, red, nullptr, gnext);
    return;
  }
  // A decision on difference sums: phase 1 (a difference pass ran for a pending decision)
  // or, in the tiny phase, phase 0 itself (the last pass was the difference + gradient
  // pass).  Its columns 0, 1 hold the raw losses at the two trials and column 2 the raw
  // loss at Y; the loss at Y is re-based on it (history too), as the host path does.
  const bool diffdec = (phase == 1) || S.tiny != 0;
  double fY = S.f;
  if (phase == 1) pre = nullptr;
  // the pass's loss sums: from the reduction launch's extra CTA when it ran, else here (same order)
  if (xred && phase == 0) pre = xred + m;
  const double t0 = (xred && phase == 1) ? dsum[0] : (pre ? pre[0] : tree_sum<1024>(losspart, nparts, stride, 0, red));
  const double t1 = (xred && phase == 1) ? dsum[1] : (pre ? pre[1] : tree_sum<1024>(losspart, nparts, stride, 1, red));
  // |g|^2 = the finish partials added in order (as the host does); staged through
  // shared memory so the serial adds do not wait on 148 serial L2 loads
  for (int b = threadIdx.x; b < nsq; b += blockDim.x) red[b] = sqprev[b];
  __syncthreads();
  if (threadIdx.x == 0) {
    double gq = 0.0;
    for (int b = 0; b < nsq; ++b) gq += red[b];
    sgsq = gq;
  }
  __syncthreads();
  const double gsq = sgsq;
  GdState R = S;
  R.t0 = t0;
  R.t1 = t1;
  R.gsq = gsq;
  R.solo = 0;
  R.solo_miss = 0;
  R.streak = 0;  // (kept only by the accepting path below)
  R.rt = 0;
  R.halv = 0;
  // the pass behind this decision was a solo pass: t1 is not there (see GdState::solo)
  const bool solo = S.solo != 0 && phase == 0 && S.tiny == 0;
  const bool rt = S.rt != 0 && !diffdec;  // a re-trial decision: natural slot order, no fp32 re-evaluation
  auto loss_of = [&](double raw) {
    if (kind == kKruskal) return sqrt(__ddiv_rn(raw, sum_sq));
    if (kind == kSammon) return __dmul_rn(__ddiv_rn(1.0, sum), raw);
    return raw;
  };
  if (diffdec) {
    const double raw_y = xred ? (phase == 1 ? dsum[2] : xred[m + 2]) : tree_sum<1024>(losspart, nparts, stride, 2, red);
    fY = loss_of(raw_y);
    R.f = fY;
    R.pending = 0;
    if (lead) history[S.it] = fY;
  }
  int acc_c = -1;
  double f_new = fY, sc_acc = 0.0;
  // phase 0, both trials within fp32 storage's resolution of f: Kruskal defers to a
  // difference pass (phase 1 decides); other kinds hand the iteration to the host
  const double tol = precise_rel * fabs(fY);
  // ... or a tested trial whose Armijo margin is inside that resolution (the decision
  // could flip against the reference's fp64 sums): the same deferral (armijo_unresolved)
  // the raw gradient at cand0 (combine_kernel's sums, in its order) -> gnext
  auto combine = [&]() {
    if (xred) {  // row-sharded: already combined and all-reduced
      for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
           k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        gnext[k] = xred[k];
      return;
    }
    const int64_t run = static_cast<int64_t>(kPT) * Q;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t r = k / Q, Rr = r / kPT;
      const int64_t e = (r % kPT) * Q + k % Q;
      double a = 0.0;
#pragma unroll
      for (int g = 0; g < kRedGroups; ++g) a += gpart[(Rr * kRedGroups + g) * run + e];
      gnext[k] = a;
    }
  };
  // solo (slot 0 = the full step, tested first): the first clause needs t1 when t0 is within
  // tol of f, and the second needs it when the full step is rejected outside tol -- both are
  // misses (below); otherwise the outcome is the two-trial one, bit for bit
  bool solo_missed = false;
  if (solo) {
    const double thr = __dsub_rn(fY, __dmul_rn(__dmul_rn(1e-4, S.step), gsq));
    const double f0 = loss_of(t0);
    const bool near_f = precise_rel > 0.0 && fabs(f0 - fY) <= tol;
    const bool near_thr = precise_rel > 0.0 && fabs(__dsub_rn(f0, thr)) <= tol;
    solo_missed = near_f || (!near_thr && !(f0 <= thr)) || !(gsq > 0.0);
  }
  if (solo_missed && ondev) {
    // the same trial pair again through the two-trial fused pass (this unit's); |g|^2 carried over
    R.tiny = 0;
    R.nextra = S.nextra + 1;
    if (lead) publish(R);
    if (threadIdx.x == 0 && static_cast<int>(blockIdx.x) < nsq) sqnext[blockIdx.x] = sqprev[blockIdx.x];
    return;
  }
  if (solo_missed) {  // the host evaluates the loss at cand1 and decides (stop = 2)
    R.stop = 2;
    R.tiny = 0;
    R.solo_miss = 1;
    if (lead) publish(R);
    combine();
    return;
  }
  const bool unresolved =
      !diffdec && !rt && precise_rel > 0.0 &&
      (solo ? armijo_unresolved(fY, S.step, gsq, loss_of(t0), loss_of(t0), tol)
            : ((fabs(loss_of(t0) - fY) <= tol && fabs(loss_of(t1) - fY) <= tol) ||
               armijo_unresolved(fY, S.step, gsq, loss_of(S.pred == 0 ? t0 : t1), loss_of(S.pred == 0 ? t1 : t0),
                                 tol)));
  if (unresolved && kind == kKruskal) {
    R.pending = 1;
    R.single = 0;
    R.ndiff = S.ndiff + 1;
    if (lead) publish(R);
    return;
  }
  if (gsq > 0.0 && !unresolved) {
    for (int c = 0; c < (solo ? 1 : 2); ++c) {  // step, then step/2 (the reference's order)
      const double sc = (c == 0) ? S.step : __dmul_rn(S.step, 0.5);
      const int slot = (rt || S.pred == 0) ? c : 1 - c;
      const double fc = loss_of(slot == 0 ? t0 : t1);
      if (fc <= __dsub_rn(fY, __dmul_rn(__dmul_rn(1e-4, sc), gsq))) {
        acc_c = c;
        f_new = fc;
        sc_acc = sc;
        break;
      }
    }
  }
  const int acc_slot = (acc_c < 0) ? -1 : ((rt || S.pred == 0) ? acc_c : 1 - acc_c);
  // (also after a two-trial difference pass -- a pending decision's, phase 1, where the borderline
  // full steps land, or the tiny phase's both-trial pass; a first-trial-only pass that rejects its
  // trial is repeated as a pending two-trial decision, below)
  const bool devok = ondev != 0 && (!diffdec || S.single == 0);
  if (devok && acc_slot == 1) {
    // The other trial was accepted (embed.cpp:244-256 with the point in slot 1): Y moves there;
    // its gradient comes from this unit's pass (MODE 1 at Y) and the next gd_step forms the
    // trials (S.fix above).  pred follows the first two trials only (fit.cu gradient_descent).
    const double decrease = __ddiv_rn(__dsub_rn(fY, f_new), fmax(fY, 1e-300));
    R.f = f_new;
    R.it = S.it + 1;
    R.step = __dmul_rn(sc_acc, 2.0);
    if (!rt) R.pred = acc_c;
    R.tiny = 0;
    if (decrease < rel_tol) {
      R.stop = 1;
      R.stalled = 1;
    } else if (R.it >= max_iters) {
      R.stop = 1;
    }
    if (!R.stop) {
      R.fix = 1;
      R.nextra = S.nextra + 1;
    }
    if (lead) {
      history[R.it] = f_new;
      publish(R);
    }
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
      Y[k] = cand1[k];
    return;
  }
  if (devok && acc_c < 0 && gsq > 0.0 && !unresolved) {
    // Neither trial accepted: the reference halves on (embed.cpp:242-250; fit.cu's loop: step / 4
    // and step / 8 next, two per round, 60 halvings at most).  The trials are re-formed from Y and
    // the scaled gradient (finish_body with scale 1: the same y - s g as axpy_cand_kernel, and the
    // same |g|^2 partials again) and this unit's fused pass evaluates them.
    const int halv = (rt ? S.halv : 0) + 2;
    R.tiny = 0;
    if (halv >= 60) {  // no descent direction at double precision (embed.cpp:252-255)
      R.stop = 1;
      R.stalled = 1;
      if (lead) publish(R);
      return;
    }
    R.rt = 1;
    R.halv = halv;
    R.step = __dmul_rn(S.step, 0.25);
    R.nextra = S.nextra + 1;
    if (lead) publish(R);
    finish_body(1.0, graw, Y, m, R.step, __dmul_rn(R.step, 0.5), cand0, cand1, sqnext, red);
    return;
  }
  if (ondev && acc_c < 0 && diffdec && phase == 0 && S.single != 0 && kind == kKruskal && gsq > 0.0) {
    // tiny phase, first trial only, rejected: both trials by differences in this unit's difference
    // slot, decided by phase 1 (whose outcomes all stay on the device)
    R.pending = 1;
    R.single = 0;
    R.tiny = 0;
    R.ndiff = S.ndiff + 1;
    if (lead) publish(R);
    return;
  }
  if (acc_c < 0 || acc_slot != 0) {  // host takes this iteration
    R.stop = 2;
    R.tiny = 0;
    R.solo_miss = solo ? 1 : 0;  // (solo: only an unresolved non-Kruskal decision gets here)
    if (lead) publish(R);
    combine();
    return;
  }
  const double decrease = __ddiv_rn(__dsub_rn(fY, f_new), fmax(fY, 1e-300));
  R.f = f_new;
  R.it = S.it + 1;
  R.step = __dmul_rn(sc_acc, 2.0);
  if (decrease < rel_tol) {
    R.stop = 1;
    R.stalled = 1;
  } else if (R.it >= max_iters) {
    R.stop = 1;
  }
  // tiny mode for the next iteration: this (difference-sum) decision changed f by less than a
  // quarter of the resolution threshold, so the doubled step will not be resolved either: the
  // next pass is the difference + gradient pass, of the first trial only when it leads the
  // slot order (if it is rejected the iteration goes to the host, which evaluates both)
  // ... or this decision, taken on difference sums, would have been unresolved on plain fp32 sums
  // (the full step sitting at the Armijo threshold, run after run in the late regime): the next
  // iteration's fused pass would need a difference pass again -- one difference + gradient pass
  // instead of the two (tiny_ok == 2: q <= 2, where that pass does not spill -- at q = 3 it measured
  // no faster than the two; GMDS_TINY_STICKY=0 keeps the magnitude rule alone)
  const bool would_unres =
      tiny_ok == 2 && diffdec && precise_rel > 0.0 &&
      ((fabs(loss_of(t0) - fY) <= tol && fabs(loss_of(t1) - fY) <= tol) ||
       armijo_unresolved(fY, S.step, gsq, loss_of(S.pred == 0 ? t0 : t1), loss_of(S.pred == 0 ? t1 : t0), tol));
  R.tiny = (tiny_ok && diffdec && (fabs(__dsub_rn(fY, f_new)) <= 0.25 * tol || would_unres)) ? 1 : 0;
  R.single = (R.tiny != 0 && S.pred == 0) ? 1 : 0;
  // solo for the next pass: the full step was just accepted on resolved fp32 sums with room to
  // spare (a change of more than 4 tol), so the doubled step's half-step loss will go unread
  R.streak = (!diffdec && !rt && S.pred == 0 && (precise_rel <= 0.0 || fabs(__dsub_rn(fY, f_new)) > 4.0 * tol))
                 ? S.streak + 1
                 : 0;
  R.solo = (solo_ok && R.tiny == 0 && R.stop == 0 && R.streak >= 2) ? 1 : 0;
  if (lead) {
    history[R.it] = f_new;
    publish(R);
  }
  // Y <- cand0 (the accepted point); graw <- scaled gradient there; next trial pair
  const double raw_acc = xred ? (phase == 1 ? dsum[0] : xred[m])
                              : (pre ? pre[2] : tree_sum<256>(losspart, nparts, stride, 0, red));
  const double scale = grad_scale(kind, raw_acc, sum_sq, sum);
  const double s0 = (S.pred == 0) ? R.step : __dmul_rn(R.step, 0.5);
  const double s1 = (S.pred == 0) ? __dmul_rn(R.step, 0.5) : R.step;
  if (R.stop) {  // final point only
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
      Y[k] = cand0[k];
    return;
  }
  combine();  // each thread its own elements: read back below by the same thread
  finish_body(scale, graw, cand0, m, s0, s1, cand0, cand1, sqnext, red, Y, gnext);
}

// out_c = Y - step_c * G for each candidate (trial = coords - step * grad, embed.cpp:243).
__global__ void axpy_cand_kernel(const double* __restrict__ Y, const double* __restrict__ G, int64_t m, Steps s,
                                 double* __restrict__ out0, double* __restrict__ out1, double* __restrict__ out2,
                                 double* __restrict__ out3) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double y = Y[k], g = G[k];
    out0[k] = y - s.v[0] * g;
    if (s.n > 1) out1[k] = y - s.v[1] * g;
    if (s.n > 2) out2[k] = y - s.v[2] * g;
    if (s.n > 3) out3[k] = y - s.v[3] * g;
  }
}

// X+ = g / n (guttman_transform's uniform branch, embed.cpp:293).
__global__ void scale_kernel(const double* __restrict__ in, int64_t m, double inv, double* __restrict__ out) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = in[k] / inv;
}

// ---------------------------------------------------------------------------
// Host launchers

template <typename TD, bool GRAD>
static void launch_pass_t(const PassArgs& a, int Q, cudaStream_t st) {
  launch_pass_td<TD, GRAD>(a, Q, st);
  count_launch();
  check_launch("stress_pass_kernel");
}

void launch_stress_pass(const PassArgs& a, int q, bool grad, gmds_dtype storage, cudaStream_t st) {
  if (q <= 4) {
    if (storage == GMDS_F32)
      grad ? launch_pass_t<float, true>(a, q, st) : launch_pass_t<float, false>(a, q, st);
    else
      grad ? launch_pass_t<double, true>(a, q, st) : launch_pass_t<double, false>(a, q, st);
    return;
  }
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, ceil_div(a.n, 128)));
  if (storage == GMDS_F32)
    stress_rows_kernel<float><<<blocks, 128, 0, st>>>(a, q, grad ? 1 : 0);
  else
    stress_rows_kernel<double><<<blocks, 128, 0, st>>>(a, q, grad ? 1 : 0);
  count_launch();
  check_launch("stress_rows_kernel");
}

template <typename TP>
static void reduce_rows_t(const TP* rowpart, const TP* colpart, const int64_t* strip_first, int64_t n, int64_t nb,
                          int q, double* out, cudaStream_t st, double* gpart, const int* halt,
                          const double* losspart, int64_t nparts, int lstride, double* sums) {
  if (gpart) {
    const bool extra = sums != nullptr && kPT * q >= 256;
    launch_pdl(reduce_groups_kernel<TP>, dim3(static_cast<unsigned>(nb * kRedGroups + (extra ? 3 : 0))),
               dim3(kPT * q), 0, st, rowpart, colpart, strip_first, nb, q, gpart, halt, losspart, nparts, lstride,
               extra ? sums : nullptr);
    count_launch();
    check_launch("reduce_groups_kernel");
    if (!out) return;  // the caller adds the groups itself (gd_step_kernel)
    launch_pdl(combine_kernel, dim3(static_cast<unsigned>(ceil_div(n * q, 256))), dim3(256), 0, st, gpart, n, q, out,
               halt);
    count_launch();
    check_launch("combine_kernel");
    return;
  }
  const int64_t m = n * q * 8;
  reduce_rows_kernel<TP><<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, st>>>(rowpart, colpart, strip_first, n,
                                                                                 nb, q, out);
  count_launch();
  check_launch("reduce_rows_kernel");
}

void launch_reduce_rows(const double* rowpart, const double* colpart, const int64_t* strip_first, int64_t n,
                        int64_t nb, int q, double* out, cudaStream_t st, double* gpart, const int* halt,
                        bool f32parts, const double* losspart, int64_t nparts, int lstride, double* sums) {
  if (f32parts)
    reduce_rows_t(reinterpret_cast<const float*>(rowpart), reinterpret_cast<const float*>(colpart), strip_first, n,
                  nb, q, out, st, gpart, halt, losspart, nparts, lstride, sums);
  else
    reduce_rows_t(rowpart, colpart, strip_first, n, nb, q, out, st, gpart, halt, losspart, nparts, lstride, sums);
}

size_t reduce_rows_scratch(int64_t nb, int q) { return static_cast<size_t>(nb) * kRedGroups * kPT * q; }

int launch_finish_grad(const double* losspart, int64_t nparts, int stride, int kind, double sum_sq, double sum,
                       double* g, const double* Y, int64_t m, double s0, double s1, double* T0, double* T1,
                       double* sqpart, double* raw_out, cudaStream_t st, const double* raw_in) {
  const int blocks = static_cast<int>(std::min<int64_t>(kSqBlocks, std::max<int64_t>(1, ceil_div(m, 256))));
  finish_grad_kernel<<<blocks, 256, 0, st>>>(losspart, nparts, stride, kind, sum_sq, sum, g, Y, m, s0, s1, T0, T1,
                                             sqpart, raw_out, raw_in);
  count_launch();
  check_launch("finish_grad_kernel");
  return blocks;
}

static bool tiny_sticky() {
  static const bool on = [] {
    const char* e = std::getenv("GMDS_TINY_STICKY");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_gd_step(GdState* st2, int par, const double* losspart, int64_t nparts, int stride, const double* sqprev,
                    int nsq, double* sqnext, int kind, double sum_sq, double sum, double* Y, double* cand0,
                    double* cand1, double* gnext, const double* gpart, int Q, double* graw, int64_t m,
                    double* history, int max_iters, double rel_tol, const double* pre, double precise_rel,
                    int phase, cudaStream_t st, const double* xred, const double* dsum, bool tiny_ok,
                    bool solo_ok, bool ondev) {
  launch_pdl(gd_step_kernel, dim3(nsq), dim3(256), 0, st, st2, par, losspart, nparts, stride, sqprev, nsq, sqnext,
             kind, sum_sq, sum, Y, cand0, cand1, gnext, gpart, Q, graw, m, history, max_iters, rel_tol, pre,
             precise_rel, phase, xred, dsum, tiny_ok ? ((tiny_sticky() && Q <= 2) ? 2 : 1) : 0, solo_ok ? 1 : 0, ondev ? 1 : 0);
  count_launch();
  check_launch("gd_step_kernel");
}

void launch_shard_collect(const double* gpart, int64_t n, int Q, const double* losspart, int64_t nparts, int stride,
                          double* xred, const int* halt, cudaStream_t st) {
  launch_pdl(shard_collect_kernel, dim3(static_cast<unsigned>(ceil_div(n * Q, 256) + 1)), dim3(256), 0, st, gpart, n, Q,
             losspart, nparts, stride, xred, halt);
  count_launch();
  check_launch("shard_collect_kernel");
}

void launch_sum_parts(const double* part, int64_t count, int stride, int m, double* out, cudaStream_t st) {
  sum_parts_kernel<<<1, 1024, 0, st>>>(part, count, stride, m, out);
  count_launch();
  check_launch("sum_parts_kernel");
}

void launch_scale_sqnorm(double* g, int64_t m, double scale, double* out, double* part, cudaStream_t st) {
  const int blocks = static_cast<int>(std::min<int64_t>(kSqBlocks, std::max<int64_t>(1, ceil_div(m, 1024))));
  scale_sqnorm_kernel<<<blocks, 256, 0, st>>>(g, m, scale, part);
  sum_parts_kernel<<<1, 1024, 0, st>>>(part, blocks, 1, 1, out);
  count_launch(2);
  check_launch("scale_sqnorm_kernel");
}

void launch_axpy_cand(const double* Y, const double* G, int64_t m, const Steps& s, double* const* outs,
                      cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 1024)));
  axpy_cand_kernel<<<blocks, 256, 0, st>>>(Y, G, m, s, outs[0], outs[1], outs[2], outs[3]);
  count_launch();
  check_launch("axpy_cand_kernel");
}

// Weighted SMACOF's X+ = V^+ (B Z) (embed.cpp:315-322): out (n x Q row-major) from the
// symmetric n x n V^+ (column-major) and BZ (n x Q row-major); thread per row, reads of V^+
// coalesced across threads, j in order
__global__ void vpinv_apply_kernel(const double* __restrict__ Vp, const double* __restrict__ bz, int64_t n, int Q,
                                   double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j = 0; j < n; ++j) {
      const double v = Vp[j * n + i];  // V+(i, j) = V+(j, i)
      for (int k = 0; k < Q; ++k) acc[k] = fma(v, bz[j * Q + k], acc[k]);
    }
    for (int k = 0; k < Q; ++k) out[i * Q + k] = acc[k];
  }
}

void launch_vpinv_apply(const double* Vp, const double* bz, int64_t n, int Q, double* out, cudaStream_t st) {
  if (Q > 4) fail(GMDS_INVALID_INPUT, "weighted smacof: embedding dimension above 4 is not supported");
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, ceil_div(n, 128)));
  vpinv_apply_kernel<<<blocks, 128, 0, st>>>(Vp, bz, n, Q, out);
  count_launch();
  check_launch("vpinv_apply_kernel");
}

void launch_scale(const double* in, int64_t m, double divisor, double* out, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 1024)));
  scale_kernel<<<blocks, 256, 0, st>>>(in, m, divisor, out);
  count_launch();
  check_launch("scale_kernel");
}

}  // namespace gmds
