// Persistent stress fit for small n (n <= 2048, q <= 4): the whole
// minimize_stress loop -- gradient_descent with Armijo backtracking
// (embed.cpp:222-272) or smacof_iterate (embed.cpp:296-347) -- runs inside ONE
// cooperative kernel on every SM, with grid-wide barriers where the host
// engine (fit.cu) needs a device->host round trip.  (A tag-polling barrier in
// which every CTA polls the G partial slots was measured slower than
// cg::grid_group::sync: 0.66 s vs 0.48 s for config 2's fits.)  At these sizes a pass over
// D is a few microseconds of work, so launch + synchronisation latency, not
// bandwidth, bounds the host-driven loop (BASELINE config 1: n = 200, 500
// iterations; config 2: n = 1000, 1000 iterations per nu).
//
// Work split: CTA c owns rows [c n / G, (c + 1) n / G); warp w of the CTA
// covers column segment w of every owned row (lanes stride over j, reading
// the dense row-major fp64 copy of D, coalesced).  Each pair is evaluated
// from both of its rows (no atomics); per-row sums go through shared memory
// in a fixed order, loss partials per CTA to global, and every CTA reduces the
// G partials in the same order -- so every CTA computes bit-identical losses
// and takes the same Armijo / convergence decisions, with no broadcast.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "small_fit.h"
#include "stress.cuh"

namespace cg = cooperative_groups;

namespace gmds {

namespace {

constexpr int kSFThreads = 256;
constexpr int kSFWarps = kSFThreads / 32;
constexpr int kSFMaxRows = 16;  // rows per CTA (n <= 2048 on >= 128 CTAs)
constexpr int kU = 2;           // j-batch per lane (loads issued together)

struct Ctx {
  const double* D;
  int n, r0, r1, j0, j1;
  int kind;
  double delta;
};

// A configuration as its readers see it, computed inline so no pass has to
// wait for a separate materialisation step:
//   kPlain   z = base
//   kStep    z = base - s * (sc * g)    (Armijo trial point, fit.cu's axpy_cand on the scaled gradient)
//   kGuttman z = g / div                (SMACOF transform (B Z) / n)
enum SrcMode { kPlain = 0, kStep = 1, kGutt = 2 };
struct Src {
  const double* base;
  const double* g;
  double s, sc, div;
  int mode;
  __device__ __forceinline__ double at(int e) const {
    if (mode == kPlain) return __ldcg(base + e);
    if (mode == kStep) {
      const double gv = __ldcg(g + e) * sc;
      return __ldcg(base + e) - s * gv;
    }
    return __ldcg(g + e) / div;
  }
};

struct Smem {
  double sg[kSFWarps][kSFMaxRows][4];
  double szi[kSFMaxRows + 4][2][4];  // own rows of the pass's configurations (+ dead-row padding)
  double sl[kSFWarps][2];
  double sq[2];
  double sred[3][kSFWarps];
};


// Pass over the CTA's rows at NC configurations: loss partial of each
// configuration (pairs i < j) into lossp[cta*4 + c]; with GRAD, the row sums
// of c_ij (z_i - z_j) into g (own rows); with mat, the CTA's own rows of
// configuration 0 written out; with gq, the partial sum over own rows of
// (gq_sc * gq)^2 into lossp[cta*4 + 2].
//
// Loop order: column batches (kU columns per lane; the column coordinates
// are loaded once per batch) outside, the CTA's rows inside in groups of kRB
// (their D values loaded together), so a pass costs a few memory round trips
// rather than one per row.  Row sums: per (row, batch) warp xor-tree, added
// by lane 0 in batch order -- fixed order, deterministic.
template <int Q, int NC, bool GRAD>
__device__ void pass(const Ctx& x, const Src* Zp, double* g, double* mat, const double* gq, double gq_sc,
                     double* lossp, Smem& sm) {
  constexpr int kRB = (Q * NC <= 4) ? 4 : 2;  // rows whose D values are loaded together
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Src Z[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) Z[c] = Zp[c];
  const int rows = x.r1 - x.r0;
  const int rq = rows * Q;  // <= 64
  // own rows -> shared memory (and the materialised copy)
#pragma unroll
  for (int c = 0; c < NC; ++c)
    for (int o = threadIdx.x; o < rq; o += blockDim.x) {
      const double v = Z[c].at(x.r0 * Q + o);
      sm.szi[o / Q][c][o % Q] = v;
      if (c == 0 && mat) mat[x.r0 * Q + o] = v;
    }
  if (GRAD && lane == 0)
    for (int r = 0; r < rows; ++r)
#pragma unroll
      for (int k = 0; k < Q; ++k) sm.sg[w][r][k] = 0.0;
  __syncthreads();
  double lacc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) lacc[c] = 0.0;
  for (int jb = x.j0; jb < x.j1; jb += 32 * kU) {
    double zj[kU][NC][Q];
    bool in[kU];
    int jj[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = jb + lane + 32 * u;
      in[u] = j < x.j1;
      jj[u] = in[u] ? j : x.j0;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int k = 0; k < Q; ++k) zj[u][c][k] = in[u] ? Z[c].at(jj[u] * Q + k) : 0.0;
    }
    for (int rb = 0; rb < rows; rb += kRB) {
      double dv[kRB][kU];
#pragma unroll
      for (int q = 0; q < kRB; ++q) {
        const int r = x.r0 + min(rb + q, rows - 1);
#pragma unroll
        for (int u = 0; u < kU; ++u) dv[q][u] = __ldg(x.D + static_cast<size_t>(r) * x.n + jj[u]);
      }
#pragma unroll
      for (int q = 0; q < kRB; ++q) {
        const bool live = rb + q < rows;  // uniform across the warp
        const int r = x.r0 + rb + q;
        double gacc[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) gacc[k] = 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int j = jb + lane + 32 * u;
          const bool ok = live && in[u] && (j != r);
          const double Dv = ok ? dv[q][u] : 1.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            double dy[Q], d2 = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              dy[k] = sm.szi[rb + q][c][k] - zj[u][c][k];
              d2 += dy[k] * dy[k];
            }
            const double dist = sqrt(d2);
            const double e = Dv - dist;
            double term, cc;
            switch (x.kind) {
              case kKruskal: term = e * e; cc = -e; break;
              case kHuber: {
                const double ae = fabs(e);
                term = (ae <= x.delta) ? 0.5 * e * e : x.delta * (ae - 0.5 * x.delta);
                cc = -fmin(fmax(e, -x.delta), x.delta);
                break;
              }
              case kSammon: term = e * e / Dv; cc = -e / Dv; break;
              default: term = e * e; cc = Dv; break;  // Guttman: smacof loss + B(Z) Z numerator
            }
            if (ok && j > r) lacc[c] += term;
            if (GRAD && c == 0 && ok && dist > 0.0) {  // the gradient belongs to configuration 0
              const double ci = cc / dist;
#pragma unroll
              for (int k = 0; k < Q; ++k) gacc[k] += ci * dy[k];
            }
          }
        }
        if (GRAD)
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            double v = gacc[k];
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            if (lane == 0 && live) sm.sg[w][rb + q][k] += v;
          }
      }
    }
  }
  // per-warp loss over all its rows (fixed lane order, fixed xor tree)
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double v = lacc[c];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) sm.sl[w][c] = v;
  }
  if (gq && threadIdx.x < 64) {
    double v = 0.0;
    if (static_cast<int>(threadIdx.x) < rq) {
      const double gv = __ldcg(gq + x.r0 * Q + threadIdx.x) * gq_sc;
      v = gv * gv;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) sm.sq[w] = v;
  }
  __syncthreads();
  if (GRAD && static_cast<int>(threadIdx.x) < rq) {
    const int rr = threadIdx.x / Q, k = threadIdx.x % Q;
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < kSFWarps; ++ww) s += sm.sg[ww][rr][k];
    g[(x.r0 + rr) * Q + k] = s;
  }
  if (threadIdx.x < NC) {
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < kSFWarps; ++ww) s += sm.sl[ww][threadIdx.x];
    lossp[blockIdx.x * 4 + threadIdx.x] = s;
  }
  if (gq && threadIdx.x == 32) lossp[blockIdx.x * 4 + 2] = sm.sq[0] + sm.sq[1];
  __syncthreads();
}

// Sums of the G per-CTA partials p[c * 4 + k], k < NK: one parallel load per
// thread, then a fixed-shape tree (identical in every CTA, so every CTA gets
// the same bits).  G <= kSFThreads.
template <int NK>
__device__ __forceinline__ void grid_totals(const double* p, double* out, Smem& sm) {
  const int t = threadIdx.x;
  double v[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    v[k] = (t < static_cast<int>(gridDim.x)) ? __ldcg(p + t * 4 + k) : 0.0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], d);
  }
  if ((t & 31) == 0)
#pragma unroll
    for (int k = 0; k < NK; ++k) sm.sred[k][t >> 5] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kSFWarps; ++w) s += sm.sred[k][w];
    out[k] = s;
  }
  __syncthreads();
}

template <int Q>
__global__ void __launch_bounds__(kSFThreads, 1) small_fit_kernel(SmallFitArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  const int n = a.n, G = gridDim.x, cta = blockIdx.x;
  Ctx x;
  x.D = a.D;
  x.n = n;
  x.r0 = static_cast<int>(static_cast<int64_t>(cta) * n / G);
  x.r1 = static_cast<int>(static_cast<int64_t>(cta + 1) * n / G);
  const int seg = (n + kSFWarps - 1) / kSFWarps;
  x.j0 = min(n, static_cast<int>(threadIdx.x >> 5) * seg);
  x.j1 = min(n, x.j0 + seg);
  x.kind = a.kind;
  x.delta = a.delta;
  const bool lead = (cta == 0 && threadIdx.x == 0);
  // a.buf: [0] Y0, [1] second coordinate slot, [2], [3] gradient / B(Z) Z double buffer.
  // Partials are double-buffered too: a CTA may start the next pass while
  // others are still reducing the previous one.
  double* Yb[2] = {a.buf[0], a.buf[1]};
  double* Gb[2] = {a.buf[2], a.buf[3]};
  int yb = 0, gb = 0, bank = 0;
  auto lp = [&]() { return a.lossp + bank * 4 * G; };
  int npass = 0, it = 0, hl = 1;
  bool conv = false;
  double f = 0.0;
  Src fin{Yb[0], nullptr, 0.0, 0.0, 1.0, kPlain};  // the fit's current coordinates
  if (a.kind == kSmacof) {
    x.kind = kGuttman;
    pass<Q, 1, true>(x, &fin, Gb[gb], nullptr, nullptr, 0.0, lp(), sm);
    ++npass;
    grid.sync();
    grid_totals<1>(lp(), &f, sm);
    bank ^= 1;
    if (lead) a.history[0] = f;
    for (; it < a.max_iters; ++it) {
      // coords = next = (B(Z) Z) / n, read inline from the gradient buffer
      fin = Src{nullptr, Gb[gb], 0.0, 0.0, static_cast<double>(n), kGutt};
      gb ^= 1;
      pass<Q, 1, true>(x, &fin, Gb[gb], nullptr, nullptr, 0.0, lp(), sm);
      ++npass;
      double f_new;
      grid.sync();
      grid_totals<1>(lp(), &f_new, sm);
      bank ^= 1;
      if (lead) a.history[hl] = f_new;
      ++hl;
      const double decrease = (f - f_new) / fmax(f, 1e-300);
      f = f_new;
      if (decrease < a.rel_tol) {
        ++it;
        conv = true;
        break;
      }
    }
  } else {
    auto loss_of = [&](double raw) {
      if (a.kind == kKruskal) return sqrt(raw / a.sum_sq);
      if (a.kind == kSammon) return (1.0 / a.sum) * raw;
      return raw;
    };
    pass<Q, 1, true>(x, &fin, Gb[gb], nullptr, nullptr, 0.0, lp(), sm);
    ++npass;
    double raw;
    grid.sync();
    grid_totals<1>(lp(), &raw, sm);
    bank ^= 1;
    f = loss_of(raw);
    if (lead) a.history[0] = f;
    double step = 1.0;
    int pred = 0;  // slot order of the next first-round trial pair (0: step in slot 0)
    for (; it < a.max_iters; ++it) {
      double scale = 1.0;
      if (a.kind == kKruskal) {
        const double ks = sqrt(raw / a.sum_sq);
        scale = (ks <= 0.0) ? 0.0 : 1.0 / (ks * a.sum_sq);  // embed.cpp:179-181
      } else if (a.kind == kSammon) {
        scale = 2.0 * (1.0 / a.sum);
      }
      // Armijo trial points in pairs (step, step/2), evaluated inline from
      // (Y, scaled gradient); the same pass yields |g|^2.  Speculation, as in the
      // tiled engine (fit.cu gradient_descent): the trial predicted to be accepted
      // (the same choice, step or step / 2, as the last first-round acceptance) sits
      // in slot 0, and the pass also takes the gradient and the coordinates there --
      // a correct prediction saves the separate gradient pass and its grid barrier.
      // The trials are still tested in the reference's order (step, then step / 2).
      Src tr[2] = {{Yb[yb], Gb[gb], step, scale, 1.0, kStep}, {Yb[yb], Gb[gb], step * 0.5, scale, 1.0, kStep}};
      bool accepted = false, stalled = false;
      int acc = 0;  // slot of the accepted trial
      double f_new = f, raw_acc = 0.0;
      for (int halvings = 0; halvings < 60; halvings += 2) {
        const int first = (halvings == 0) ? pred : 0;  // slot of `step` (later rounds: natural order)
        tr[first].s = step;
        tr[first ^ 1].s = step * 0.5;
        pass<Q, 2, true>(x, tr, Gb[gb ^ 1], Yb[yb ^ 1], Gb[gb], scale, lp(), sm);
        ++npass;
        double tot[3];
        grid.sync();
        grid_totals<3>(lp(), tot, sm);
        bank ^= 1;
        if (tot[2] <= 0.0) {  // grad_sq <= 0: the reference stops before any trial
          stalled = true;
          break;
        }
        const double f0 = loss_of(tot[first]), f1 = loss_of(tot[first ^ 1]);  // at step, at step / 2
        if (f0 <= f - 1e-4 * step * tot[2]) {
          accepted = true;
          acc = first;
          f_new = f0;
          raw_acc = tot[first];
          if (halvings == 0) pred = 0;
          break;
        }
        if (f1 <= f - 1e-4 * (step * 0.5) * tot[2]) {
          accepted = true;
          acc = first ^ 1;
          f_new = f1;
          raw_acc = tot[first ^ 1];
          step *= 0.5;
          if (halvings == 0) pred = 1;
          break;
        }
        step *= 0.25;
      }
      if (stalled || !accepted) {
        conv = true;
        break;
      }
      fin = tr[acc];
      if (lead) a.history[hl] = f_new;
      ++hl;
      const double decrease = (f - f_new) / fmax(f, 1e-300);
      f = f_new;
      step *= 2.0;
      if (decrease < a.rel_tol) {
        ++it;
        conv = true;
        break;
      }
      if (acc == 0) {
        // predicted: the trial pass left the gradient, the coordinates and the raw loss there
        gb ^= 1;
        yb ^= 1;
        fin = Src{Yb[yb], nullptr, 0.0, 0.0, 1.0, kPlain};
        raw = raw_acc;
        continue;
      }
      // gradient pass at the accepted point; it also materialises its own rows
      pass<Q, 1, true>(x, &fin, Gb[gb ^ 1], Yb[yb ^ 1], nullptr, 0.0, lp(), sm);
      ++npass;
      gb ^= 1;
      yb ^= 1;
      fin = Src{Yb[yb], nullptr, 0.0, 0.0, 1.0, kPlain};
      grid.sync();
      grid_totals<1>(lp(), &raw, sm);
      bank ^= 1;
    }
  }
  // final coordinates (own rows) to the output buffer
  for (int e = x.r0 * Q + threadIdx.x; e < x.r1 * Q; e += blockDim.x) a.Yout[e] = fin.at(e);
  if (lead) {
    a.out[0] = f;
    a.iout[0] = it;
    a.iout[1] = (conv || it < a.max_iters) ? 1 : 0;
    a.iout[2] = hl;
    a.iout[3] = npass;
  }
}

template <int Q>
void launch_q(SmallFitArgs a, int grid, cudaStream_t st) {
  void* args[] = {&a};
  GMDS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(small_fit_kernel<Q>), dim3(grid), dim3(kSFThreads),
                                        args, 0, st));
}

}  // namespace

bool small_fit_supported(int64_t n, int q) { return n >= 2 && n <= kSmallFitMaxN && q >= 1 && q <= 4; }

int small_fit_grid(int64_t n) {
  int dev = 0, sms = 0;
  GMDS_CUDA(cudaGetDevice(&dev));
  GMDS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int g = static_cast<int>(std::min<int64_t>(sms, n));
  if (ceil_div(n, static_cast<int64_t>(g)) > kSFMaxRows) return 0;  // too few SMs: host engine instead
  return g;
}

void launch_small_fit(const SmallFitArgs& a, int q, int grid, cudaStream_t st) {
  switch (q) {
    case 1: launch_q<1>(a, grid, st); break;
    case 2: launch_q<2>(a, grid, st); break;
    case 3: launch_q<3>(a, grid, st); break;
    default: launch_q<4>(a, grid, st); break;
  }
  count_launch();
  check_launch("small_fit_kernel");
}

}  // namespace gmds
