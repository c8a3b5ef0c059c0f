// Host orchestration of the stress path and its C-ABI: device DistanceMatrix
// handles, stress_loss / stress_gradient / kruskal_stress, classical_mds
// (cuSOLVER syevd on the double-centred Gram matrix), and minimize_stress
// (Armijo gradient descent for kruskal / huber / sammon, SMACOF majorisation)
// with the reference's control flow (embed.cpp:222-272, 296-347, 491-532).
//
// Per gradient-descent iteration the device makes two passes over D: one
// gradient pass at Y (which also yields the loss at Y), and one loss pass that
// evaluates up to four Armijo trial points (step, step/2, step/4, step/8) at
// once; the host takes the first one that satisfies the reference's Armijo
// test, so the accepted point is the one the reference's sequential
// halving loop would accept.  SMACOF needs one pass per iteration: the pass
// at Z yields loss(Z) and the Guttman transform of Z together.
#include <cusolverDn.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "dmat.cuh"
#include "dmat_kernels.cuh"
#include "fit.h"
#include "kernels.cuh"
#include "lib_internal.h"
#include "small_fit.h"
#include "classical_topq.h"
#include "stress.cuh"

namespace gmds {

// Blocks per CTA of a tiled pass (one block row): 8 at large n (measured best
// at n = 20000 with programmatic dependent launch: 2,730 it/s vs 2,706 at 4,
// 2,595 at 16; profiles/r1_stress_chunk_sweep.txt), fewer when that would leave the pass short of ~8 CTAs per SM
// (n = 5000: 820 blocks -> 1 per CTA); GMDS_STRESS_CHUNK overrides (tuning).
int64_t chunk_blocks(int64_t nb) {
  if (const char* e = std::getenv("GMDS_STRESS_CHUNK")) {
    const int64_t c = std::atoll(e);
    if (c > 0) return c;
  }
  const int64_t nblk = nb * (nb + 1) / 2;
  return std::max<int64_t>(1, std::min<int64_t>(8, nblk / (148 * 8)));
}

// (I, J0) of every chunk, in packed order
void chunk_list(int64_t nb, int64_t len, std::vector<int64_t>& cI, std::vector<int64_t>& cJ) {
  for (int64_t I = 0; I < nb; ++I)
    for (int64_t J0 = I; J0 < nb; J0 += len) {
      cI.push_back(I);
      cJ.push_back(J0);
    }
}

namespace {
int64_t blk_of(int64_t I, int64_t J, int64_t nb) { return I * nb - (I * (I - 1)) / 2 + (J - I); }
}  // namespace

// Rank `rank`'s packed blocks [blk_lo, blk_hi): the chunks whose preceding block count
// reaches nblk * rank / size start the share (the split grad_raw_shard uses).
void shard_blocks(int64_t n, int rank, int size, int64_t& blk_lo, int64_t& blk_hi) {
  const int64_t nb = ceil_div(n, kPT), nblk = nb * (nb + 1) / 2;
  std::vector<int64_t> cI, cJ;
  chunk_list(nb, chunk_blocks(nb), cI, cJ);
  auto edge = [&](int r) {
    if (r >= size) return nblk;
    for (size_t c = 0; c < cI.size(); ++c) {
      const int64_t before = blk_of(cI[c], cJ[c], nb);
      if (before * size >= nblk * r) return before;
    }
    return nblk;
  };
  blk_lo = edge(rank);
  blk_hi = edge(rank + 1);
}

namespace {
constexpr double kTiny = 1e-300;  // embed.cpp:13
constexpr double kPreciseRel = 1e-6;  // fp32-storage loss changes below this are re-evaluated in fp64

int padded_q(int q) { return q <= 4 ? q : q; }

// One cuSOLVER handle per (host thread, device), created on first use and kept:
// creating one costs milliseconds, which dominated small classical fits.
cusolverDnHandle_t solver_handle(cudaStream_t st) {
  static thread_local std::map<int, cusolverDnHandle_t> handles;
  int dev = 0;
  GMDS_CUDA(cudaGetDevice(&dev));
  cusolverDnHandle_t& h = handles[dev];
  if (!h && cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) {
    h = nullptr;
    fail(GMDS_CUDA_ERROR, "cusolverDnCreate failed");
  }
  cusolverDnSetStream(h, st);
  return h;
}

}  // namespace

// ---------------------------------------------------------------------------
Engine::Engine(const gmds_dmat* Dm, int q_, cudaStream_t st_, Comm* comm_) : D(Dm), q(q_), st(st_), comm(comm_) {
  n = D->n;
  nb = ceil_div(n, kPT);
  Q = padded_q(q);
  rows_mode = (q > 4);
  if (D->sharded() && (rows_mode || !comm)) fail(GMDS_INVALID_INPUT, "row-sharded distance matrix: q <= 4 and its comm");
  if (!rows_mode) {
    chunk_len = chunk_blocks(nb);
    std::vector<int64_t> aI, aJ, cI, cJ, sf;
    chunk_list(nb, chunk_len, aI, aJ);
    for (size_t c = 0; c < aI.size(); ++c) {  // row-sharded: this rank's chunks only
      const int64_t b = blk_of(aI[c], aJ[c], nb);
      if (D->sharded() && (b < D->blk_lo || b >= D->blk_hi)) continue;
      cI.push_back(aI[c]);
      cJ.push_back(aJ[c]);
    }
    for (int64_t I = 0, c = 0; I <= nb; ++I) {  // strip I's chunks: [sf[I], sf[I + 1])
      while (c < static_cast<int64_t>(cI.size()) && cI[c] < I) ++c;
      sf.push_back(c);
    }
    nchunks = static_cast<int64_t>(cI.size());
    chunk_I.alloc(std::max<size_t>(1, cI.size()));
    chunk_J0.alloc(std::max<size_t>(1, cJ.size()));
    strip_first.alloc(sf.size());
    if (nchunks) {
      GMDS_CUDA(cudaMemcpyAsync(chunk_I.get(), cI.data(), cI.size() * 8, cudaMemcpyHostToDevice, st));
      GMDS_CUDA(cudaMemcpyAsync(chunk_J0.get(), cJ.data(), cJ.size() * 8, cudaMemcpyHostToDevice, st));
    }
    GMDS_CUDA(cudaMemcpyAsync(strip_first.get(), sf.data(), sf.size() * 8, cudaMemcpyHostToDevice, st));
    const int64_t nblk = nb * (nb + 1) / 2;
    stride_row = std::max<int64_t>(1, nchunks) * kPT * Q;
    stride_col = nblk * kPT * Q;
    rowpart.alloc(static_cast<size_t>(stride_row));
    colpart.alloc(static_cast<size_t>(stride_col));
    gpart.alloc(reduce_rows_scratch(nb, Q));
    losspart.alloc(static_cast<size_t>(std::max<int64_t>(1, nchunks) * kMaxCand));
    if (D->sharded()) {  // foreign blocks' column partials are never written: zero once
      GMDS_CUDA(cudaMemsetAsync(colpart.get(), 0, colpart.n * sizeof(double), st));
      GMDS_CUDA(cudaMemsetAsync(rowpart.get(), 0, rowpart.n * sizeof(double), st));
      GMDS_CUDA(cudaMemsetAsync(losspart.get(), 0, losspart.n * sizeof(double), st));
      xred.alloc(static_cast<size_t>(n * Q + 8));
      dsum.alloc(4);
      rawy.alloc(1);
    }
  } else {
    nchunks = n;
    rowpart.alloc(static_cast<size_t>(n * Q));
    losspart.alloc(static_cast<size_t>(n * kMaxCand));
  }
  graw.alloc(static_cast<size_t>(n * Q));
  Y.alloc(static_cast<size_t>(n * Q));
  for (auto& b : cand) b.alloc(static_cast<size_t>(n * Q));
  scal.alloc(8);
  sqpart.alloc(kSqBlocks);
  GMDS_CUDA(cudaStreamSynchronize(st));
}

void Engine::allreduce(double* d, size_t count) {
  if (comm) comm->allreduce(d, count, RedOp::kSum, st);
}

void Engine::upload(const double* coords_colmajor, double* dst) {
  std::vector<double> h(static_cast<size_t>(n * Q), 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < q; ++k) h[i * Q + k] = coords_colmajor[k * n + i];
  GMDS_CUDA(cudaMemcpyAsync(dst, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
}

void Engine::download(const double* src, double* coords_colmajor) {
  std::vector<double> h(static_cast<size_t>(n * Q));
  GMDS_CUDA(cudaMemcpyAsync(h.data(), src, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < q; ++k) coords_colmajor[k * n + i] = h[i * Q + k];
}

PassArgs Engine::args(int kind, double delta) const {
  PassArgs a{};
  a.chunk_I = nullptr;
  a.D = D->ptr();
  a.W = W;
  a.n = n;
  a.nb = nb;
  a.kind = kind;
  a.huber_delta = delta;
  a.chunk_I = chunk_I.get();
  a.chunk_J0 = chunk_J0.get();
  a.chunk_len = chunk_len;
  a.nchunks = nchunks;
  a.rowpart = rowpart.get();
  a.colpart = colpart.get();
  a.losspart = losspart.get();
  a.cand_stride_row = stride_row;
  a.cand_stride_col = stride_col;
  return a;
}

std::vector<double> Engine::loss_raw(int kind, double delta, const double* const* Ys, int nc) {
  PassArgs a = args(kind, delta);
  for (int c = 0; c < nc; ++c) a.Y[c] = Ys[c];
  a.ncand = nc;
  launch_stress_pass(a, Q, false, D->storage, st);
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, nc, scal.get(), st);
  allreduce(scal.get(), static_cast<size_t>(nc));
  std::vector<double> out(static_cast<size_t>(nc));
  GMDS_CUDA(cudaMemcpyAsync(out.data(), scal.get(), nc * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  ++passes;
  return out;
}

std::vector<double> Engine::loss_raw_precise(int kind, double delta, const double* const* Ys, int nc) {
  PassArgs a = args(kind, delta);
  for (int c = 0; c < nc; ++c) a.Y[c] = Ys[c];
  a.ncand = nc;
  launch_pass_precise(a, Q, st);
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, nc, scal.get(), st);
  allreduce(scal.get(), static_cast<size_t>(nc));
  std::vector<double> out(static_cast<size_t>(nc));
  GMDS_CUDA(cudaMemcpyAsync(out.data(), scal.get(), nc * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  ++passes;
  return out;
}

std::vector<double> Engine::loss_diff(int kind, double s0, double s1) {
  PassArgs a = args(kind, 0.0);
  a.Y[0] = Y.get();
  a.Y[1] = graw.get();
  a.ncand = 2;
  a.dstep[0] = s0;
  a.dstep[1] = s1;
  launch_pass_diff_f32(a, Q, st);
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, 3, scal.get(), st);
  allreduce(scal.get(), 3);
  double h[3];
  GMDS_CUDA(cudaMemcpyAsync(h, scal.get(), sizeof h, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  ++passes;
  return {h[2], h[0], h[1]};  // Y, Y - s0 g, Y - s1 g (losspart column 0: the first trial, as a trial pass)
}

double Engine::grad_raw(int kind, double delta, const double* Yd) {
  if (q > 64) fail(GMDS_INVALID_INPUT, "stress gradient: embedding dimension above 64 is not supported");
  PassArgs a = args(kind, delta);
  a.Y[0] = Yd;
  a.ncand = 1;
  launch_stress_pass(a, Q, true, D->storage, st);
  if (!rows_mode)
    launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, graw.get(), st, gpart.get(), nullptr, f32parts());
  else
    GMDS_CUDA(cudaMemcpyAsync(graw.get(), rowpart.get(), sizeof(double) * n * Q, cudaMemcpyDeviceToDevice, st));
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, 1, scal.get(), st);
  if (comm) {  // row-sharded: [gradient | raw loss] summed over the ranks
    double* bufs[2] = {graw.get(), scal.get()};
    const size_t counts[2] = {static_cast<size_t>(n * Q), 1};
    comm->allreduce_group(bufs, counts, 2, st);
    GMDS_CUDA(cudaMemcpyAsync(rawy.get(), scal.get(), sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  double out = 0.0;
  GMDS_CUDA(cudaMemcpyAsync(&out, scal.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  ++passes;
  return out;
}

// Raw sums over the chunks of shard `shard` of `nshards` (rows of the other
// shards' chunks contribute nothing): the per-rank pass of a sharded fit,
// summed across ranks by an all-reduce.
double Engine::grad_raw_shard(int kind, double delta, const double* Yd, int shard, int nshards) {
  if (rows_mode) fail(GMDS_INVALID_INPUT, "stress_partial: sharded passes support q <= 4");
  // chunk c covers up to chunk_len blocks... weight = number of blocks; split the prefix sum evenly
  std::vector<int64_t> cI(static_cast<size_t>(nchunks)), cJ(static_cast<size_t>(nchunks));
  GMDS_CUDA(cudaMemcpyAsync(cI.data(), chunk_I.get(), nchunks * 8, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(cJ.data(), chunk_J0.get(), nchunks * 8, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  const int64_t nblk = nb * (nb + 1) / 2;
  int64_t acc = 0, c0 = nchunks, c1 = nchunks;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t before = acc;
    acc += std::min<int64_t>(chunk_len, nb - cJ[c]);
    if (c0 == nchunks && before * nshards >= nblk * shard) c0 = c;
    if (c1 == nchunks && before * nshards >= nblk * (shard + 1)) c1 = c;
  }
  // zero the partial buffers of foreign chunks/blocks, then run the pass on the sub-range
  GMDS_CUDA(cudaMemsetAsync(rowpart.get(), 0, rowpart.n * sizeof(double), st));
  GMDS_CUDA(cudaMemsetAsync(colpart.get(), 0, colpart.n * sizeof(double), st));
  GMDS_CUDA(cudaMemsetAsync(losspart.get(), 0, losspart.n * sizeof(double), st));
  PassArgs a = args(kind, delta);
  a.Y[0] = Yd;
  a.ncand = 1;
  a.chunk_I = chunk_I.get() + c0;
  a.chunk_J0 = chunk_J0.get() + c0;
  a.nchunks = c1 - c0;
  a.rowpart = f32parts() ? reinterpret_cast<double*>(reinterpret_cast<float*>(rowpart.get()) + c0 * kPT * Q)
                        : rowpart.get() + c0 * kPT * Q;
  a.losspart = losspart.get() + c0 * kMaxCand;
  if (a.nchunks > 0) launch_stress_pass(a, Q, true, D->storage, st);
  launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, graw.get(), st, gpart.get(), nullptr, f32parts());
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, 1, scal.get(), st);
  double out = 0.0;
  GMDS_CUDA(cudaMemcpyAsync(&out, scal.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  ++passes;
  return out;
}

Engine::GradTrials Engine::grad_and_trials(int kind, double delta, double s0, double s1) {
  if (comm) fail(GMDS_INVALID_CONFIG, "row-sharded fits run on fp32 storage");
  if (q > 64) fail(GMDS_INVALID_INPUT, "stress gradient: embedding dimension above 64 is not supported");
  PassArgs a = args(kind, delta);
  a.Y[0] = Y.get();
  a.ncand = 1;
  launch_stress_pass(a, Q, true, D->storage, st);
  if (!rows_mode)
    launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, graw.get(), st, gpart.get(), nullptr, f32parts());
  else
    GMDS_CUDA(cudaMemcpyAsync(graw.get(), rowpart.get(), sizeof(double) * n * Q, cudaMemcpyDeviceToDevice, st));
  const int nsq = launch_finish_grad(losspart.get(), nchunks, kMaxCand, kind, D->sum_sq, D->sum, graw.get(), Y.get(),
                                     n * Q, s0, s1, cand[0].get(), cand[1].get(), sqpart.get(), scal.get(), st);
  PassArgs b = args(kind, delta);
  b.Y[0] = cand[0].get();
  b.Y[1] = cand[1].get();
  b.ncand = 2;
  launch_stress_pass(b, Q, false, D->storage, st);
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, 2, scal.get() + 1, st);
  double h[3];
  std::vector<double> sq(static_cast<size_t>(nsq));
  GMDS_CUDA(cudaMemcpyAsync(h, scal.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(sq.data(), sqpart.get(), nsq * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  passes += 2;
  GradTrials r;
  r.raw = h[0];
  r.trial[0] = h[1];
  r.trial[1] = h[2];
  r.gsq = 0.0;
  for (double v : sq) r.gsq += v;  // fixed order
  return r;
}

Engine::GradTrials Engine::fused_trials(int kind, double delta, double s0, double s1) {
  if (!gnext.get()) gnext.alloc(static_cast<size_t>(n * Q));
  const int nsq = launch_finish_grad(losspart.get(), nchunks, kMaxCand, kind, D->sum_sq, D->sum, graw.get(), Y.get(),
                                     n * Q, s0, s1, cand[0].get(), cand[1].get(), sqpart.get(), scal.get(), st,
                                     comm ? rawy.get() : nullptr);
  PassArgs b = args(kind, delta);
  b.Y[0] = cand[0].get();
  b.Y[1] = cand[1].get();
  b.ncand = 2;
  launch_pass_fused_f32(b, Q, st);
  launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, gnext.get(), st, gpart.get(), nullptr, f32parts());
  launch_sum_parts(losspart.get(), nchunks, kMaxCand, 2, scal.get() + 1, st);
  if (comm) {  // row-sharded: [gradient at cand0 | both trial losses] over the ranks
    double* bufs[2] = {gnext.get(), scal.get() + 1};
    const size_t counts[2] = {static_cast<size_t>(n * Q), 2};
    comm->allreduce_group(bufs, counts, 2, st);
    // the raw loss at cand0: the next finish's loss at Y when that trial is accepted
    GMDS_CUDA(cudaMemcpyAsync(rawy.get(), scal.get() + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  double h[3];
  std::vector<double> sq(static_cast<size_t>(nsq));
  GMDS_CUDA(cudaMemcpyAsync(h, scal.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(sq.data(), sqpart.get(), nsq * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  passes += 1;
  GradTrials r;
  r.raw = h[0];
  r.trial[0] = h[1];
  r.trial[1] = h[2];
  r.gsq = 0.0;
  for (double v : sq) r.gsq += v;  // fixed order
  return r;
}

// need_grad: graw does not hold the gradient at Y -- the loop is primed with the one-point pass at Y and
// the fix state (its first gd_step forms the trials, as after a slot-1 acceptance); init: that pass is the
// fit's first, its loss is f(Y0) = history[it] (embed.cpp:226).
GdState Engine::device_gd(int kind, double delta, double f, double step, int it, int pred, int max_iters,
                          double rel_tol, std::vector<double>& history, double precise_rel, bool need_grad,
                          bool init) {
  if (!sq2.get()) {
    sq2.alloc(2 * kSqBlocks);
    gdst.alloc(2);
  }
  if (hist.n < static_cast<size_t>(max_iters) + 1) hist.alloc(static_cast<size_t>(max_iters) + 1);
  if (!gnext.get()) gnext.alloc(static_cast<size_t>(n * Q));
  const double s0 = pred == 0 ? step : step * 0.5, s1 = pred == 0 ? step * 0.5 : step;
  PassArgs b = args(kind, delta);
  int nsq;
  if (need_grad) {
    // prime: the gradient pass at Y (as grad_raw, without the round trip); gd_step's fix block finishes it
    nsq = static_cast<int>(std::min<int64_t>(kSqBlocks, std::max<int64_t>(1, ceil_div(n * Q, 256))));
    PassArgs g1 = args(kind, delta);
    g1.Y[0] = Y.get();
    g1.ncand = 1;
    launch_stress_pass(g1, Q, true, D->storage, st);
  } else {
    // prime: the trial pair of iteration `it` and its fused pass (as fused_trials, without the round trip)
    nsq = launch_finish_grad(losspart.get(), nchunks, kMaxCand, kind, D->sum_sq, D->sum, graw.get(), Y.get(), n * Q,
                             s0, s1, cand[0].get(), cand[1].get(), sq2.get(), scal.get(), st,
                             comm ? rawy.get() : nullptr);
  }
  b.Y[0] = cand[0].get();
  b.Y[1] = cand[1].get();
  b.ncand = 2;
  if (!need_grad) launch_pass_fused_f32(b, Q, st);
  double* pre = scal.get() + 5;  // the pass's loss sums (reduction launch's extra CTA; q >= 2)
  const bool have_pre = kPT * Q >= 256 && !comm;
  // row-sharded: this rank's [gradient | trial loss sums] -> xred, all-reduced (one collective per pass)
  double* xr = comm ? xred.get() : nullptr;
  auto collect = [&](const int* halt) {
    if (!comm) return;
    launch_shard_collect(gpart.get(), n, Q, losspart.get(), nchunks, kMaxCand, xr, halt, st);
    comm->allreduce(xr, static_cast<size_t>(n * Q + 3), RedOp::kSum, st);
  };
  launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, nullptr, st, gpart.get(), nullptr,
                     f32parts(), losspart.get(), nchunks, kMaxCand, have_pre ? pre : nullptr);
  collect(nullptr);
  ++passes;
  GdState S{};
  S.f = f;
  S.step = step;
  S.it = it;
  S.pred = pred;
  S.fix = need_grad ? 1 : 0;
  S.init = (need_grad && init) ? 1 : 0;
  GMDS_CUDA(cudaMemcpyAsync(gdst.get(), &S, sizeof S, cudaMemcpyHostToDevice, st));
  // history[it] lives on the device for the loop: a decision on difference sums re-bases it (as the host
  // loop re-bases history.back()); read back below
  const bool entry_hist = !(need_grad && init) && !history.empty();
  double f_entry = entry_hist ? history.back() : 0.0;
  if (entry_hist) GMDS_CUDA(cudaMemcpyAsync(hist.get() + it, &f_entry, sizeof(double), cudaMemcpyHostToDevice, st));
  int par = 0;  // state buffer (flips per gd_step launch)
  int sqp = 0;  // |g|^2 partials buffer (flips per iteration)
  int issued = it;
  PassArgs dpa = args(kind, delta);  // the device loop's difference pass (runs only when a decision is pending)
  dpa.Y[0] = Y.get();
  dpa.Y[1] = graw.get();
  dpa.ncand = 2;
  const bool dev_diff = precise_rel > 0.0 && kind == kKruskal && !W;
  // the tiny phase's difference + gradient pass (q <= 3); GMDS_NO_TINY=1: every sub-resolution
  // decision takes the fused pass and a difference pass (the host loop's two passes)
  const bool tiny_ok = dev_diff && Q <= 3 && !std::getenv("GMDS_NO_TINY");
  // slot-1 acceptances, further halvings and solo misses decided on the device (GdState::fix / rt);
  // GMDS_NO_ONDEV=1: those iterations go back to the host loop
  const bool ondev = !std::getenv("GMDS_NO_ONDEV");
  // solo passes (GdState::solo): slot 0 only, while the full step keeps being accepted on resolved sums;
  // GMDS_NO_SOLO=1: always the two-trial fused pass.  (Row-sharded fits: only with the on-device
  // miss handling -- the host's miss path is a loss pass without the all-reduce.)
  const bool solo_ok = (!comm || ondev) && !std::getenv("GMDS_NO_SOLO");
  // kruskal, q <= 3: the difference passes behind one launch and the fused / one-point pass behind one (stress_tma_multi_kernel)
  const bool multi = tiny_ok && ondev && !std::getenv("GMDS_NO_MULTI");
  for (;;) {
    // units per batch: an iteration takes one unit, or two when it needs a fix / re-trial unit
    const int left = max_iters - S.it;
    const int batch = std::max(1, std::min(16, left + (ondev ? std::min(left, 4) : 0)));
    for (int k = 0; k < batch; ++k) {
      for (int phase = 0; phase < (dev_diff ? 2 : 1); ++phase) {
        launch_gd_step(gdst.get(), par, losspart.get(), nchunks, kMaxCand, sq2.get() + sqp * kSqBlocks, nsq,
                       sq2.get() + (sqp ^ 1) * kSqBlocks, kind, D->sum_sq, D->sum, Y.get(), cand[0].get(),
                       cand[1].get(), gnext.get(), gpart.get(), Q, graw.get(), n * Q, hist.get(), max_iters,
                       rel_tol, have_pre ? pre : nullptr, precise_rel, phase, st, xr, comm ? dsum.get() : nullptr,
                       tiny_ok, solo_ok, ondev);
        par ^= 1;
        if (phase == 0 && dev_diff) {
          dpa.gds = gdst.get() + par;
          if (multi) {
            PassArgs b0 = b;
            b0.gds = dpa.gds;
            launch_pass_multi_f32(b0, dpa, Q, 0, st);
          } else {
            launch_pass_diff_f32(dpa, Q, st);   // both trials (runs unless the decision is single)
            launch_pass_diff1_f32(dpa, Q, st);  // the first trial only (runs if single)
          }
          if (comm) {  // the difference sums over the ranks (read by phase 1 only when pending)
            launch_sum_parts(losspart.get(), nchunks, kMaxCand, 3, dsum.get(), st);
            comm->allreduce(dsum.get(), 3, RedOp::kSum, st);
          }
        }
      }
      sqp ^= 1;
      b.halt = &gdst.get()[par].halt_fused;
      b.gds = gdst.get() + par;
      b.Y[2] = Y.get();
      PassArgs gp = args(kind, delta);  // tiny phase: one difference + gradient pass
      gp.Y[0] = Y.get();
      gp.Y[1] = graw.get();
      gp.ncand = 2;
      gp.gds = gdst.get() + par;
      if (multi) {
        launch_pass_multi_f32(b, gp, Q, 1, st);      // fused / one point
        launch_pass_diffgrad_f32(gp, Q, false, st);  // tiny phase, both trials (merged, the two bodies
        launch_pass_diffgrad_f32(gp, Q, true, st);   // spilled 384 B at q = 2 against 168 / 100 B apart)
      } else {
        launch_pass_fused_f32(b, Q, st);                        // both trials (exits when the state says one point)
        if (solo_ok || ondev) launch_pass_solo_f32(b, Q, st);   // slot 0 (solo) or Y after a slot-1 acceptance (fix)
        if (tiny_ok) {  // (the kernels exit unless tiny)
          launch_pass_diffgrad_f32(gp, Q, false, st);  // both trials
          launch_pass_diffgrad_f32(gp, Q, true, st);   // the first trial (when it leads the slot order)
        }
      }
      b.halt = &gdst.get()[par].stop;
      launch_reduce_rows(rowpart.get(), colpart.get(), strip_first.get(), n, nb, Q, nullptr, st, gpart.get(),
                         b.halt, f32parts(), losspart.get(), nchunks, kMaxCand, have_pre ? pre : nullptr);
      collect(b.halt);
    }
    issued += batch;
    GMDS_CUDA(cudaMemcpyAsync(&S, gdst.get() + par, sizeof S, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    if (std::getenv("GMDS_TRACE"))
      std::fprintf(stderr,
                   "[gmds] device_gd: it=%d step=%.3e f=%.9g pred=%d tiny=%d solo=%d pending=%d stop=%d miss=%d fix=%d rt=%d "
                   "halv=%d nextra=%d ndiff=%d t0=%.12g t1=%.12g gsq=%.6g\n",
                   S.it, S.step, S.f, S.pred, S.tiny, S.solo, S.pending, S.stop, S.solo_miss, S.fix, S.rt, S.halv,
                   S.nextra, S.ndiff, S.t0, S.t1, S.gsq);
    if (S.stop != 0) break;
  }
  // passes: the prime plus one per decision that continued (all accepted ones but a final stop)
  passes += (S.it - it) - (S.stop == 1 ? 1 : 0) + S.ndiff + S.nextra;  // + difference / fix / re-trial passes
  if (S.stop == 2 && S.solo_miss) {
    // the solo pass left the half step's loss unevaluated: one loss pass over both trial points
    // (slot 0 is recomputed to the same bits; losspart column 0 stays the loss at cand0)
    const double* Ys[2] = {cand[0].get(), cand[1].get()};
    const std::vector<double> raws = loss_raw(kind, delta, Ys, 2);
    S.t1 = raws[1];
  }
  if ((need_grad && init) || entry_hist) {  // f(Y0) written by the fix block / the entry value, re-based or not
    double f0 = 0.0;
    GMDS_CUDA(cudaMemcpyAsync(&f0, hist.get() + it, sizeof(double), cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    if (entry_hist) history.back() = f0; else history.push_back(f0);
  }
  if (S.it > it) {
    std::vector<double> h(static_cast<size_t>(S.it - it));
    GMDS_CUDA(cudaMemcpyAsync(h.data(), hist.get() + it + 1, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    history.insert(history.end(), h.begin(), h.end());
  }
  return S;
}

double Engine::scale_grad(double scale) {
  launch_scale_sqnorm(graw.get(), n * Q, scale, scal.get() + 4, sqpart.get(), st);
  double gsq = 0.0;
  GMDS_CUDA(cudaMemcpyAsync(&gsq, scal.get() + 4, sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return gsq;
}

// loss value of a kind from its raw pass sum (loss_value, embed.cpp:111-159)
double Engine::loss_of(int kind, double raw) const {
  switch (kind) {
    case kKruskal: return std::sqrt(raw / D->sum_sq);
    case kSammon: return (1.0 / D->sum) * raw;
    default: return raw;
  }
}

EngineLease acquire_engine(const gmds_dmat* D, int q, cudaStream_t st) {
  EngineLease L;
  L.D = D;
  {
    std::lock_guard<std::mutex> g(D->mu);
    for (size_t k = 0; k < D->engines.size(); ++k)
      if (D->engines[k].first == q && !D->busy[k]) {
        D->busy[k] = true;
        L.e = D->engines[k].second;
        L.slot = static_cast<int>(k);
        break;
      }
  }
  if (!L.e) {
    auto e = std::make_shared<Engine>(D, q, st);
    std::lock_guard<std::mutex> g(D->mu);
    D->engines.emplace_back(q, e);
    D->busy.push_back(true);
    L.e = e;
    L.slot = static_cast<int>(D->engines.size()) - 1;
  }
  L.e->st = st;
  L.e->W = nullptr;
  L.e->passes = 0;
  return L;
}

EngineLease::~EngineLease() {
  if (D && slot >= 0) {
    std::lock_guard<std::mutex> g(D->mu);
    D->busy[static_cast<size_t>(slot)] = false;
  }
}

// ---------------------------------------------------------------------------
namespace {

void not_sharded(const gmds_dmat* D, const char* who) {
  if (D && D->sharded())
    fail(GMDS_INVALID_INPUT, std::string(who) + ": row-sharded distance matrix (use the *_sharded entry points)");
}

void check_coords(const gmds_dmat* D, const double* coords, int q, const char* who) {
  // embed.cpp:15-21
  if (!D) fail(GMDS_INVALID_INPUT, std::string(who) + ": null distance matrix");
  if (q < 1) fail(GMDS_INVALID_INPUT, std::string(who) + ": coords have no columns");
  for (int64_t k = 0; k < D->n * q; ++k)
    if (!std::isfinite(coords[k])) fail(GMDS_INVALID_INPUT, std::string(who) + ": non-finite coordinates");
}

struct Resolved {
  int kind;
  double delta = 0.0;
  bool weighted = false;
};

// resolve_params (embed.cpp:54-109)
Resolved resolve(const gmds_dmat* D, int kind, double huber_delta, const double* weights, const char* who) {
  Resolved r;
  r.kind = kind;
  const std::string w(who);
  switch (kind) {
    case kKruskal:
      if (D->sum_sq <= 0.0) fail(GMDS_DEGENERATE_INPUT, w + ": all-zero distance matrix");
      break;
    case kHuber:
      if (std::isnan(huber_delta))
        fail(GMDS_INVALID_CONFIG,
             w + ": huber_delta auto mode is resolved by minimize_stress; pass an explicit delta here");
      if (!(huber_delta > 0.0)) fail(GMDS_INVALID_CONFIG, w + ": huber_delta must be > 0");
      r.delta = huber_delta;
      break;
    case kSammon:
      if (D->n >= 2 && !(D->min_off > 0.0))
        fail(GMDS_DEGENERATE_INPUT,
             w + ": Sammon loss requires strictly positive off-diagonal distances (deduplicate points first)");
      break;
    case kSmacof:
      if (weights) {
        const int64_t n = D->n;
        for (int64_t i = 0; i < n; ++i)
          for (int64_t j = i + 1; j < n; ++j) {
            const double a = weights[j * n + i], b = weights[i * n + j];
            if (!(a >= 0.0) || std::abs(a - b) > 0.0)
              fail(GMDS_INVALID_CONFIG, w + ": smacof_weights must be symmetric and nonnegative");
          }
        r.weighted = true;
      }
      break;
    default:
      fail(GMDS_INVALID_CONFIG, w + ": unknown stress kind");
  }
  return r;
}

// Packed image of the SMACOF weights (same layout and storage as D).
DevBuf<unsigned char> upload_weights(const gmds_dmat* D, const double* weights, cudaStream_t st) {
  const int64_t n = D->n;
  DevBuf<double> full(static_cast<size_t>(n * n));
  GMDS_CUDA(cudaMemcpyAsync(full.get(), weights, sizeof(double) * n * n, cudaMemcpyHostToDevice, st));
  DevBuf<unsigned char> out(static_cast<size_t>(packed_elems(n)) * dtype_size(D->storage));
  // weights(i, j) column-major == full[j*n + i]; the packer reads full[i*n + j] for i < j, i.e. weights(j, i):
  // symmetric by validation, so either triangle is the same value.
  pack_full(full.get(), n, D->storage, out.get(), st);
  GMDS_CUDA(cudaStreamSynchronize(st));
  return out;
}

struct IterResult {
  double loss = 0.0;
  bool converged = true;
  int iterations = 0;
  std::vector<double> history;
};

// gradient_descent (embed.cpp:222-272) with batched Armijo trials.  With fp32
// storage the first trial batch also carries both trial gradients, so an
// accepted trial hands the next iteration its gradient: one pass of D per
// iteration in the common case (step or step/2 accepted).
IterResult gradient_descent(Engine& E, const Resolved& rp, int max_iters, double rel_tol) {
  IterResult r;
  const int kind = rp.kind;
  // One host round trip per iteration in the common case: the gradient pass,
  // the scale, |g|^2 and the first trial pair (step, step/2) are queued
  // together (Engine::grad_and_trials).  Further halvings, when neither is
  // accepted, are loss-only passes of four (fp64) or two (fp32) trial points.
  // (A variant carrying both trial gradients in the trial pass was measured at
  // 800 us per pass vs 333 + 239 us for separate gradient and loss passes at
  // n = 20000, so trial passes compute losses only.)
  // Speculation (fp32 storage, q <= 4): the trial pass also carries the
  // gradient at the trial point predicted to be accepted (the same choice,
  // step or step/2, as the previous iteration -- Armijo acceptance is sticky),
  // so a correct prediction saves the next iteration's gradient pass: one
  // pass over D per iteration.  The arithmetic is unchanged; only the order
  // in which the two trial points sit in the pass differs.
  double* Yc[kMaxCand];
  double f = 0.0;
  double step = 1.0;
  constexpr double armijo = 1e-4;
  int it = 0;
  bool stalled = false;
  const bool spec = E.fused_ok() && !std::getenv("GMDS_NO_SPECULATION");
  bool have_grad = false;  // graw holds the raw gradient at Y (speculative mode)
  int pred = 0;            // 0: step accepted last time, 1: step/2
  // Device-resident loop (fp32 storage): iterations whose predicted trial is
  // accepted run without a host round trip (gd_step_kernel); GMDS_HOST_GD=1
  // keeps every decision on the host (same arithmetic, same trajectory).
  const bool devloop = spec && !std::getenv("GMDS_HOST_GD");
  const bool dev_nograd = devloop && !std::getenv("GMDS_NO_ONDEV");
  const bool precise_ok = !std::getenv("GMDS_NO_PRECISE");
  const bool diff_ok = !std::getenv("GMDS_NO_DIFF");  // GMDS_NO_DIFF=1: fp64-arithmetic re-evaluation instead
  for (; it < max_iters; ++it) {
    Engine::GradTrials gt;
    int slot_of[2] = {0, 1};  // slot of (step, step/2) in gt.trial / E.cand
    bool decided_on_device = false;
    // (without the gradient at Y -- the first iteration, or after an iteration decided here -- the device
    // loop primes itself with the gradient pass; GMDS_NO_ONDEV=1: the host takes that pass and the trials)
    if (devloop && (have_grad || dev_nograd)) {
      const bool first = r.history.empty();
      const GdState S = E.device_gd(kind, rp.delta, f, step, it, pred, max_iters, rel_tol, r.history,
                                    precise_ok ? kPreciseRel : 0.0, !have_grad, first);
      it = S.it;
      f = S.f;
      step = S.step;
      pred = S.pred;
      if (S.stop == 1) {
        stalled = S.stalled != 0;
        break;
      }
      // stop 2: iteration `it` is decided here, from the device's sums
      gt.raw = 0.0;
      gt.gsq = S.gsq;
      gt.trial[0] = S.t0;
      gt.trial[1] = S.t1;
      if (pred == 1) {
        slot_of[0] = 1;
        slot_of[1] = 0;
      }
      decided_on_device = true;
    }
    if (decided_on_device) {
    } else if (spec) {
      if (!have_grad) {
        const double raw0 = E.grad_raw(kind, rp.delta, E.Y.get());
        if (it == 0) {
          f = E.loss_of(kind, raw0);  // f = loss_value(coords) before the loop
          r.history.push_back(f);
        }
      }
      if (pred == 1) {
        slot_of[0] = 1;
        slot_of[1] = 0;
      }
      gt = E.fused_trials(kind, rp.delta, pred == 0 ? step : step * 0.5, pred == 0 ? step * 0.5 : step);
    } else {
      gt = E.grad_and_trials(kind, rp.delta, step, step * 0.5);
      if (it == 0) {
        f = E.loss_of(kind, gt.raw);  // f = loss_value(coords) before the loop
        r.history.push_back(f);
      }
    }
    const double grad_sq = gt.gsq;
    if (grad_sq <= 0.0) {
      stalled = true;
      break;
    }
    // fp32 storage resolves a change of the loss only above ~1e-7 relative (one pair's
    // e = D - dist changes by less than its ulp).  When both trials are within
    // kPreciseRel of f, the decision is taken on fp64-arithmetic losses of Y and both
    // trial points (one extra pass): the reference's first iterations, whose losses
    // change by ~1e-13, are then followed instead of stalling on equal fp32 sums.
    if (E.D->storage == GMDS_F32 && precise_ok) {
      const double tol = kPreciseRel * std::abs(f);
      // ... and whenever a tested trial's Armijo margin is inside that resolution
      const double f_step = E.loss_of(kind, gt.trial[slot_of[0]]), f_half = E.loss_of(kind, gt.trial[slot_of[1]]);
      if ((std::abs(E.loss_of(kind, gt.trial[0]) - f) <= tol && std::abs(E.loss_of(kind, gt.trial[1]) - f) <= tol) ||
          armijo_unresolved(f, step, grad_sq, f_step, f_half, tol)) {
        // Kruskal: the fp32 difference pass (the trial steps in slot order); other kinds:
        // fp64 arithmetic over the fp32 image
        std::vector<double> raws;
        if (kind == kKruskal && !E.W && diff_ok) {
          const double sf = (slot_of[0] == 0) ? step : step * 0.5, ss = (slot_of[0] == 0) ? step * 0.5 : step;
          raws = E.loss_diff(kind, sf, ss);
        } else {
          // trial points first: losspart column 0 keeps the first trial's loss, which the
          // next iteration's finish reads as the loss at the accepted point
          const double* Ys[3] = {E.cand[0].get(), E.cand[1].get(), E.Y.get()};
          const std::vector<double> r3 = E.loss_raw_precise(kind, rp.delta, Ys, 3);
          raws = {r3[2], r3[0], r3[1]};
        }
        f = E.loss_of(kind, raws[0]);
        if (!r.history.empty()) r.history.back() = f;  // the loss at Y, now in fp64 arithmetic
        gt.trial[0] = raws[1];
        gt.trial[1] = raws[2];
      }
    }
    double f_new = f;
    bool accepted = false;
    int acc_c = -1;
    for (int c = 0; c < 2 && !accepted; ++c) {  // step first, then step/2 (the reference's order)
      const double sc = (c == 0) ? step : step * 0.5;
      const double fc = E.loss_of(kind, gt.trial[slot_of[c]]);
      if (fc <= f - armijo * sc * grad_sq) {
        accepted = true;
        acc_c = slot_of[c];
        f_new = fc;
        step = sc;
        pred = c;
      }
    }
    if (spec) have_grad = accepted && acc_c == 0;  // the fused pass computed the gradient at cand[0]
    if (!accepted) step *= 0.25;
    for (int halvings = 2; halvings < 60 && !accepted;) {
      Steps s{};
      s.n = std::min(E.D->storage == GMDS_F32 ? 2 : kMaxCand, 60 - halvings);
      double sv = step;
      for (int c = 0; c < s.n; ++c) {
        s.v[c] = sv;
        sv *= 0.5;
      }
      for (int c = 0; c < kMaxCand; ++c) Yc[c] = E.cand[c].get();
      launch_axpy_cand(E.Y.get(), E.graw.get(), E.n * E.Q, s, Yc, E.st);
      const std::vector<double> raws = E.loss_raw(kind, rp.delta, Yc, s.n);
      for (int c = 0; c < s.n; ++c) {
        const double fc = E.loss_of(kind, raws[c]);
        if (fc <= f - armijo * s.v[c] * grad_sq) {
          accepted = true;
          acc_c = c;
          f_new = fc;
          step = s.v[c];
          break;
        }
      }
      if (!accepted) step = sv;  // halved s.n times
      halvings += s.n;
    }
    if (!accepted) {
      stalled = true;
      break;
    }
    if (std::getenv("GMDS_TRACE"))
      std::fprintf(stderr, "[gmds] host gd: it=%d step=%.4e slot=%d pred=%d have_grad=%d from_device=%d f_new=%.12g\n", it,
                   step, acc_c, pred, have_grad ? 1 : 0, decided_on_device ? 1 : 0, f_new);
    std::swap(E.Y, E.cand[acc_c]);
    if (have_grad) std::swap(E.graw, E.gnext);
    r.history.push_back(f_new);
    const double decrease = (f - f_new) / std::max(f, kTiny);
    f = f_new;
    step *= 2.0;
    if (decrease < rel_tol) {
      ++it;
      stalled = true;
      break;
    }
  }
  r.loss = f;
  r.iterations = it;
  r.converged = stalled || it < max_iters;
  return r;
}

// smacof_iterate (embed.cpp:296-347).  pass(Z) -> (loss(Z), B(Z) Z).
IterResult smacof_iterate(Engine& E, const Resolved& rp, const double* dVpinv, int max_iters, double rel_tol) {
  IterResult r;
  const int64_t n = E.n;
  double* next = E.cand[0].get();
  auto transform = [&](double raw_loss_unused) {
    (void)raw_loss_unused;
    if (!dVpinv) {
      launch_scale(E.graw.get(), n * E.Q, static_cast<double>(n), next, E.st);  // (B Z) / n
    } else {
      launch_vpinv_apply(dVpinv, E.graw.get(), n, E.Q, next, E.st);  // X+ = V^+ (B Z)
    }
  };
  double f = E.grad_raw(kGuttman, 0.0, E.Y.get());  // loss(Z0) and B(Z0) Z0
  transform(f);
  r.history.push_back(f);
  int it = 0;
  bool reached = false;
  for (; it < max_iters; ++it) {
    std::swap(E.Y, E.cand[0]);  // coords = next
    next = E.cand[0].get();
    const double f_new = E.grad_raw(kGuttman, 0.0, E.Y.get());  // loss(next) (+ next transform)
    r.history.push_back(f_new);
    const double decrease = (f - f_new) / std::max(f, kTiny);
    f = f_new;
    if (decrease < rel_tol) {
      ++it;
      reached = true;
      break;
    }
    if (it + 1 < max_iters) transform(f_new);
  }
  r.loss = f;
  r.iterations = it;
  r.converged = reached || it < max_iters;
  return r;
}

// V^+ for weighted SMACOF (embed.cpp:303-322), n x n column-major on the device.
DevBuf<double> weights_pinv(const double* weights, int64_t n, cudaStream_t st);

}  // namespace

namespace {

// The reference's bookkeeping after the eigensolver (embed.cpp:428-458): the
// clamped mass over the full spectrum lam (ascending, n values), then for the
// top q eigenpairs the sign rule (largest-|v| entry positive, first index
// wins) and coords = v sqrt(max(lambda, 0)).  V: the top q eigenvectors,
// column c = the c-th largest.
void classical_finish(int64_t n, int q, const std::vector<double>& lam, const double* V, double* coords,
                      double* eigvals, int* clamped_count, double* clamped_mass) {
  double negative_mass = 0.0, total_mass = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    total_mass += std::abs(lam[i]);
    if (lam[i] < 0.0) negative_mass += -lam[i];
  }
  *clamped_mass = total_mass > 0.0 ? negative_mass / total_mass : 0.0;
  *clamped_count = 0;
  for (int c = 0; c < q; ++c) {
    const double lambda = lam[n - 1 - c];
    eigvals[c] = lambda;
    const double* v = V + static_cast<size_t>(c) * n;
    int64_t arg = 0;
    double best = std::abs(v[0]);
    for (int64_t i = 1; i < n; ++i)
      if (std::abs(v[i]) > best) {
        best = std::abs(v[i]);
        arg = i;
      }
    const double sgn = (v[arg] < 0.0) ? -1.0 : 1.0;
    if (lambda < 0.0) ++*clamped_count;
    const double sc = std::sqrt(std::max(lambda, 0.0));
    for (int64_t i = 0; i < n; ++i) coords[static_cast<size_t>(c) * n + i] = (sgn * v[i]) * sc;
  }
}

void check_classical_q(int64_t n, int q) {
  if (q < 1 || q > n - 1)
    fail(GMDS_INVALID_INPUT, "classical_mds: target dimension must satisfy 1 <= p <= n-1, got p=" +
                                 std::to_string(q) + " with n=" + std::to_string(n));
}

double kruskal_at(const gmds_dmat* D, const double* coords, int q, cudaStream_t st) {
  if (!(D->sum_sq > 0.0)) return 0.0;
  EngineLease L = acquire_engine(D, q, st);
  Engine& E = *L;
  E.upload(coords, E.Y.get());
  const double* y = E.Y.get();
  return E.loss_of(kKruskal, E.loss_raw(kKruskal, 0.0, &y, 1)[0]);
}

}  // namespace

// classical_mds (embed.cpp:415-460)
void classical_mds_dev(const gmds_dmat* D, int q, double* coords, double* eigvals, int* clamped_count,
                       double* clamped_mass, double* stress, cudaStream_t st) {
  const int64_t n = D->n;
  check_classical_q(n, q);
  DevBuf<double> B(static_cast<size_t>(n * n));
  unpack_full(D->ptr(), D->storage, n, B.get(), true, st);  // S = D o D
  double_center_dev(B.get(), n, st);
  cusolverDnHandle_t h = solver_handle(st);
  DevBuf<double> w(static_cast<size_t>(n));
  int lwork = 0;
  if (cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), B.get(),
                                  static_cast<int>(n), w.get(), &lwork) != CUSOLVER_STATUS_SUCCESS)
    fail(GMDS_NUMERIC_FAILURE, "classical_mds: eigensolver failed");
  DevBuf<double> work(static_cast<size_t>(lwork));
  DevBuf<int> info(1);
  if (cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), B.get(),
                       static_cast<int>(n), w.get(), work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
    fail(GMDS_NUMERIC_FAILURE, "classical_mds: eigensolver failed");
  count_launch();
  int hinfo = 0;
  std::vector<double> lam(static_cast<size_t>(n));
  GMDS_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(lam.data(), w.get(), n * sizeof(double), cudaMemcpyDeviceToHost, st));
  std::vector<double> V(static_cast<size_t>(n) * q);
  for (int c = 0; c < q; ++c)
    GMDS_CUDA(cudaMemcpyAsync(V.data() + static_cast<size_t>(c) * n, B.get() + (n - 1 - c) * n, n * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0) fail(GMDS_NUMERIC_FAILURE, "classical_mds: eigensolver failed");
  classical_finish(n, q, lam, V.data(), coords, eigvals, clamped_count, clamped_mass);
  if (stress) *stress = kruskal_at(D, coords, q, st);
}

// classical_mds of several same-size matrices (the grid cells of one tune_nu
// fold): one batched eigensolver call (cusolverDnXsyevBatched) instead of one
// dense solve per cell.  Results per matrix as classical_mds_dev; false when
// the batched solver is not available for this size (caller goes one by one).
bool classical_mds_batch_dev(const std::vector<const gmds_dmat*>& Ds, int q, std::vector<std::vector<double>>& coords,
                             std::vector<double>& stress, cudaStream_t st) {
  const int64_t n = Ds[0]->n;
  check_classical_q(n, q);
  const int64_t bs = static_cast<int64_t>(Ds.size());
  const size_t nn = static_cast<size_t>(n) * n;
  DevBuf<double> B(nn * bs), w(static_cast<size_t>(n * bs));
  for (int64_t b = 0; b < bs; ++b) {
    unpack_full(Ds[b]->ptr(), Ds[b]->storage, n, B.get() + b * nn, true, st);
    double_center_dev(B.get() + b * nn, n, st);
  }
  cusolverDnHandle_t h = solver_handle(st);
  cusolverDnParams_t params = nullptr;
  if (cusolverDnCreateParams(&params) != CUSOLVER_STATUS_SUCCESS) return false;
  struct P {
    cusolverDnParams_t p;
    ~P() { cusolverDnDestroyParams(p); }
  } pg{params};
  size_t dws = 0, hws = 0;
  if (cusolverDnXsyevBatched_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F,
                                        B.get(), n, CUDA_R_64F, w.get(), CUDA_R_64F, &dws, &hws,
                                        bs) != CUSOLVER_STATUS_SUCCESS)
    return false;
  DevBuf<unsigned char> dwork(std::max<size_t>(dws, 1));
  std::vector<unsigned char> hwork(std::max<size_t>(hws, 1));
  DevBuf<int> info(static_cast<size_t>(bs));
  if (cusolverDnXsyevBatched(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, B.get(), n,
                             CUDA_R_64F, w.get(), CUDA_R_64F, dwork.get(), dws, hwork.data(), hws, info.get(),
                             bs) != CUSOLVER_STATUS_SUCCESS)
    return false;
  count_launch();
  std::vector<int> hinfo(static_cast<size_t>(bs));
  std::vector<double> lam(static_cast<size_t>(n * bs));
  std::vector<double> V(static_cast<size_t>(n) * q * bs);
  GMDS_CUDA(cudaMemcpyAsync(hinfo.data(), info.get(), bs * sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(lam.data(), w.get(), lam.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  for (int64_t b = 0; b < bs; ++b)
    for (int c = 0; c < q; ++c)
      GMDS_CUDA(cudaMemcpyAsync(V.data() + (static_cast<size_t>(b) * q + c) * n, B.get() + b * nn + (n - 1 - c) * n,
                                n * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  for (int64_t b = 0; b < bs; ++b)
    if (hinfo[b] != 0) fail(GMDS_NUMERIC_FAILURE, "classical_mds: eigensolver failed");
  coords.assign(static_cast<size_t>(bs), std::vector<double>(static_cast<size_t>(n) * q));
  stress.assign(static_cast<size_t>(bs), 0.0);
  std::vector<double> ev(static_cast<size_t>(q));
  for (int64_t b = 0; b < bs; ++b) {
    const std::vector<double> lb(lam.begin() + b * n, lam.begin() + (b + 1) * n);
    int cc = 0;
    double cm = 0.0;
    classical_finish(n, q, lb, V.data() + static_cast<size_t>(b) * q * n, coords[b].data(), ev.data(), &cc, &cm);
    stress[b] = kruskal_at(Ds[b], coords[b].data(), q, st);
  }
  return true;
}

namespace {

DevBuf<double> weights_pinv(const double* weights, int64_t n, cudaStream_t st) {
  std::vector<double> V(static_cast<size_t>(n * n), 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (i == j) continue;
      const double w = weights[j * n + i];  // column-major (i, j)
      V[j * n + i] = -w;
      V[i * n + i] += w;
    }
  DevBuf<double> dV(static_cast<size_t>(n * n));
  GMDS_CUDA(cudaMemcpyAsync(dV.get(), V.data(), V.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  cusolverDnHandle_t h = solver_handle(st);
  DevBuf<double> w(static_cast<size_t>(n));
  int lwork = 0;
  cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), dV.get(),
                              static_cast<int>(n), w.get(), &lwork);
  DevBuf<double> work(static_cast<size_t>(lwork));
  DevBuf<int> info(1);
  if (cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), dV.get(),
                       static_cast<int>(n), w.get(), work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
    fail(GMDS_NUMERIC_FAILURE, "smacof: eigensolver failed on V");
  count_launch();
  std::vector<double> lam(static_cast<size_t>(n)), U(static_cast<size_t>(n * n));
  int hinfo = 0;
  GMDS_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(lam.data(), w.get(), n * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(U.data(), dV.get(), U.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0) fail(GMDS_NUMERIC_FAILURE, "smacof: eigensolver failed on V");
  double amax = 0.0;
  for (double l : lam) amax = std::max(amax, std::abs(l));
  const double cutoff = 1e-12 * std::max(amax, 1.0);
  // pinv = U diag(inv) U^T (host; weighted SMACOF is a small-n feature)
  std::vector<double> P(static_cast<size_t>(n * n), 0.0);
  for (int64_t k = 0; k < n; ++k) {
    if (!(lam[k] > cutoff)) continue;
    const double inv = 1.0 / lam[k];
    const double* u = U.data() + k * n;
    for (int64_t j = 0; j < n; ++j) {
      const double uj = u[j] * inv;
      for (int64_t i = 0; i < n; ++i) P[j * n + i] += u[i] * uj;
    }
  }
  DevBuf<double> dP(static_cast<size_t>(n * n));
  GMDS_CUDA(cudaMemcpyAsync(dP.get(), P.data(), P.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return dP;
}

// The whole fit in one cooperative persistent kernel (small_fit.cu): same control flow as
// gradient_descent / smacof_iterate above, no host round trip per pass.
bool small_fit(const gmds_dmat* D, int q, const gmds_stress_cfg& cfg, const Resolved& rp,
               const std::vector<double>& init, gmds_fit_result* res, cudaStream_t st) {
  const int64_t n = D->n;
  const int grid = small_fit_grid(n);
  if (grid == 0) return false;
  std::shared_ptr<DevBuf<double>> dense;
  {
    std::lock_guard<std::mutex> g(D->mu);
    if (!D->dense) {
      auto b = std::make_shared<DevBuf<double>>(static_cast<size_t>(n * n));
      unpack_full(D->ptr(), D->storage, n, b->get(), false, st);
      // complete before publishing: another thread's fit on another stream may read it next
      GMDS_CUDA(cudaStreamSynchronize(st));
      D->dense = b;
    }
    dense = D->dense;
  }
  const size_t nq = static_cast<size_t>(n) * q;
  const size_t hist = static_cast<size_t>(cfg.max_iters) + 2;
  // Yout | history | out | 4 slots | partials
  DevBuf<double> buf(nq + hist + 1 + 4 * nq + 8 * static_cast<size_t>(grid));
  DevBuf<int> ibuf(4);
  std::vector<double> h(nq);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < q; ++k) h[static_cast<size_t>(i) * q + k] = init[static_cast<size_t>(k) * n + i];
  SmallFitArgs a{};
  a.D = dense->get();
  a.Yout = buf.get();
  a.history = a.Yout + nq;
  a.out = a.history + hist;
  for (int s = 0; s < 4; ++s) a.buf[s] = a.out + 1 + s * nq;
  a.lossp = a.buf[3] + nq;
  a.iout = ibuf.get();
  GMDS_CUDA(cudaMemcpyAsync(a.buf[0], h.data(), nq * sizeof(double), cudaMemcpyHostToDevice, st));
  a.n = static_cast<int>(n);
  a.kind = rp.kind;
  a.delta = rp.delta;
  a.sum = D->sum;
  a.sum_sq = D->sum_sq;
  a.max_iters = cfg.max_iters;
  a.rel_tol = cfg.rel_tol;
  launch_small_fit(a, q, grid, st);
  std::vector<double> back(nq + hist + 1);
  int iv[4];
  GMDS_CUDA(cudaMemcpyAsync(back.data(), a.Yout, back.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(iv, a.iout, sizeof(iv), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < q; ++k) res->coords[static_cast<size_t>(k) * n + i] = back[static_cast<size_t>(i) * q + k];
  res->history_len = iv[2];
  if (res->history)
    for (int64_t t = 0; t < std::min<int64_t>(res->history_len, res->history_cap); ++t)
      res->history[t] = back[nq + static_cast<size_t>(t)];
  res->iterations = iv[0];
  res->converged = iv[1];
  res->stress = back[nq + hist];
  res->huber_delta = (cfg.kind == GMDS_HUBER) ? cfg.huber_delta : 0.0;
  res->passes = iv[3];
  return true;
}

}  // namespace

// minimize_stress (embed.cpp:491-532)
void minimize_stress_dev(const gmds_dmat* D, int q, const gmds_stress_cfg& cfg, const double* Y0, gmds_fit_result* res,
                         cudaStream_t st, const double* init_cache) {
  if (cfg.max_iters < 1) fail(GMDS_INVALID_CONFIG, "minimize_stress: max_iters must be >= 1");
  if (!(cfg.rel_tol > 0.0)) fail(GMDS_INVALID_CONFIG, "minimize_stress: rel_tol must be > 0");
  const int64_t n = D->n;
  std::vector<double> init(static_cast<size_t>(n) * q);
  if (Y0) {
    std::memcpy(init.data(), Y0, init.size() * sizeof(double));
  } else if (init_cache) {
    std::memcpy(init.data(), init_cache, init.size() * sizeof(double));
  } else {
    std::vector<double> ev(static_cast<size_t>(q));
    int cc = 0;
    double cm = 0.0;
    // classical init: only the coordinates are used, so large n takes the
    // top-q subspace solver instead of the O(n^3) dense one
    const char* mode = std::getenv("GMDS_CLASSICAL");
    const bool dense = mode ? std::string(mode) == "dense" : n <= kDenseEigMaxN;
    bool done = false;
    if (!dense && q <= 16) {
      try {
        int its = 0;
        classical_topq_dev(D, q, 1e-10, 2000, init.data(), ev.data(), &cc, &its, st);
        done = true;
      } catch (const Failure& e) {
        if (e.status != GMDS_NUMERIC_FAILURE) throw;  // not separated / not converged: dense path
      }
    }
    if (!done) classical_mds_dev(D, q, init.data(), ev.data(), &cc, &cm, nullptr, st);
  }
  if (cfg.kind == GMDS_HUBER && std::isnan(cfg.huber_delta)) {
    const double med = packed_median(D->ptr(), D->storage, n, st);
    const double base = med > 0.0 ? med : 1.0;
    double best_ks = std::numeric_limits<double>::infinity();
    std::vector<double> best_coords(static_cast<size_t>(n) * q), coords(static_cast<size_t>(n) * q);
    std::vector<double> best_hist;
    gmds_fit_result best{};
    for (const double factor : {0.5, 1.0, 2.0}) {
      gmds_stress_cfg trial = cfg;
      trial.huber_delta = factor * base;
      std::vector<double> hist(static_cast<size_t>(cfg.max_iters) + 2);
      gmds_fit_result rr{};
      rr.coords = coords.data();
      rr.history = hist.data();
      rr.history_cap = static_cast<int64_t>(hist.size());
      minimize_stress_dev(D, q, trial, nullptr, &rr, st, init.data());
      // kruskal_stress(e.coords, D) (embed.cpp:508)
      if (D->sum_sq <= 0.0) fail(GMDS_DEGENERATE_INPUT, "kruskal_stress: all-zero distance matrix");
      EngineLease L = acquire_engine(D, q, st);
      Engine& E = *L;
      E.upload(coords.data(), E.Y.get());
      const double* y = E.Y.get();
      const double ks = E.loss_of(kKruskal, E.loss_raw(kKruskal, 0.0, &y, 1)[0]);
      if (ks < best_ks) {
        best_ks = ks;
        best = rr;
        best_coords = coords;
        best_hist.assign(hist.begin(), hist.begin() + std::min<int64_t>(rr.history_len, rr.history_cap));
      }
    }
    std::memcpy(res->coords, best_coords.data(), best_coords.size() * sizeof(double));
    res->history_len = best.history_len;
    if (res->history)
      for (int64_t t = 0; t < std::min<int64_t>(static_cast<int64_t>(best_hist.size()), res->history_cap); ++t)
        res->history[t] = best_hist[static_cast<size_t>(t)];
    res->iterations = best.iterations;
    res->converged = best.converged;
    res->stress = best.stress;
    res->huber_delta = best.huber_delta;
    return;
  }
  const Resolved rp = resolve(D, cfg.kind, cfg.huber_delta, cfg.smacof_weights, "minimize_stress");
  if (!rp.weighted && small_fit_supported(n, q) && !std::getenv("GMDS_NO_SMALL_FIT")) {
    if (small_fit(D, q, cfg, rp, init, res, st)) return;
  }
  EngineLease L = acquire_engine(D, q, st);
  Engine& E = *L;
  DevBuf<unsigned char> W;
  if (rp.weighted) {
    W = upload_weights(D, cfg.smacof_weights, st);
    E.W = W.get();
  }
  E.upload(init.data(), E.Y.get());
  IterResult r;
  if (cfg.kind == GMDS_SMACOF) {
    DevBuf<double> vp;
    if (rp.weighted) vp = weights_pinv(cfg.smacof_weights, n, st);
    r = smacof_iterate(E, rp, rp.weighted ? vp.get() : nullptr, cfg.max_iters, cfg.rel_tol);
  } else {
    r = gradient_descent(E, rp, cfg.max_iters, cfg.rel_tol);
  }
  E.download(E.Y.get(), res->coords);
  res->history_len = static_cast<int64_t>(r.history.size());
  if (res->history)
    for (int64_t t = 0; t < std::min<int64_t>(res->history_len, res->history_cap); ++t)
      res->history[t] = r.history[static_cast<size_t>(t)];
  res->iterations = r.iterations;
  res->converged = r.converged ? 1 : 0;
  res->stress = r.loss;
  res->huber_delta = (cfg.kind == GMDS_HUBER) ? cfg.huber_delta : 0.0;
  res->passes = E.passes;
}

// DistanceMatrix::from_matrix (metrics.cpp:169-191) on a host column-major matrix.
std::vector<double> validate_full(const double* M, int64_t n) {
  if (n < 1) fail(GMDS_INVALID_INPUT, "DistanceMatrix: matrix is empty");
  double scale = 0.0;
  bool has_nan = false;
  for (int64_t k = 0; k < n * n; ++k) {
    if (std::isnan(M[k])) has_nan = true;
    scale = std::max(scale, std::abs(M[k]));
  }
  (void)has_nan;
  const double tol = 1e-12 * std::max(scale, 1.0);
  std::vector<double> out(static_cast<size_t>(n * n), 0.0);  // row-major image of the validated matrix
  for (int64_t i = 0; i < n; ++i) {
    if (std::abs(M[i * n + i]) > tol) fail(GMDS_INVALID_INPUT, "DistanceMatrix: nonzero diagonal");
    for (int64_t j = i + 1; j < n; ++j) {
      const double a = M[j * n + i];  // (i, j) column-major
      const double b = M[i * n + j];  // (j, i)
      if (!std::isfinite(a) || !std::isfinite(b)) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
      if (std::abs(a - b) > tol) fail(GMDS_INVALID_INPUT, "DistanceMatrix: asymmetric entries");
      if (a < -tol || b < -tol) fail(GMDS_INVALID_INPUT, "DistanceMatrix: negative entry");
      const double v = std::max(0.0, a);
      out[i * n + j] = v;
      out[j * n + i] = v;
    }
  }
  return out;
}

void dmat_finish(gmds_dmat* d, cudaStream_t st) {  // stats used by resolve_params
  const DStats s = packed_stats(d->ptr(), d->storage, d->n, st);
  d->sum_sq = s.sum_sq;
  d->sum = s.sum;
  d->min_off = d->n >= 2 ? s.min_off : 0.0;
  d->max_val = d->n >= 2 ? std::max(0.0, s.max_off) : 0.0;
  d->stats = true;
}

// DistanceMatrix::matrix() for a device handle: the full fp64 matrix into caller (pageable)
// host memory without a device-side n x n image or a pageable cudaMemcpy.  Row stripes of
// ~64 MB are unpacked on the device, copied into pinned staging (two buffers, so stripe s + 1
// moves while stripe s is copied out) and spread into the destination by host threads.
void download_full(const gmds_dmat* d, double* dst, cudaStream_t st) {
  const int64_t n = d->n;
  const int64_t R = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(64) << 20) / (8 * n)));
  const size_t stripe = static_cast<size_t>(R * n);
  struct Pinned {
    double* p[2] = {nullptr, nullptr};
    size_t cap = 0;
    ~Pinned() {
      for (double* q : p)
        if (q) cudaFreeHost(q);
    }
  };
  static thread_local Pinned pin;
  if (pin.cap < stripe) {
    for (double*& q : pin.p) {
      if (q) cudaFreeHost(q);
      q = nullptr;
      GMDS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&q), stripe * sizeof(double), cudaHostAllocDefault));
    }
    pin.cap = stripe;
  }
  DevBuf<double> dev[2];
  for (auto& b : dev) b.alloc(stripe);
  cudaEvent_t ev[2];
  for (auto& e : ev) GMDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Ev {
    cudaEvent_t* e;
    ~Ev() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } evg{ev};
  const int64_t nstripes = ceil_div(n, R);
  // The destination is usually a fresh pageable allocation (an Eigen matrix): its 4 KB first-touch
  // faults add to the copy-out.  Ask for huge pages; optionally populate the stripes ahead of the
  // copy threads (MADV_POPULATE_WRITE leaves contents alone; both hints may be refused -- ignored).
  const uintptr_t page = 4096;
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(dst) + page - 1) & ~(page - 1);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(dst) + static_cast<size_t>(n) * n * sizeof(double)) & ~(page - 1);
  std::atomic<int64_t> pf_next{0};
  std::vector<std::thread> pf;
  // GMDS_PREFAULT = "none" | "huge" (default) | "pop" | "both".  Measured on the B200 box (metric shape,
  // 3.2 GB, tools/facade_ab.py): none 437 ms, huge 425, pop 723, both 534 per facade call -- the copy-out
  // is bound by host memory traffic, not by faults, so only the huge-page hint stays on.
  const char* pfm = std::getenv("GMDS_PREFAULT");
  const bool pf_huge = !pfm || !std::strcmp(pfm, "huge") || !std::strcmp(pfm, "both");
  const bool pf_pop = pfm && (!std::strcmp(pfm, "pop") || !std::strcmp(pfm, "both"));
  if (a1 > a0 && (pf_huge || pf_pop)) {
    if (pf_huge) madvise(reinterpret_cast<void*>(a0), a1 - a0, MADV_HUGEPAGE);
    for (int t = 0; t < (pf_pop ? 4 : 0); ++t)
      pf.emplace_back([&, a0, a1] {
        for (;;) {
          const int64_t s = pf_next.fetch_add(1);
          if (s >= nstripes) break;
          const uintptr_t b0 = std::max(a0, (reinterpret_cast<uintptr_t>(dst + static_cast<size_t>(s * R * n)) + page - 1) & ~(page - 1));
          const uintptr_t b1 = std::min(a1, reinterpret_cast<uintptr_t>(dst + static_cast<size_t>(std::min(n, (s + 1) * R) * n)) & ~(page - 1));
          if (b1 > b0 && madvise(reinterpret_cast<void*>(b0), b1 - b0, 23 /* MADV_POPULATE_WRITE */) != 0) break;
        }
      });
  }
  struct Join {
    std::vector<std::thread>& v;
    ~Join() {
      for (auto& x : v) x.join();
    }
  } pfj{pf};
  auto enqueue = [&](int64_t s) {
    const int b = static_cast<int>(s & 1);
    const int64_t r0 = s * R, r1 = std::min(n, r0 + R);
    unpack_rows(d->ptr(), d->storage, n, r0, r1, dev[b].get(), st);
    GMDS_CUDA(cudaMemcpyAsync(pin.p[b], dev[b].get(), static_cast<size_t>((r1 - r0) * n) * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaEventRecord(ev[b], st));
  };
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  enqueue(0);
  for (int64_t s = 0; s < nstripes; ++s) {
    if (s + 1 < nstripes) enqueue(s + 1);  // its buffer's previous copy-out (stripe s - 1) is done
    const int b = static_cast<int>(s & 1);
    GMDS_CUDA(cudaEventSynchronize(ev[b]));
    const int64_t r0 = s * R, r1 = std::min(n, r0 + R);
    const size_t count = static_cast<size_t>((r1 - r0) * n);
    const double* src = pin.p[b];
    double* out = dst + static_cast<size_t>(r0 * n);
    const size_t per = (count + hw - 1) / hw;
    std::vector<std::thread> th;
    for (unsigned t = 1; t < hw && t * per < count; ++t)
      th.emplace_back([=] { std::memcpy(out + t * per, src + t * per, std::min(per, count - t * per) * sizeof(double)); });
    std::memcpy(out, src, std::min(per, count) * sizeof(double));
    for (auto& x : th) x.join();
  }
}

}  // namespace gmds

using namespace gmds;

extern "C" {

gmds_status gmds_dmat_from_host(const double* D, int64_t n, gmds_dtype storage, gmds_dmat** out) {
  return guard([&] {
    *out = nullptr;
    std::vector<double> full = validate_full(D, n);
    require_device();
    Stream st;
    auto* d = new gmds_dmat();
    d->n = n;
    d->storage = storage;
    try {
      d->buf.alloc(static_cast<size_t>(packed_elems(n)) * dtype_size(storage));
      DevBuf<double> dfull(full.size());
      GMDS_CUDA(cudaMemcpyAsync(dfull.get(), full.data(), full.size() * sizeof(double), cudaMemcpyHostToDevice, st.s));
      pack_full(dfull.get(), n, storage, d->buf.get(), st.s);
      dmat_finish(d, st.s);
    } catch (...) {
      delete d;
      throw;
    }
    *out = d;
  });
}

static void dmat_gini_common(const void* dX, gmds_dtype xt, int64_t n, int64_t p, double nu, gmds_dtype storage,
                             gmds_dmat** out, cudaStream_t st) {
  auto* d = new gmds_dmat();
  d->n = n;
  d->storage = storage;
  try {
    const size_t bytes = static_cast<size_t>(packed_elems(n)) * dtype_size(storage);
    d->buf.alloc(bytes);
    GMDS_CUDA(cudaMemsetAsync(d->buf.get(), 0, bytes, st));
    DevBuf<int> flag(1);
    GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    run_gini(dX, xt, n, p, &nu, 1, storage, 1, d->buf.get(), 0, 1, st, flag.get());
    check_flag(flag.get(), st);
    dmat_finish(d, st);
  } catch (...) {
    delete d;
    throw;
  }
  *out = d;
}

gmds_status gmds_dmat_gini(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, double nu,
                           gmds_dtype storage, gmds_dmat** out) {
  return guard([&] {
    *out = nullptr;
    check_nu(nu);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    require_device();
    Stream st;
    std::vector<float> narrowed;
    X = narrow_exact_f32(X, xt, n * p, narrowed);
    DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
    dmat_gini_common(dX.get(), xt, n, p, nu, storage, out, st.s);
  });
}

gmds_status gmds_dmat_gini_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, double nu, gmds_dtype storage,
                                  gmds_dmat** out) {
  return guard([&] {
    *out = nullptr;
    check_nu(nu);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    require_device();
    Stream st;
    dmat_gini_common(dX, xt, n, p, nu, storage, out, st.s);
  });
}

gmds_status gmds_dmat_download(const gmds_dmat* d, double* D_full) {
  return guard([&] {
    if (!d) fail(GMDS_INVALID_INPUT, "dmat_download: null handle");
    if (d->sharded()) fail(GMDS_INVALID_INPUT, "dmat_download: row-sharded distance matrix");
    Stream st;
    download_full(d, D_full, st.s);
  });
}

int64_t gmds_dmat_n(const gmds_dmat* d) { return d ? d->n : 0; }

gmds_status gmds_dmat_stats(const gmds_dmat* d, double* stats4) {
  return guard([&] {
    if (!d) fail(GMDS_INVALID_INPUT, "dmat_stats: null handle");
    stats4[0] = d->sum_sq;
    stats4[1] = d->sum;
    stats4[2] = d->min_off;
    stats4[3] = d->max_val;
  });
}
void gmds_dmat_free(gmds_dmat* d) { delete d; }

gmds_status gmds_kruskal_stress(const gmds_dmat* D, const double* coords, int32_t q, double* out) {
  return guard([&] {
    check_coords(D, coords, q, "kruskal_stress");
    not_sharded(D, "kruskal_stress");
    if (D->sum_sq <= 0.0) fail(GMDS_DEGENERATE_INPUT, "kruskal_stress: all-zero distance matrix");
    Stream st;
    EngineLease L = acquire_engine(D, q, st.s);
    Engine& E = *L;
    E.upload(coords, E.Y.get());
    const double* y = E.Y.get();
    *out = E.loss_of(kKruskal, E.loss_raw(kKruskal, 0.0, &y, 1)[0]);
  });
}

gmds_status gmds_stress_loss(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q, double huber_delta,
                             const double* weights, double* out) {
  return guard([&] {
    check_coords(D, coords, q, "stress_loss");
    not_sharded(D, "stress_loss");
    const Resolved rp = resolve(D, kind, huber_delta, weights, "stress_loss");
    Stream st;
    EngineLease L = acquire_engine(D, q, st.s);
    Engine& E = *L;
    DevBuf<unsigned char> W;
    if (rp.weighted) {
      W = upload_weights(D, weights, st.s);
      E.W = W.get();
    }
    E.upload(coords, E.Y.get());
    const double* y = E.Y.get();
    *out = E.loss_of(kind, E.loss_raw(kind, rp.delta, &y, 1)[0]);
  });
}

gmds_status gmds_stress_gradient(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q,
                                 double huber_delta, const double* weights, double* grad) {
  return guard([&] {
    check_coords(D, coords, q, "stress_gradient");
    not_sharded(D, "stress_gradient");
    const Resolved rp = resolve(D, kind, huber_delta, weights, "stress_gradient");
    Stream st;
    EngineLease L = acquire_engine(D, q, st.s);
    Engine& E = *L;
    DevBuf<unsigned char> W;
    if (rp.weighted) {
      W = upload_weights(D, weights, st.s);
      E.W = W.get();
    }
    E.upload(coords, E.Y.get());
    const double raw = E.grad_raw(kind, rp.delta, E.Y.get());
    double scale = 1.0;
    if (kind == kKruskal) {
      const double ks = std::sqrt(raw / D->sum_sq);
      scale = (ks <= 0.0) ? 0.0 : 1.0 / (ks * D->sum_sq);
    } else if (kind == kSammon) {
      scale = 2.0 * (1.0 / D->sum);
    }
    E.scale_grad(scale);
    E.download(E.graw.get(), grad);
  });
}

gmds_status gmds_stress_partial(int32_t kind, const gmds_dmat* D, const double* coords, int32_t q, double huber_delta,
                                int32_t shard, int32_t nshards, double* raw_loss, double* raw_grad) {
  return guard([&] {
    check_coords(D, coords, q, "stress_partial");
    not_sharded(D, "stress_partial");
    if (nshards < 1 || shard < 0 || shard >= nshards) fail(GMDS_INVALID_CONFIG, "stress_partial: bad shard");
    if (q > 4) fail(GMDS_INVALID_INPUT, "stress_partial: sharded passes support q <= 4");
    // resolve_params (embed.cpp:54-109): NaN / non-positive Huber delta, unknown kinds,
    // all-zero D (Kruskal), non-positive off-diagonals (Sammon) are rejected as the reference does
    const Resolved rp = (kind == kGuttman) ? Resolved{kGuttman} : resolve(D, kind, huber_delta, nullptr, "stress_partial");
    Stream st;
    EngineLease L = acquire_engine(D, q, st.s);
    Engine& E = *L;
    E.upload(coords, E.Y.get());
    // this shard's chunks: a contiguous, pair-balanced slice of the chunk list
    *raw_loss = E.grad_raw_shard(rp.kind, rp.delta, E.Y.get(), shard, nshards);
    E.download(E.graw.get(), raw_grad);
  });
}

gmds_status gmds_classical_mds(const gmds_dmat* D, int32_t q, double* coords, double* eigvals, int32_t* clamped_count,
                               double* clamped_mass, double* stress) {
  return guard([&] {
    if (!D) fail(GMDS_INVALID_INPUT, "classical_mds: null distance matrix");
    not_sharded(D, "classical_mds");
    Stream st;
    int cc = 0;
    classical_mds_dev(D, q, coords, eigvals, &cc, clamped_mass, stress, st.s);
    *clamped_count = cc;
  });
}

gmds_status gmds_classical_mds_topq(const gmds_dmat* D, int32_t q, double tol, int32_t max_iters, double* coords,
                                    double* eigvals, int32_t* clamped_count, int32_t* iterations) {
  return guard([&] {
    if (!D) fail(GMDS_INVALID_INPUT, "classical_mds: null distance matrix");
    not_sharded(D, "classical_mds");
    Stream st;
    int cc = 0, its = 0;
    classical_topq_dev(D, q, tol, max_iters, coords, eigvals, &cc, &its, st.s);
    *clamped_count = cc;
    if (iterations) *iterations = its;
  });
}

// ---- row-sharded multi-GPU path ----

namespace {
// every rank's flag bits OR-ed (max of the value) so a failure is taken by the whole group
int group_flag(gmds::Comm& c, int local, cudaStream_t st) {
  DevBuf<double> v(1);
  const double h = static_cast<double>(local);
  GMDS_CUDA(cudaMemcpyAsync(v.get(), &h, sizeof h, cudaMemcpyHostToDevice, st));
  c.allreduce(v.get(), 1, RedOp::kMax, st);
  double out = 0.0;
  GMDS_CUDA(cudaMemcpyAsync(&out, v.get(), sizeof out, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return static_cast<int>(out);
}
}  // namespace

gmds_status gmds_dmat_gini_sharded(gmds_comm* comm, const void* dX, gmds_dtype xt, int64_t n, int64_t p, double nu,
                                   gmds_dtype storage, gmds_dmat** out) {
  return guard([&] {
    *out = nullptr;
    if (!comm) fail(GMDS_INVALID_INPUT, "pairwise_matrix (sharded): null comm");
    check_nu(nu);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    require_device();
    Stream st;
    Comm& c = *comm->impl;
    int64_t range[2];
    shard_blocks(n, c.rank, c.size, range[0], range[1]);
    if (group_flag(c, range[1] <= range[0] ? 1 : 0, st.s))
      fail(GMDS_INVALID_CONFIG, "pairwise_matrix (sharded): more ranks than work chunks");
    auto* d = new gmds_dmat();
    d->n = n;
    d->storage = storage;
    d->blk_lo = range[0];
    d->blk_hi = range[1];
    try {
      const size_t bytes = static_cast<size_t>(range[1] - range[0]) * kPT * kPT * dtype_size(storage);
      d->buf.alloc(bytes);
      GMDS_CUDA(cudaMemsetAsync(d->buf.get(), 0, bytes, st.s));
      DevBuf<int> flag(1);
      GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st.s));
      launch_finite_check(dX, xt, n * p, flag.get(), st.s);
      // only this rank's blocks: the tile rows covering them, filtered per tile in the kernels
      run_gini(dX, xt, n, p, &nu, 1, storage, 1, const_cast<void*>(d->ptr()), 0, 1, st.s, flag.get(), nullptr,
               nullptr, range);
      int hflag = 0;
      GMDS_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st.s));
      GMDS_CUDA(cudaStreamSynchronize(st.s));
      const int g = group_flag(c, hflag, st.s);
      if (g & 4) fail(GMDS_INVALID_INPUT, "gen_gini_directed: non-finite input");
      if (g & 1) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
      // per-fit constants over the whole matrix: sums, min and max all-reduced
      const DStats s = packed_stats(d->ptr(), storage, n, st.s, range[0], range[1]);
      DevBuf<double> v(4);
      const double hv[4] = {s.sum_sq, s.sum, s.min_off, s.max_off};
      GMDS_CUDA(cudaMemcpyAsync(v.get(), hv, sizeof hv, cudaMemcpyHostToDevice, st.s));
      c.allreduce(v.get(), 2, RedOp::kSum, st.s);
      c.allreduce(v.get() + 2, 1, RedOp::kMin, st.s);
      c.allreduce(v.get() + 3, 1, RedOp::kMax, st.s);
      double r[4];
      GMDS_CUDA(cudaMemcpyAsync(r, v.get(), sizeof r, cudaMemcpyDeviceToHost, st.s));
      GMDS_CUDA(cudaStreamSynchronize(st.s));
      d->sum_sq = r[0];
      d->sum = r[1];
      d->min_off = r[2];
      d->max_val = std::max(0.0, r[3]);
      d->stats = true;
    } catch (...) {
      delete d;
      throw;
    }
    *out = d;
  });
}

gmds_status gmds_minimize_stress_sharded(gmds_comm* comm, const gmds_dmat* D, int32_t q, const gmds_stress_cfg* cfg,
                                         const double* Y0, gmds_fit_result* res) {
  return guard([&] {
    if (!comm) fail(GMDS_INVALID_INPUT, "minimize_stress (sharded): null comm");
    if (!D) fail(GMDS_INVALID_INPUT, "minimize_stress: null distance matrix");
    if (!D->sharded()) fail(GMDS_INVALID_INPUT, "minimize_stress (sharded): D is not row-sharded");
    if (D->storage != GMDS_F32) fail(GMDS_INVALID_CONFIG, "minimize_stress (sharded): fp32 storage only");
    if (q < 1 || q > 4) fail(GMDS_INVALID_INPUT, "minimize_stress (sharded): 1 <= q <= 4");
    if (!Y0) fail(GMDS_INVALID_CONFIG, "minimize_stress (sharded): needs the seeded start Y0");
    if (cfg->max_iters < 1) fail(GMDS_INVALID_CONFIG, "minimize_stress: max_iters must be >= 1");
    if (!(cfg->rel_tol > 0.0)) fail(GMDS_INVALID_CONFIG, "minimize_stress: rel_tol must be > 0");
    if (cfg->smacof_weights) fail(GMDS_INVALID_CONFIG, "minimize_stress (sharded): uniform SMACOF weights only");
    if (cfg->kind == GMDS_HUBER && std::isnan(cfg->huber_delta))
      fail(GMDS_INVALID_CONFIG, "minimize_stress (sharded): huber needs an explicit huber_delta");
    check_coords(D, Y0, q, "minimize_stress");
    const Resolved rp = resolve(D, cfg->kind, cfg->huber_delta, nullptr, "minimize_stress");
    Stream st;
    Engine E(D, q, st.s, comm->impl.get());
    E.upload(Y0, E.Y.get());
    const IterResult r = (cfg->kind == GMDS_SMACOF) ? smacof_iterate(E, rp, nullptr, cfg->max_iters, cfg->rel_tol)
                                                    : gradient_descent(E, rp, cfg->max_iters, cfg->rel_tol);
    E.download(E.Y.get(), res->coords);
    res->history_len = static_cast<int64_t>(r.history.size());
    if (res->history)
      for (int64_t t = 0; t < std::min<int64_t>(res->history_len, res->history_cap); ++t)
        res->history[t] = r.history[static_cast<size_t>(t)];
    res->iterations = r.iterations;
    res->converged = r.converged ? 1 : 0;
    res->stress = r.loss;
    res->huber_delta = (cfg->kind == GMDS_HUBER) ? cfg->huber_delta : 0.0;
    res->passes = E.passes;
  });
}

gmds_status gmds_minimize_stress(const gmds_dmat* D, int32_t q, const gmds_stress_cfg* cfg, const double* Y0,
                                 gmds_fit_result* res) {
  return guard([&] {
    if (!D) fail(GMDS_INVALID_INPUT, "minimize_stress: null distance matrix");
    not_sharded(D, "minimize_stress");
    if (Y0) check_coords(D, Y0, q, "minimize_stress");
    Stream st;
    minimize_stress_dev(D, q, *cfg, Y0, res, st.s, nullptr);
  });
}

}  // extern "C"
