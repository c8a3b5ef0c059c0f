// tune_nu / alternating_tune (tune.cpp:85-167) over the device engine.
//
// The reference builds one n x n matrix per (nu, fold) cell.  Here every
// fold's distance matrices for ALL grid values come out of one launch (one
// sort per pair serves every nu), stay on the device in packed form, and
// are embedded and scored there; only scalars and the final embedding come
// back to the host.  Host control flow (folds, argmin with ties to the
// smaller nu, refit) follows the reference line by line.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "dmat.cuh"
#include "dmat_kernels.cuh"
#include "fit.h"
#include "kernels.cuh"
#include "lib_internal.h"

namespace gmds {

namespace {

// Rng::uniform_below + shuffle_indices (rng.cpp:29-37, 65-70) on std::mt19937_64.
uint64_t uniform_below(std::mt19937_64& g, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t limit = bound * ((~uint64_t{0}) / bound);
  for (;;) {
    const uint64_t x = g();
    if (x < limit) return x % bound;
  }
}

// make_folds (tune.cpp:39-56)
std::vector<std::vector<int>> make_folds(int n, int k, uint64_t seed) {
  std::vector<int> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), 0);
  std::mt19937_64 g(seed);
  for (size_t i = idx.size(); i > 1; --i) std::swap(idx[i - 1], idx[static_cast<size_t>(uniform_below(g, i))]);
  std::vector<std::vector<int>> folds(static_cast<size_t>(k));
  const int base = n / k, extra = n % k;
  int off = 0;
  for (int f = 0; f < k; ++f) {
    const int size = base + (f < extra ? 1 : 0);
    folds[f].assign(idx.begin() + off, idx.begin() + off + size);
    std::sort(folds[f].begin(), folds[f].end());
    off += size;
  }
  return folds;
}

// NuGrid::from_values (tune.cpp:74-83)
void check_grid(const double* g, int m) {
  if (m < 1) fail(GMDS_INVALID_CONFIG, "NuGrid: empty grid");
  for (int i = 0; i < m; ++i) {
    if (!(g[i] > 1.0)) fail(GMDS_INVALID_CONFIG, "NuGrid: every value must be > 1");
    if (i > 0 && !(g[i] > g[i - 1]))
      fail(GMDS_INVALID_CONFIG, "NuGrid: values must be strictly increasing (no duplicates)");
  }
}

// Distance matrices of X (device, row-major) for several nu from one launch.
std::vector<std::unique_ptr<gmds_dmat>> gini_multi(const void* dX, gmds_dtype xt, int64_t n, int64_t p,
                                                   const double* nus, int nnu, cudaStream_t st) {
  const int64_t per = packed_elems(n);
  auto buf = std::make_shared<DevBuf<unsigned char>>(static_cast<size_t>(per) * nnu * sizeof(double));
  GMDS_CUDA(cudaMemsetAsync(buf->get(), 0, static_cast<size_t>(per) * nnu * sizeof(double), st));
  DevBuf<int> flag(1);
  GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
  run_gini(dX, xt, n, p, nus, nnu, GMDS_F64, 1, buf->get(), 0, 1, st, flag.get());
  check_flag(flag.get(), st);
  std::vector<std::unique_ptr<gmds_dmat>> out;
  for (int v = 0; v < nnu; ++v) {
    auto d = std::make_unique<gmds_dmat>();
    d->n = n;
    d->storage = GMDS_F64;
    d->shared = buf;
    d->offset = static_cast<size_t>(per) * v * sizeof(double);
    dmat_finish(d.get(), st);
    out.push_back(std::move(d));
  }
  return out;
}

struct Emb {
  std::vector<double> coords, eigenvalues, history;
  double stress = 0.0, clamped_mass = 0.0, huber_delta = 0.0;
  int method = GMDS_M_CLASSICAL, clamped_count = 0, iterations = 0, converged = 1;

  void put(gmds_embedding* out) const {  // Embedding by value, into the caller's buffers
    std::memcpy(out->coords, coords.data(), coords.size() * sizeof(double));
    out->n_eigenvalues = static_cast<int32_t>(eigenvalues.size());
    if (out->eigenvalues)
      std::memcpy(out->eigenvalues, eigenvalues.data(), eigenvalues.size() * sizeof(double));
    out->history_len = static_cast<int64_t>(history.size());
    if (out->history)
      for (int64_t t = 0; t < std::min<int64_t>(out->history_len, out->history_cap); ++t)
        out->history[t] = history[static_cast<size_t>(t)];
    out->method = method;
    out->clamped_count = clamped_count;
    out->iterations = iterations;
    out->converged = converged;
    out->clamped_mass = clamped_mass;
    out->stress = stress;
    out->huber_delta = huber_delta;
  }
};

// embed_distances (tune.cpp:20-33): classical, or minimize_stress with a default StressConfig;
// every Embedding field as the reference fills it (embed.cpp:415-460, 491-532)
Emb embed(const gmds_dmat* D, int q, int method, uint64_t seed, cudaStream_t st) {
  Emb e;
  e.method = method;
  e.coords.assign(static_cast<size_t>(D->n) * q, 0.0);
  if (method == GMDS_M_CLASSICAL) {
    e.eigenvalues.assign(static_cast<size_t>(q), 0.0);
    classical_mds_dev(D, q, e.coords.data(), e.eigenvalues.data(), &e.clamped_count, &e.clamped_mass, &e.stress, st);
    return e;
  }
  gmds_stress_cfg cfg{};
  cfg.kind = method - 1;  // EmbeddingMethod -> StressKind
  cfg.huber_delta = std::nan("");
  cfg.smacof_weights = nullptr;
  cfg.max_iters = 300;
  cfg.rel_tol = 1e-6;
  cfg.seed = seed;
  e.history.assign(static_cast<size_t>(cfg.max_iters) + 2, 0.0);
  gmds_fit_result r{};
  r.coords = e.coords.data();
  r.history = e.history.data();
  r.history_cap = static_cast<int64_t>(e.history.size());
  minimize_stress_dev(D, q, cfg, nullptr, &r, st, nullptr);
  e.history.resize(static_cast<size_t>(std::min<int64_t>(r.history_len, r.history_cap)));
  e.stress = r.stress;
  e.iterations = r.iterations;
  e.converged = r.converged;
  e.huber_delta = r.huber_delta;
  return e;
}

double kruskal_of(const gmds_dmat* D, const double* coords, int q, cudaStream_t st) {
  // kruskal_stress (embed.cpp:462-475)
  if (D->sum_sq <= 0.0) fail(GMDS_DEGENERATE_INPUT, "kruskal_stress: all-zero distance matrix");
  EngineLease L = acquire_engine(D, q, st);
  Engine& E = *L;
  E.upload(coords, E.Y.get());
  const double* y = E.Y.get();
  return E.loss_of(kKruskal, E.loss_raw(kKruskal, 0.0, &y, 1)[0]);
}

std::vector<double> rows_of(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                            const std::vector<int>& rows) {
  // select_rows (tune.cpp:14-18) into a row-major fp64 block (fp32 widens exactly)
  std::vector<double> out(rows.size() * static_cast<size_t>(p));
  for (size_t r = 0; r < rows.size(); ++r)
    for (int64_t c = 0; c < p; ++c) {
      const int64_t idx = (lx == GMDS_ROW_MAJOR) ? rows[r] * p + c : c * n + rows[r];
      out[r * p + c] = (xt == GMDS_F32) ? static_cast<double>(static_cast<const float*>(X)[idx])
                                        : static_cast<const double*>(X)[idx];
    }
  return out;
}

// kruskal_stress(Y, D_nu) for every grid nu from ONE distance pass (SURVEY
// 8f-1): the distance kernels run in score mode and never store D_nu.  Falls
// back to materialised matrices when a pair needs the overflow path.
void sweep_kruskal(const void* dX, gmds_dtype xt, int64_t n, int64_t p, const double* grid, int m,
                   const double* coords_colmajor, int q, cudaStream_t st, double* ks) {
  std::vector<double> Yr(static_cast<size_t>(n) * q);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < q; ++k) Yr[i * q + k] = coords_colmajor[k * n + i];
  DevBuf<double> dY(Yr.size());
  GMDS_CUDA(cudaMemcpyAsync(dY.get(), Yr.data(), Yr.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  std::vector<double> num(static_cast<size_t>(m)), den(static_cast<size_t>(m));
  ScoreSpec sc;
  sc.dY = dY.get();
  sc.q = q;
  sc.num = num.data();
  sc.den = den.data();
  DevBuf<int> flag(1);
  GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
  run_gini(dX, xt, n, p, grid, m, GMDS_F64, 1, nullptr, 0, 1, st, flag.get(), &sc);
  if (sc.ok) {
    int hflag = 0;
    GMDS_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    if (hflag & 1) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
    for (int g = 0; g < m; ++g) {
      if (den[g] <= 0.0) fail(GMDS_DEGENERATE_INPUT, "kruskal_stress: all-zero distance matrix");
      ks[g] = std::sqrt(num[g] / den[g]);
    }
    return;
  }
  const auto Ds = gini_multi(dX, xt, n, p, grid, m, st);
  for (int g = 0; g < m; ++g) ks[g] = kruskal_of(Ds[g].get(), coords_colmajor, q, st);
}

DevBuf<double> upload_f64(const std::vector<double>& h, cudaStream_t st) {
  DevBuf<double> d(h.size());
  GMDS_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return d;
}

}  // namespace

}  // namespace gmds

using namespace gmds;

extern "C" {

gmds_status gmds_tune_nu_ex(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                            const double* grid, int32_t m, int32_t k_folds, int32_t method, uint64_t seed,
                            double* mean_stress, double* nu_star, gmds_embedding* best_emb) {
  return guard([&] {
    if (!best_emb || !best_emb->coords) fail(GMDS_INVALID_INPUT, "tune_nu: null embedding buffers");
    check_grid(grid, m);
    if (k_folds < 1) fail(GMDS_INVALID_CONFIG, "tune_nu: k_folds must be >= 1");
    if (n < k_folds) fail(GMDS_INVALID_CONFIG, "tune_nu: more folds than rows");
    const auto folds = make_folds(static_cast<int>(n), k_folds, seed);
    for (const auto& f : folds)
      if (static_cast<int>(f.size()) < q + 1)
        fail(GMDS_INVALID_CONFIG, "tune_nu: a fold has " + std::to_string(f.size()) +
                                      " points, need at least p + 1 = " + std::to_string(q + 1));
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    require_device();
    Stream st;
    std::vector<double> cell(static_cast<size_t>(m) * k_folds, 0.0);
    for (int f = 0; f < k_folds; ++f) {
      const std::vector<double> Xf = rows_of(X, xt, lx, n, p, folds[f]);
      const int64_t nf = static_cast<int64_t>(folds[f].size());
      if (nf < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
      DevBuf<double> dX = upload_f64(Xf, st.s);
      const auto Ds = gini_multi(dX.get(), GMDS_F64, nf, p, grid, m, st.s);
      std::vector<int> todo;
      for (int g = 0; g < m; ++g) {
        if (Ds[g]->max_val <= 0.0)  // all points coincide (tune.cpp:106-110)
          cell[static_cast<size_t>(g) * k_folds + f] = 0.0;
        else
          todo.push_back(g);
      }
      if (method == GMDS_M_CLASSICAL && !std::getenv("GMDS_NO_BATCHED_EIG")) {
        // the fold's grid cells are same-size classical MDS problems: batched
        // eigensolver, at most ~2 GB of Gram matrices per call
        const int64_t per = std::max<int64_t>(1, (int64_t(2) << 30) / std::max<int64_t>(1, nf * nf * 8));
        size_t i0 = 0;
        while (i0 < todo.size()) {
          const size_t i1 = std::min(todo.size(), i0 + static_cast<size_t>(per));
          std::vector<const gmds_dmat*> batch;
          for (size_t i = i0; i < i1; ++i) batch.push_back(Ds[todo[i]].get());
          std::vector<std::vector<double>> bc;
          std::vector<double> bst;
          if (!classical_mds_batch_dev(batch, q, bc, bst, st.s)) break;
          for (size_t i = i0; i < i1; ++i) cell[static_cast<size_t>(todo[i]) * k_folds + f] = bst[i - i0];
          i0 = i1;
        }
        todo.erase(todo.begin(), todo.begin() + static_cast<std::ptrdiff_t>(i0));
      }
      for (const int g : todo) {
        const gmds_dmat* D = Ds[g].get();
        const Emb e = embed(D, q, method, seed, st.s);
        cell[static_cast<size_t>(g) * k_folds + f] = kruskal_of(D, e.coords.data(), q, st.s);
      }
    }
    for (int g = 0; g < m; ++g) {
      double acc = 0.0;
      for (int f = 0; f < k_folds; ++f) acc += cell[static_cast<size_t>(g) * k_folds + f];
      mean_stress[g] = acc / static_cast<double>(k_folds);
    }
    int best = 0;
    for (int g = 1; g < m; ++g)
      if (mean_stress[g] < mean_stress[best]) best = g;  // ties keep the smaller nu
    *nu_star = grid[best];
    std::vector<int> all(static_cast<size_t>(n));
    std::iota(all.begin(), all.end(), 0);
    DevBuf<double> dX = upload_f64(rows_of(X, xt, lx, n, p, all), st.s);
    const auto Dfull = gini_multi(dX.get(), GMDS_F64, n, p, nu_star, 1, st.s);
    embed(Dfull[0].get(), q, method, seed, st.s).put(best_emb);
  });
}

gmds_status gmds_tune_nu(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                         const double* grid, int32_t m, int32_t k_folds, int32_t method, uint64_t seed,
                         double* mean_stress, double* nu_star, double* coords, double* stress) {
  gmds_embedding e{};
  e.coords = coords;
  const gmds_status s = gmds_tune_nu_ex(X, xt, lx, n, p, q, grid, m, k_folds, method, seed, mean_stress, nu_star, &e);
  if (s == GMDS_OK) *stress = e.stress;
  return s;
}

gmds_status gmds_nu_sweep_kruskal(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                                  const double* Y, int32_t q, const double* grid, int32_t m, double* ks) {
  return guard([&] {
    check_grid(grid, m);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    if (q < 1) fail(GMDS_INVALID_INPUT, "kruskal_stress: coords have no columns");
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    for (int64_t k = 0; k < n * q; ++k)
      if (!std::isfinite(Y[k])) fail(GMDS_INVALID_INPUT, "kruskal_stress: non-finite coordinates");
    require_device();
    Stream st;
    DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
    sweep_kruskal(dX.get(), xt, n, p, grid, m, Y, q, st.s, ks);
  });
}

gmds_status gmds_nu_sweep_kruskal_sharded(gmds_comm* comm, const void* X, gmds_dtype xt, gmds_layout lx, int64_t n,
                                          int64_t p, const double* Y, int32_t q, const double* grid, int32_t m,
                                          double* ks) {
  return guard([&] {
    if (!comm) fail(GMDS_INVALID_INPUT, "nu sweep (sharded): null comm");
    check_grid(grid, m);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    if (q < 1) fail(GMDS_INVALID_INPUT, "kruskal_stress: coords have no columns");
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    for (int64_t k = 0; k < n * q; ++k)
      if (!std::isfinite(Y[k])) fail(GMDS_INVALID_INPUT, "kruskal_stress: non-finite coordinates");
    require_device();
    Stream st;
    Comm& c = *comm->impl;
    // this rank's contiguous block of the grid (replicas: no exchange until the scores)
    int64_t g0 = 0, g1 = 0;
    share_of(m, c.rank, c.size, g0, g1);
    std::vector<double> mine(static_cast<size_t>(m), 0.0);
    int err = 0;
    std::string msg;
    gmds_status code = GMDS_OK;
    if (g1 > g0) {
      try {
        DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
        sweep_kruskal(dX.get(), xt, n, p, grid + g0, static_cast<int>(g1 - g0), Y, q, st.s, mine.data() + g0);
      } catch (const Failure& e) {  // every rank learns of it below, so no rank is left waiting
        err = 1;
        code = e.status;
        msg = e.what();
      }
    }
    DevBuf<double> v(static_cast<size_t>(m) + 1);
    mine.push_back(static_cast<double>(err));
    GMDS_CUDA(cudaMemcpyAsync(v.get(), mine.data(), mine.size() * sizeof(double), cudaMemcpyHostToDevice, st.s));
    c.allreduce(v.get(), mine.size(), RedOp::kSum, st.s);  // other ranks' slots are 0: a gather
    GMDS_CUDA(cudaMemcpyAsync(mine.data(), v.get(), mine.size() * sizeof(double), cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
    if (err) fail(code, msg);
    if (mine[static_cast<size_t>(m)] != 0.0) fail(GMDS_ERROR, "nu sweep (sharded): another rank failed");
    std::memcpy(ks, mine.data(), static_cast<size_t>(m) * sizeof(double));
  });
}

gmds_status gmds_alternating_tune_ex(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                                     int32_t outer_iters, const double* grid, int32_t m, uint64_t seed,
                                     double* nu_path, double* nu_star, gmds_embedding* out) {
  return guard([&] {
    if (!out || !out->coords) fail(GMDS_INVALID_INPUT, "alternating_tune: null embedding buffers");
    if (outer_iters < 1) fail(GMDS_INVALID_CONFIG, "alternating_tune: need at least one outer iteration");
    check_grid(grid, m);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    require_device();
    Stream st;
    std::vector<int> all(static_cast<size_t>(n));
    std::iota(all.begin(), all.end(), 0);
    DevBuf<double> dX = upload_f64(rows_of(X, xt, lx, n, p, all), st.s);
    double nu = 2.0;
    Emb emb;
    for (int t = 0; t < outer_iters; ++t) {
      const auto D = gini_multi(dX.get(), GMDS_F64, n, p, &nu, 1, st.s);
      emb = embed(D[0].get(), q, GMDS_M_SAMMON, seed, st.s);
      // grid sweep: every grid nu scored against the current embedding in one pass (no D_nu stored)
      int best = 0;
      std::vector<double> sweep(static_cast<size_t>(m));
      sweep_kruskal(dX.get(), GMDS_F64, n, p, grid, m, emb.coords.data(), q, st.s, sweep.data());
      for (int g = 1; g < m; ++g)
        if (sweep[g] < sweep[best]) best = g;
      nu = grid[best];
      nu_path[t] = nu;
    }
    *nu_star = nu;
    emb.put(out);
  });
}

gmds_status gmds_alternating_tune(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, int32_t q,
                                  int32_t outer_iters, const double* grid, int32_t m, uint64_t seed, double* nu_path,
                                  double* nu_star, double* coords, double* stress) {
  gmds_embedding e{};
  e.coords = coords;
  const gmds_status s =
      gmds_alternating_tune_ex(X, xt, lx, n, p, q, outer_iters, grid, m, seed, nu_path, nu_star, &e);
  if (s == GMDS_OK) *stress = e.stress;
  return s;
}

}  // extern "C"
