// Host orchestration of the Gini distance kernels (run_gini): row-store
// preparation (bitmask-sparse rows when X is sparse), kernel and tile-size
// selection, and the overflow pass.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "gini_gmd.cuh"
#include "gini_merge.cuh"
#include "kernels.cuh"
#include "lib_internal.h"

namespace gmds {

template <int KMAX>
void launch_gini_split(const SplitArgs& sa, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, size_t smem,
                       unsigned blocks, cudaStream_t st);
template <int K>
void launch_gini_list(GiniTileArgs a, const void* dX, gmds_dtype xt, const int64_t* pairs, int64_t npairs, void* dout,
                      gmds_dtype ot, cudaStream_t st);

void launch_row_sort(const void* vals, gmds_dtype xt, const uint16_t* fidx, const int64_t* rowptr, const int* rows,
                     int nrows, int K, uint16_t* sidx, void* svs, uint16_t* pmap, double* suf, double* s1,
                     double* tm, uint32_t* tiew, cudaStream_t st);

namespace {

// GMDS_TRACE=1: host-side phase timings of run_gini on stderr (observability)
struct Trace {
  bool on = std::getenv("GMDS_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gmds] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// warp per row: presence masks, running popcounts, per-row nonzero counts
template <typename T>
__global__ void row_mask_kernel(const T* __restrict__ X, int64_t n, int p, int W, uint32_t* __restrict__ masks,
                                uint16_t* __restrict__ prefix, int* __restrict__ counts, int* __restrict__ negflag) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n;
       row += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    int run = 0;
    for (int w = 0; w < W; ++w) {
      const int e = w * 32 + lane;
      const T xv = (e < p) ? X[row * p + e] : T(0);
      const bool nz = xv != T(0);
      if (xv < T(0)) atomicOr(negflag, 1);
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      if (lane == 0) {
        masks[row * W + w] = m;
        prefix[row * W + w] = static_cast<uint16_t>(run);
      }
      run += __popc(m);
    }
    if (lane == 0) counts[row] = run;
  }
}

template <typename T>
__global__ void row_fill_kernel(const T* __restrict__ X, int64_t n, int p, int W, const uint32_t* __restrict__ masks,
                                const uint16_t* __restrict__ prefix, const int64_t* __restrict__ rowptr,
                                T* __restrict__ vals, uint16_t* __restrict__ fidx) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n;
       row += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    for (int w = 0; w < W; ++w) {
      const int e = w * 32 + lane;
      const unsigned m = masks[row * W + w];
      if ((m >> lane) & 1u) {
        const int64_t o = rowptr[row] + prefix[row * W + w] + __popc(m & lt);
        vals[o] = X[row * p + e];
        fidx[o] = static_cast<uint16_t>(e);
      }
    }
  }
}

struct RowStore {
  DevBuf<uint16_t> fidx, sidx;
  DevBuf<unsigned char> svs;  // values in ascending order per row (merge path)
  DevBuf<uint16_t> pmap;      // sorted position of each nonzero (feature order; linear-weight path)
  DevBuf<double> suf;         // suffix sums of the sorted values (linear-weight path)
  DevBuf<double> s1, tm;      // per row: sum of values, sum_k v_(k) k
  DevBuf<uint32_t> tiew;      // per row, 8 words: bit g = (v_(g) == v_(g+1)) (rows of <= 256 nonzeros)
  bool nonneg = false;
  DevBuf<uint32_t> masks;
  DevBuf<uint16_t> prefix;
  DevBuf<int64_t> rowptr;
  DevBuf<unsigned char> vals;
  int W = 0;
  int maxnnz = 0;
  double density = 1.0;
};

RowStore build_rows(const void* dX, gmds_dtype xt, int64_t n, int p, cudaStream_t st, bool fill_if_sparse) {
  RowStore rs;
  rs.W = (p + 31) / 32;
  rs.masks.alloc(static_cast<size_t>(n) * rs.W);
  rs.prefix.alloc(static_cast<size_t>(n) * rs.W);
  DevBuf<int> counts(static_cast<size_t>(n));
  DevBuf<int> negflag(1);
  GMDS_CUDA(cudaMemsetAsync(negflag.get(), 0, sizeof(int), st));
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), 148 * 16)));
  if (xt == GMDS_F32)
    row_mask_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dX), n, p, rs.W, rs.masks.get(),
                                                   rs.prefix.get(), counts.get(), negflag.get());
  else
    row_mask_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dX), n, p, rs.W, rs.masks.get(),
                                                    rs.prefix.get(), counts.get(), negflag.get());
  count_launch();
  check_launch("row_mask_kernel");
  std::vector<int> hc(static_cast<size_t>(n));
  int hneg = 0;
  GMDS_CUDA(cudaMemcpyAsync(hc.data(), counts.get(), n * sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaMemcpyAsync(&hneg, negflag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  rs.nonneg = (hneg == 0);
  std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    rp[i + 1] = rp[i] + hc[i];
    rs.maxnnz = std::max(rs.maxnnz, hc[i]);
  }
  rs.density = static_cast<double>(rp[n]) / (static_cast<double>(n) * p);
  if (!fill_if_sparse || rs.density >= 0.5) return rs;
  rs.rowptr.alloc(rp.size());
  GMDS_CUDA(cudaMemcpyAsync(rs.rowptr.get(), rp.data(), rp.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  rs.vals.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])) * dtype_size(xt));
  rs.fidx.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])));
  if (xt == GMDS_F32)
    row_fill_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dX), n, p, rs.W, rs.masks.get(),
                                                   rs.prefix.get(), rs.rowptr.get(), reinterpret_cast<float*>(rs.vals.get()), rs.fidx.get());
  else
    row_fill_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dX), n, p, rs.W, rs.masks.get(),
                                                    rs.prefix.get(), rs.rowptr.get(),
                                                    reinterpret_cast<double*>(rs.vals.get()), rs.fidx.get());
  count_launch();
  check_launch("row_fill_kernel");
  if (rs.nonneg) {
    // value-sorted feature order per row (the merge kernel's runs); rows bucketed by sort width
    rs.sidx.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])));
    rs.svs.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])) * dtype_size(xt));
    rs.pmap.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])));
    rs.suf.alloc(static_cast<size_t>(std::max<int64_t>(1, rp[n])));
    rs.s1.alloc(static_cast<size_t>(n));
    rs.tm.alloc(static_cast<size_t>(n));
    rs.tiew.alloc(static_cast<size_t>(n) * 8);
    GMDS_CUDA(cudaMemsetAsync(rs.tiew.get(), 0, static_cast<size_t>(n) * 8 * sizeof(uint32_t), st));
    std::vector<std::vector<int>> buckets(6);
    for (int64_t i = 0; i < n; ++i) {
      int K = 1;
      while (32 * K < hc[i]) K <<= 1;
      int bk = 0;
      while ((1 << bk) < K) ++bk;
      buckets[bk].push_back(static_cast<int>(i));
    }
    for (int bk = 0; bk < 6; ++bk) {
      if (buckets[bk].empty()) continue;
      DevBuf<int> rows(buckets[bk].size());
      GMDS_CUDA(cudaMemcpyAsync(rows.get(), buckets[bk].data(), buckets[bk].size() * sizeof(int),
                                cudaMemcpyHostToDevice, st));
      launch_row_sort(rs.vals.get(), xt, rs.fidx.get(), rs.rowptr.get(), rows.get(),
                      static_cast<int>(buckets[bk].size()), 1 << bk, rs.sidx.get(), rs.svs.get(), rs.pmap.get(),
                      rs.suf.get(), rs.s1.get(), rs.tm.get(), rs.tiew.get(), st);
      GMDS_CUDA(cudaStreamSynchronize(st));
    }
  }
  return rs;
}

size_t split_smem(int tile, int p, int W, int maxnnz, size_t sz, int nnu, bool sparse) {
  size_t s = static_cast<size_t>(8) * kSplitCap * 8 + static_cast<size_t>(nnu) * tile * (tile + 1) * 8;
  if (sparse)
    s += ((2 * static_cast<size_t>(tile) * W * 6 + 15) & ~static_cast<size_t>(15)) +
         2 * static_cast<size_t>(tile) * maxnnz * sz;
  else
    s += 2 * static_cast<size_t>(tile) * p * sz;
  return s;
}

}  // namespace

// CTAs per SM of the split kernel instance p selects (K = 8 for p <= 256)
inline int split_detail_min_blocks(int64_t p) { return split_min_blocks(p <= 256 ? 8 : 16); }

void run_gini(const void* dX, gmds_dtype xt, int64_t n, int64_t p, const double* nus, int nnu, gmds_dtype ot,
              int packed, void* dD, int shard, int nshards, cudaStream_t st, int* dflag, ScoreSpec* score,
              RowSink* sink, const int64_t* blk_range) {
  Trace tr;
  if (blk_range && (!packed || score || nshards != 1)) fail(GMDS_ERROR, "run_gini: block ranges are for packed stores");
  // this launch's tiles: shard `shard` of the tile list, or (row-sharded packed builds) the tile
  // rows covering packed block strips [strip(lo), strip(hi - 1)], filtered per tile in the kernels
  auto set_range = [&](GiniTileArgs& g, int64_t units, int64_t decode_nbt) {
    if (!blk_range) {
      g.tile_begin = units * shard / nshards;
      g.tile_end = units * (shard + 1) / nshards;
      return;
    }
    g.blk_lo = blk_range[0];
    g.blk_hi = blk_range[1];
    const int64_t nb = g.nb_packed;
    auto bstart = [nb](int64_t r) { return r * nb - (r * (r - 1)) / 2; };
    int64_t sI = 0, eI = 0;
    while (bstart(sI + 1) <= g.blk_lo) ++sI;
    eI = sI;
    while (bstart(eI + 1) <= g.blk_hi - 1) ++eI;
    const int64_t r = kPT / g.tile;  // tile rows per block strip
    auto tstart = [decode_nbt](int64_t R) {
      R = std::min(R, decode_nbt);
      return R * decode_nbt - (R * (R - 1)) / 2;
    };
    g.tile_begin = tstart(sI * r);
    g.tile_end = tstart((eI + 1) * r);
  };
  if (packed || score || nshards != 1) sink = nullptr;
  // Launch tiles [a.tile_begin, a.tile_end) -- in block-row chunks when a sink
  // wants the finished rows as they complete.
  auto chunked = [&](GiniTileArgs& ga, auto&& launch) {
    if (!sink) {
      launch(ga);
      return;
    }
    // Chunks of about equal work, each covering at most nbt/24 block rows: the
    // rows left to copy after the last launch (the tail the caller waits for)
    // stay a few percent of the matrix even though late block rows hold few tiles.
    const int64_t nbt = ga.nbt, b0 = ga.tile_begin, b1 = ga.tile_end;
    auto start = [nbt](int64_t r) { return r * nbt - (r * (r - 1)) / 2; };
    const int64_t max_rows = std::max<int64_t>(1, nbt / 24);
    int64_t R = 0;
    for (int c = 1; R < nbt; ++c) {
      const int64_t target = b0 + (b1 - b0) * std::min(c, sink->chunks) / sink->chunks;
      int64_t R1 = R;
      while (R1 < nbt && R1 - R < max_rows && (R1 == R || start(R1 + 1) <= target)) ++R1;
      ga.tile_begin = start(R);
      ga.tile_end = start(R1);
      launch(ga);
      sink->rows_done(std::min<int64_t>(n, R1 * ga.tile), st);
      R = R1;
    }
    ga.tile_begin = b0;
    ga.tile_end = b1;
  };
  if (score && (p > 1024 || nnu > kMaxScoreNu)) {  // block path / too many nu: caller falls back
    score->ok = false;
    return;
  }
  // score mode: persistent grid (per-CTA partials), no D written
  DevBuf<double> spart;
  const int64_t score_grid = 148 * 2;
  auto grid_of = [&](int64_t units_) -> int64_t { return score ? std::min<int64_t>(units_, score_grid) : units_; };
  auto finish_score = [&](int64_t grid) {
    if (!score) return;
    int hflag = 0;
    GMDS_CUDA(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    std::vector<double> h(static_cast<size_t>(grid) * 2 * nnu);
    GMDS_CUDA(cudaMemcpyAsync(h.data(), spart.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    score->ok = (hflag & 2) == 0;
    for (int v = 0; v < nnu; ++v) {
      double sn = 0.0, sd = 0.0;
      for (int64_t b = 0; b < grid; ++b) {  // fixed order: deterministic
        sn += h[(b * nnu + v) * 2];
        sd += h[(b * nnu + v) * 2 + 1];
      }
      score->num[v] = sn;
      score->den[v] = sd;
    }
  };
  const std::vector<double> lut = build_lut(static_cast<int>(p), nus, nnu);
  DevBuf<double> dlut(lut.size());
  GMDS_CUDA(cudaMemcpyAsync(dlut.get(), lut.data(), lut.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  tr.mark("lut", st);
  GiniTileArgs a{};
  a.n = n;
  a.d = static_cast<int>(p);
  a.lut = dlut.get();
  a.nnu = nnu;
  a.packed = packed;
  a.nb_packed = ceil_div(n, kPT);
  a.out_stride = packed ? packed_elems(n) : n * n;
  a.flag = dflag;
  if (!packed && !score && shard == 0) {
    // full layout: the tiles write i != j only; the diagonal is D(i, i) = 0
    // (pairwise_matrix starts from Matrix::Zero, metrics.cpp:210)
    const size_t es = dtype_size(ot);
    for (int v = 0; v < nnu; ++v)
      GMDS_CUDA(cudaMemset2DAsync(static_cast<unsigned char*>(dD) + static_cast<size_t>(v) * a.out_stride * es,
                                  static_cast<size_t>(n + 1) * es, 0, es, static_cast<size_t>(n), st));
  }
  if (score) {
    spart.alloc(static_cast<size_t>(score_grid) * 2 * nnu);
    GMDS_CUDA(cudaMemsetAsync(spart.get(), 0, spart.n * sizeof(double), st));
    a.Y = score->dY;
    a.q = score->q;
    a.score_part = spart.get();
  }
  if (p > 1024) {  // CTA-per-pair block sort
    a.tile = 1;
    a.nbt = n;
    const int64_t units = n * (n - 1) / 2;
    set_range(a, units, n - 1);
    launch_gini(a, dX, xt, dD, ot, st);
    GMDS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const size_t sz = dtype_size(xt);
  RowStore rs = build_rows(dX, xt, n, static_cast<int>(p), st, true);
  tr.mark("row store", st);
  const bool sparse = rs.density < 0.5;
  auto full_kernel = [&]() {  // the all-keys warp kernel (dense data with large p)
    a.tile = gini_tile_size(static_cast<int>(p), xt, nnu);
    a.nbt = ceil_div(n, a.tile);
    const int64_t units = a.nbt * (a.nbt + 1) / 2;
    set_range(a, units, a.nbt);
    chunked(a, [&](GiniTileArgs& ga) { launch_gini(ga, dX, xt, dD, ot, st, score ? score_grid : 0); });
    finish_score(score ? std::min<int64_t>(a.tile_end - a.tile_begin, score_grid) : 0);
  };
  if (!sparse && p > 512) {
    full_kernel();
    GMDS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // split kernel: split_min_blocks(K) CTAs per SM (its __launch_bounds__) share ~226 KB of smem
  const size_t two_per_sm = (split_detail_min_blocks(p) >= 3 ? 74 : 113) * 1024, one_per_sm = 220 * 1024;
  bool linear = (score == nullptr) && !std::getenv("GMDS_NO_LINEAR");
  for (int v = 0; v < nnu; ++v)
    if (nus[v] != 2.0 && nus[v] != 3.0) linear = false;
  // warps per CTA of the linear-weight kernel: the most that fit in shared memory
  // and the panel stride (nonzeros per staged row): rows with more nonzeros than the
  // stride go to the overflow list, so a few dense rows do not push every pair
  // off this kernel
  int gmd_warps = 0;
  int gmd_stride = std::min(std::max(1, rs.maxnnz), gmd_detail::kMaxC);
  const size_t gmd_budget = 227 * 1024 - 4096;  // dynamic shared memory; the general kernel has 3 KB static
  for (int nw : {28, 24})  // 28: 72 registers, no spills (217 ms vs 221 at 24; 32 spills: 230 ms)
    if (!gmd_warps && gmd_smem(rs.W, gmd_stride, nnu, nw) <= gmd_budget) gmd_warps = nw;
  if (!gmd_warps) {
    gmd_warps = 24;
    while (gmd_stride > 32 && gmd_smem(rs.W, gmd_stride, nnu, gmd_warps) > gmd_budget) gmd_stride -= 8;
    if (gmd_smem(rs.W, gmd_stride, nnu, gmd_warps) > gmd_budget) gmd_warps = 0;
  }
  if (const char* e = std::getenv("GMDS_GMD_WARPS")) gmd_warps = std::atoi(e);
  // nu in {2, 3}: gini_gmd2_kernel (batched F lists, bucket search; rows of <= 255 nonzeros staged);
  // GMDS_GMD_V1=1: the round-1 kernel
  const bool gmd2 = linear && !std::getenv("GMDS_GMD_V1");
  int gmd2_warps = 0, gmd2_stride = std::min(std::max(1, rs.maxnnz), gmd2_detail::kMaxC2);
  if (gmd2) {
    for (int nw : {28, 24})
      if (!gmd2_warps && gmd2_smem(rs.W, gmd2_stride, nnu, nw) <= gmd_budget) gmd2_warps = nw;
    if (!gmd2_warps) {
      gmd2_warps = 24;
      while (gmd2_stride > 32 && gmd2_smem(rs.W, gmd2_stride, nnu, gmd2_warps) > gmd_budget) gmd2_stride -= 8;
      if (gmd2_smem(rs.W, gmd2_stride, nnu, gmd2_warps) > gmd_budget) gmd2_warps = 0;
    }
    if (const char* e = std::getenv("GMDS_GMD_WARPS")) gmd2_warps = std::atoi(e);
  }
  bool use2 = gmd2 && gmd2_warps > 0;
  // other nu (at most 4 per launch, store mode): the general counting kernel on the same panels
  const bool general = !linear && score == nullptr && nnu <= 4 && !std::getenv("GMDS_NO_GEN");
  // ... as gini_gen2_kernel (the same three changes; GMDS_GEN_V1=1: the round-1 kernel)
  if (general && !std::getenv("GMDS_GEN_V1")) {
    for (int nw : {28, 24})
      if (!gmd2_warps && gen2_smem(rs.W, gmd2_stride, nnu, nw) <= gmd_budget) gmd2_warps = nw;
    if (!gmd2_warps) {
      gmd2_warps = 24;
      while (gmd2_stride > 32 && gen2_smem(rs.W, gmd2_stride, nnu, gmd2_warps) > gmd_budget) gmd2_stride -= 8;
      if (gen2_smem(rs.W, gmd2_stride, nnu, gmd2_warps) > gmd_budget) gmd2_warps = 0;
    }
    if (const char* e = std::getenv("GMDS_GMD_WARPS")) gmd2_warps = std::atoi(e);
    use2 = gmd2_warps > 0;
  }
  if ((linear || general) && sparse && rs.nonneg && p > 32 && xt == GMDS_F32 && gmd_warps > 0) {
    // nu in {2, 3}: D from per-row prefix sums and the shared features (gini_gmd.cuh);
    // other nu: midranks counted from the same structures, one LUT pass (gini_gen_kernel)
    const size_t gsm = !use2 ? gmd_smem(rs.W, gmd_stride, nnu, gmd_warps)
                             : (linear ? gmd2_smem(rs.W, gmd2_stride, nnu, gmd2_warps)
                                       : gen2_smem(rs.W, gmd2_stride, nnu, gmd2_warps));
    a.tile = gmd_detail::kTile;
    a.nbt = ceil_div(n, a.tile);
    const int64_t units = a.nbt * (a.nbt + 1) / 2;
    set_range(a, units, a.nbt);
    if (a.tile_end <= a.tile_begin) return;
    GmdArgs ga{};
    ga.s.g = a;
    ga.s.masks = rs.masks.get();
    ga.s.prefix = rs.prefix.get();
    ga.s.rowptr = rs.rowptr.get();
    ga.s.vals = rs.vals.get();
    ga.s.W = rs.W;
    ga.s.maxnnz = use2 ? gmd2_stride : gmd_stride;  // panel stride; longer rows overflow
    ga.s.sparse = 1;
    ga.pmap = rs.pmap.get();
    ga.svs = reinterpret_cast<const float*>(rs.svs.get());
    ga.suf = rs.suf.get();
    ga.s1 = rs.s1.get();
    ga.tm = rs.tm.get();
    ga.tiew = rs.tiew.get();
    DevBuf<uint8_t> bkt;
    DevBuf<float> bscale;
    if (use2) {  // per-row bucket tables of the sorted values
      bkt.alloc(static_cast<size_t>(n) * 256);
      bscale.alloc(static_cast<size_t>(n));
      launch_row_buckets(ga.svs, rs.rowptr.get(), n, bkt.get(), bscale.get(), st);
      count_launch();
      check_launch("row_bucket_kernel");
      ga.bkt = bkt.get();
      ga.bscale = bscale.get();
    }
    const int64_t shard_pairs = (a.tile_end - a.tile_begin) * static_cast<int64_t>(a.tile) * a.tile;
    ga.s.ovf_cap = std::min<int64_t>(shard_pairs, int64_t(1) << 20);
    DevBuf<int64_t> ovf(static_cast<size_t>(2 * ga.s.ovf_cap));
    DevBuf<unsigned long long> ovf_count(1);
    GMDS_CUDA(cudaMemsetAsync(ovf_count.get(), 0, sizeof(unsigned long long), st));
    ga.s.ovf_pairs = ovf.get();
    ga.s.ovf_count = ovf_count.get();
    chunked(a, [&](GiniTileArgs& g) {
      ga.s.g = g;
      const unsigned blk = static_cast<unsigned>(std::min<int64_t>(g.tile_end - g.tile_begin, int64_t(1) << 30));
      if (use2 && linear)
        launch_gini_gmd2(ga, dD, ot, gsm, blk, gmd2_warps, st);
      else if (use2)
        launch_gini_gen2(ga, dD, ot, gsm, blk, gmd2_warps, st);
      else if (linear)
        launch_gini_gmd(ga, dD, ot, gsm, blk, gmd_warps, st);
      else
        launch_gini_gen(ga, dD, ot, gsm, blk, gmd_warps, st);
      count_launch();
      check_launch(linear ? "gini_gmd_kernel" : "gini_gen_kernel");
    });
    ga.s.g = a;
    tr.mark(linear ? "gini_gmd_kernel" : "gini_gen_kernel", st);
    unsigned long long novf = 0;
    GMDS_CUDA(cudaMemcpyAsync(&novf, ovf_count.get(), sizeof novf, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    if (tr.on) std::fprintf(stderr, "[gmds] gmd overflow pairs: %llu\n", novf);
    if (novf == 0) return;
    if (sink) sink->late_writes = true;
    if (static_cast<int64_t>(novf) > ga.s.ovf_cap) {
      sink = nullptr;
      full_kernel();
    } else {
      launch_gini_list<32>(a, dX, xt, ovf.get(), static_cast<int64_t>(novf), dD, ot, st);
      count_launch();
      check_launch("gini_list_kernel");
    }
    GMDS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (sparse && rs.nonneg && p > 32 && xt == GMDS_F32) {  // merge path (exact u32 keys need fp32 inputs): pre-sorted row runs + one bitonic merge per sign half
    int mt = 32;
    while (mt > 4 && merge_smem(mt, rs.W, std::max(1, rs.maxnnz), sz, nnu) > one_per_sm) mt >>= 1;
    const size_t msm = merge_smem(mt, rs.W, std::max(1, rs.maxnnz), sz, nnu);
    if (msm <= one_per_sm) {
      a.tile = mt;
      a.nbt = ceil_div(n, mt);
      const int64_t munits = a.nbt * (a.nbt + 1) / 2;
      set_range(a, munits, a.nbt);
      if (a.tile_end <= a.tile_begin) return;
      MergeArgs ma{};
      ma.s.g = a;
      ma.s.masks = rs.masks.get();
      ma.s.prefix = rs.prefix.get();
      ma.s.rowptr = rs.rowptr.get();
      ma.s.vals = rs.vals.get();
      ma.s.W = rs.W;
      ma.s.maxnnz = std::max(1, rs.maxnnz);
      ma.s.sparse = 1;
      ma.sidx = rs.sidx.get();
      ma.svs = rs.svs.get();
      // rank-by-counting first: exact, but measured slower than the merge path on the
      // metric data (0.83 vs 0.72 s), so opt-in (GMDS_MERGE_FAST=1)
      ma.fast = std::getenv("GMDS_MERGE_FAST") ? 1 : 0;
      DevBuf<unsigned long long> miss;
      if (tr.on) {
        miss.alloc(1);
        GMDS_CUDA(cudaMemsetAsync(miss.get(), 0, sizeof(unsigned long long), st));
        ma.fast_miss = miss.get();
      }
      const int64_t shard_pairs = (a.tile_end - a.tile_begin) * static_cast<int64_t>(mt) * mt;
      ma.s.ovf_cap = (p > 512) ? std::min<int64_t>(shard_pairs, int64_t(1) << 20) : 0;
      DevBuf<int64_t> ovf(static_cast<size_t>(std::max<int64_t>(1, 2 * ma.s.ovf_cap)));
      DevBuf<unsigned long long> ovf_count(1);
      GMDS_CUDA(cudaMemsetAsync(ovf_count.get(), 0, sizeof(unsigned long long), st));
      tr.mark("overflow buffers", st);
      ma.s.ovf_pairs = ovf.get();
      ma.s.ovf_count = ovf_count.get();
      const unsigned mblocks =
          static_cast<unsigned>(grid_of(std::min<int64_t>(a.tile_end - a.tile_begin, int64_t(1) << 30)));
      ma.s.g = a;
      chunked(a, [&](GiniTileArgs& ga) {
        ma.s.g = ga;
        const unsigned blk = static_cast<unsigned>(grid_of(std::min<int64_t>(ga.tile_end - ga.tile_begin, int64_t(1) << 30)));
        launch_gini_merge(ma, dX, xt, dD, ot, msm, blk, st);
        count_launch();
        check_launch("gini_merge_kernel");
      });
      ma.s.g = a;
      tr.mark("gini_merge_kernel", st);
      if (tr.on) {
        unsigned long long hm = 0;
        GMDS_CUDA(cudaMemcpyAsync(&hm, miss.get(), sizeof hm, cudaMemcpyDeviceToHost, st));
        GMDS_CUDA(cudaStreamSynchronize(st));
        std::fprintf(stderr, "[gmds] merge fast path: %llu of %lld pairs fell back\n", hm,
                     static_cast<long long>(n * (n - 1) / 2));
      }
      unsigned long long novf = 0;
      GMDS_CUDA(cudaMemcpyAsync(&novf, ovf_count.get(), sizeof novf, cudaMemcpyDeviceToHost, st));
      GMDS_CUDA(cudaStreamSynchronize(st));
      finish_score(mblocks);
      if (novf == 0 || score) return;
      if (sink) sink->late_writes = true;
      if (static_cast<int64_t>(novf) > ma.s.ovf_cap) {
        RowSink* keep = sink;
        sink = nullptr;  // rewrites already-copied rows
        full_kernel();
        sink = keep;
      } else {
        launch_gini_list<32>(a, dX, xt, ovf.get(), static_cast<int64_t>(novf), dD, ot, st);
        count_launch();
        check_launch("gini_list_kernel");
      }
      GMDS_CUDA(cudaStreamSynchronize(st));
      return;
    }
  }
  int tile = 32;
  while (tile > 4 && split_smem(tile, static_cast<int>(p), rs.W, rs.maxnnz, sz, nnu, sparse) > two_per_sm) tile >>= 1;
  if (split_smem(tile, static_cast<int>(p), rs.W, rs.maxnnz, sz, nnu, sparse) > two_per_sm) {
    tile = 32;
    while (tile > 1 && split_smem(tile, static_cast<int>(p), rs.W, rs.maxnnz, sz, nnu, sparse) > one_per_sm) tile >>= 1;
  }
  const size_t smem = split_smem(tile, static_cast<int>(p), rs.W, rs.maxnnz, sz, nnu, sparse);
  if (smem > one_per_sm) {
    full_kernel();
    GMDS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  a.tile = tile;
  a.nbt = ceil_div(n, tile);
  const int64_t units = a.nbt * (a.nbt + 1) / 2;
  set_range(a, units, a.nbt);
  if (a.tile_end <= a.tile_begin) return;
  SplitArgs sa{};
  sa.g = a;
  sa.masks = rs.masks.get();
  sa.prefix = rs.prefix.get();
  sa.rowptr = rs.rowptr.get();
  sa.vals = rs.vals.get();
  sa.W = rs.W;
  sa.maxnnz = std::max(1, rs.maxnnz);
  sa.sparse = sparse ? 1 : 0;
  const int64_t shard_pairs = (a.tile_end - a.tile_begin) * static_cast<int64_t>(tile) * tile;
  sa.ovf_cap = (p > 512) ? std::min<int64_t>(shard_pairs, int64_t(1) << 20) : 0;
  DevBuf<int64_t> ovf(static_cast<size_t>(std::max<int64_t>(1, 2 * sa.ovf_cap)));
  DevBuf<unsigned long long> ovf_count(1);
  GMDS_CUDA(cudaMemsetAsync(ovf_count.get(), 0, sizeof(unsigned long long), st));
  sa.ovf_pairs = ovf.get();
  sa.ovf_count = ovf_count.get();
  const unsigned blocks = static_cast<unsigned>(grid_of(std::min<int64_t>(a.tile_end - a.tile_begin, 1 << 30)));
  sa.g = a;
  (void)blocks;
  chunked(a, [&](GiniTileArgs& ga) {
    sa.g = ga;
    const unsigned blk = static_cast<unsigned>(grid_of(std::min<int64_t>(ga.tile_end - ga.tile_begin, 1 << 30)));
    if (p <= 256)
      launch_gini_split<8>(sa, dX, xt, dD, ot, smem, blk, st);
    else
      launch_gini_split<16>(sa, dX, xt, dD, ot, smem, blk, st);
    count_launch();
    check_launch("gini_split_kernel");
  });
  sa.g = a;
  unsigned long long novf = 0;
  GMDS_CUDA(cudaMemcpyAsync(&novf, ovf_count.get(), sizeof novf, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  finish_score(blocks);
  if (novf == 0 || score) return;
  if (sink) sink->late_writes = true;
  if (static_cast<int64_t>(novf) > sa.ovf_cap) {  // list too long: redo these tiles with the all-keys kernel
    sink = nullptr;
    full_kernel();
    GMDS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // p > 512 here, so the full sort needs 1024 keys (K = 32)
  launch_gini_list<32>(a, dX, xt, ovf.get(), static_cast<int64_t>(novf), dD, ot, st);
  count_launch();
  check_launch("gini_list_kernel");
  GMDS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gmds
