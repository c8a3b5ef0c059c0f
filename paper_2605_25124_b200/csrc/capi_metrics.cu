// C-ABI: rank and distance entry points (metrics.hpp / metrics.cpp).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "lib_internal.h"

namespace gmds {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(GMDS_CUDA_ERROR, "libgmds: no CUDA device visible (the engine has no CPU fallback)");
  }
}

void check_nu(double nu) {
  // GiniParams (metrics.hpp:35-36)
  if (!(nu > 1.0)) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "GiniParams: nu must be > 1, got %f", nu);
    fail(GMDS_INVALID_CONFIG, buf);
  }
}

void check_finite_host(const void* X, gmds_dtype xt, int64_t count, const char* who) {
  bool ok = true;
  if (xt == GMDS_F32) {
    const float* p = static_cast<const float*>(X);
    for (int64_t k = 0; k < count && ok; ++k) ok = std::isfinite(p[k]);
  } else {
    const double* p = static_cast<const double*>(X);
    for (int64_t k = 0; k < count && ok; ++k) ok = std::isfinite(p[k]);
  }
  if (!ok) fail(GMDS_INVALID_INPUT, std::string(who) + ": non-finite input entry");
}

// pow-table of gen_gini_directed_impl (metrics.cpp:73-79), folded for both
// directions: L[h] = (pow(S(p+1-R), e) - c) - (pow(S(R), e) - c), h = 2R - 1.
std::vector<double> build_lut(int d, const double* nus, int nnu) {
  std::vector<double> lut(static_cast<size_t>(nnu) * 2 * d, 0.0);
  const double inv_d = 1.0 / static_cast<double>(d);
  for (int v = 0; v < nnu; ++v) {
    const double exponent = nus[v] - 1.0;
    const double c = std::pow(0.5, exponent);
    for (int h = 1; h < 2 * d; ++h) {
      const double rank = 0.5 * static_cast<double>(h + 1);
      const double s_fwd = 1.0 - (rank - 0.5) * inv_d;
      const double rank_bwd = static_cast<double>(d) + 1.0 - rank;
      const double s_bwd = 1.0 - (rank_bwd - 0.5) * inv_d;
      const double t_fwd = std::pow(s_fwd, exponent) - c;
      const double t_bwd = std::pow(s_bwd, exponent) - c;
      lut[static_cast<size_t>(v) * 2 * d + h] = t_bwd - t_fwd;
    }
  }
  return lut;
}

// Host X (row- or column-major) -> device row-major copy.
// fp64 input whose every value is exactly an fp32 value (data stored as double by the caller,
// e.g. an Eigen::MatrixXd of image intensities): the same values as fp32, so the kernels that
// need exact 32-bit keys (the linear-weight, general-nu and merge paths) serve it.  The
// distances are functions of the values only, so nothing but the dispatch changes.
const void* narrow_exact_f32(const void* X, gmds_dtype& xt, int64_t m, std::vector<float>& buf) {
  if (xt != GMDS_F64) return X;
  const double* x = static_cast<const double*>(X);
  buf.resize(static_cast<size_t>(m));
  for (int64_t k = 0; k < m; ++k) {
    const float f = static_cast<float>(x[k]);
    if (static_cast<double>(f) != x[k] || (x[k] == 0.0 && std::signbit(x[k]))) return X;  // keep fp64
    buf[static_cast<size_t>(k)] = f;
  }
  xt = GMDS_F32;
  return buf.data();
}

DevBuf<unsigned char> upload_rows(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                                  cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(n) * p * dtype_size(xt);
  DevBuf<unsigned char> out(bytes);
  if (lx == GMDS_ROW_MAJOR || p == 1 || n == 1) {
    GMDS_CUDA(cudaMemcpyAsync(out.get(), X, bytes, cudaMemcpyHostToDevice, st));
  } else {
    DevBuf<unsigned char> tmp(bytes);
    GMDS_CUDA(cudaMemcpyAsync(tmp.get(), X, bytes, cudaMemcpyHostToDevice, st));
    launch_transpose(tmp.get(), xt, n, p, out.get(), st);
    GMDS_CUDA(cudaStreamSynchronize(st));
  }
  return out;
}

namespace {
template <typename T>
__global__ void finite_check_kernel(const T* __restrict__ X, int64_t m, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(X[k]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 4);
}
}  // namespace

void launch_finite_check(const void* dX, gmds_dtype xt, int64_t m, int* dflag, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 148 * 8)));
  if (xt == GMDS_F32)
    finite_check_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dX), m, dflag);
  else
    finite_check_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dX), m, dflag);
  count_launch();
  check_launch("finite_check_kernel");
}

void check_flag(int* dflag, cudaStream_t st) {
  int flag = 0;
  GMDS_CUDA(cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  if (flag & 1) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
}

namespace {
thread_local cudaStream_t g_user_stream = nullptr;
thread_local bool g_user_stream_set = false;
}  // namespace

// Calls use the caller's stream when one was set with gmds_set_stream (bench
// timing with CUDA events on that stream); otherwise a private stream.
Stream::Stream() {
  if (g_user_stream_set) {
    s = g_user_stream;
    owned = false;
  } else {
    GMDS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  call_stream_push(s, &prev);
}
Stream::~Stream() {
  call_stream_pop(prev);
  if (s && owned) cudaStreamDestroy(s);
}

// ALU roofline probe: independent FFMA (fma pipe) and IADD3/LOP3 (alu pipe)
// chains, interleaved so both pipes issue every cycle.  Counts lane-ops.
__global__ void alu_probe_kernel(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  unsigned b0 = threadIdx.x, b1 = b0 * 3u, b2 = b0 * 5u, b3 = b0 * 7u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, 0.999f, 1e-4f);
      b0 = (b0 + 0x9e3779b9u) ^ b1;
      a1 = fmaf(a1, 0.999f, 1e-4f);
      b1 = (b1 + 0x7f4a7c15u) ^ b2;
      a2 = fmaf(a2, 0.999f, 1e-4f);
      b2 = (b2 + 0x94d049bbu) ^ b3;
      a3 = fmaf(a3, 0.999f, 1e-4f);
      b3 = (b3 + 0xbf58476du) ^ b0;
    }
  }
  if (a0 + a1 + a2 + a3 == 1234.5f && (b0 ^ b1 ^ b2 ^ b3) == 77u) out[0] = 1.f;
}

}  // namespace gmds

using namespace gmds;

extern "C" {

const char* gmds_last_error(void) { return g_last_error.c_str(); }
const char* gmds_version(void) { return "gmds-b200 0.1.0 (sm_100a); reference ginimds 0.1.0"; }

int gmds_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

gmds_status gmds_set_device(int device) {
  return guard([&] { GMDS_CUDA(cudaSetDevice(device)); });
}

int64_t gmds_launch_count(void) { return launch_count(); }

gmds_status gmds_set_stream(void* stream) {
  g_user_stream = static_cast<cudaStream_t>(stream);
  g_user_stream_set = (stream != nullptr);
  return GMDS_OK;
}

gmds_status gmds_probe_alu(double* lane_ops_per_sec) {
  return guard([&] {
    require_device();
    int dev = 0, sms = 0;
    GMDS_CUDA(cudaGetDevice(&dev));
    GMDS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DevBuf<float> out(1);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    GMDS_CUDA(cudaEventCreate(&e0));
    GMDS_CUDA(cudaEventCreate(&e1));
    alu_probe_kernel<<<blocks, threads>>>(out.get(), 64);  // warm-up
    GMDS_CUDA(cudaEventRecord(e0));
    alu_probe_kernel<<<blocks, threads>>>(out.get(), iters);
    GMDS_CUDA(cudaEventRecord(e1));
    GMDS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    GMDS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // per inner unroll: 4 FFMA + 4 x (IADD3 + LOP3) = 12 lane-ops
    const double ops = static_cast<double>(blocks) * threads * iters * 16.0 * 12.0;
    *lane_ops_per_sec = ops / (ms * 1e-3);
  });
}

int64_t gmds_packed_elems(int64_t n) { return packed_elems(n); }

gmds_status gmds_midrank_batch(const double* v, int64_t m, int64_t d, double* ranks) {
  return guard([&] {
    if (d < 1) fail(GMDS_INVALID_INPUT, "midrank: input vector is empty");
    check_finite_host(v, GMDS_F64, m * d, "midrank");
    if (m == 0) return;
    require_device();
    Stream st;
    DevBuf<double> dv(static_cast<size_t>(m * d)), dr(static_cast<size_t>(m * d));
    GMDS_CUDA(cudaMemcpyAsync(dv.get(), v, sizeof(double) * m * d, cudaMemcpyHostToDevice, st.s));
    launch_midrank(dv.get(), nullptr, GMDS_F64, nullptr, m, static_cast<int>(d), dr.get(), st.s);
    GMDS_CUDA(cudaMemcpyAsync(ranks, dr.get(), sizeof(double) * m * d, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
  });
}

gmds_status gmds_pair_midranks(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                               const int64_t* pairs, int64_t npairs, double* ranks) {
  return guard([&] {
    if (p < 1) fail(GMDS_INVALID_INPUT, "gen_gini_directed: input vector is empty");
    check_finite_host(X, xt, n * p, "gen_gini_directed");
    for (int64_t k = 0; k < 2 * npairs; ++k)
      if (pairs[k] < 0 || pairs[k] >= n) fail(GMDS_INVALID_INPUT, "pair_midranks: row index out of range");
    if (npairs == 0) return;
    require_device();
    Stream st;
    DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
    DevBuf<int64_t> dp(static_cast<size_t>(2 * npairs));
    DevBuf<double> dr(static_cast<size_t>(npairs * p));
    GMDS_CUDA(cudaMemcpyAsync(dp.get(), pairs, sizeof(int64_t) * 2 * npairs, cudaMemcpyHostToDevice, st.s));
    launch_midrank(nullptr, dX.get(), xt, dp.get(), npairs, static_cast<int>(p), dr.get(), st.s);
    GMDS_CUDA(cudaMemcpyAsync(ranks, dr.get(), sizeof(double) * npairs * p, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
  });
}

gmds_status gmds_gen_gini_distance(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out) {
  return guard([&] {
    check_nu(nu);
    if (dx != dy)
      fail(GMDS_INVALID_INPUT,
           "gen_gini_directed: length mismatch (" + std::to_string(dx) + " vs " + std::to_string(dy) + ")");
    if (dx < 1) fail(GMDS_INVALID_INPUT, "gen_gini_directed: input vector is empty");
    check_finite_host(x, GMDS_F64, dx, "gen_gini_directed");
    check_finite_host(y, GMDS_F64, dy, "gen_gini_directed");
    require_device();
    Stream st;
    std::vector<double> X2(static_cast<size_t>(2 * dx));
    std::memcpy(X2.data(), x, sizeof(double) * dx);
    std::memcpy(X2.data() + dx, y, sizeof(double) * dx);
    DevBuf<double> dX(X2.size()), dD(4);
    DevBuf<int> flag(1);
    GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st.s));
    GMDS_CUDA(cudaMemsetAsync(dD.get(), 0, 4 * sizeof(double), st.s));
    GMDS_CUDA(cudaMemcpyAsync(dX.get(), X2.data(), sizeof(double) * X2.size(), cudaMemcpyHostToDevice, st.s));
    run_gini(dX.get(), GMDS_F64, 2, dx, &nu, 1, GMDS_F64, 0, dD.get(), 0, 1, st.s, flag.get());
    double D[4];
    GMDS_CUDA(cudaMemcpyAsync(D, dD.get(), sizeof D, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
    *out = D[1];  // +inf propagates as in the reference's scalar API (no matrix validation here)
  });
}

gmds_status gmds_pairwise_gini(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                               const double* nus, int32_t nnu, gmds_dtype out_t, void* D) {
  return guard([&] {
    if (nnu < 1) fail(GMDS_INVALID_CONFIG, "pairwise_matrix: no nu value given");
    for (int v = 0; v < nnu; ++v) check_nu(nus[v]);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    require_device();
    Stream st;
    std::vector<float> narrowed;
    X = narrow_exact_f32(X, xt, n * p, narrowed);
    DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
    DevBuf<int> flag(1);
    GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st.s));
    // gen_gini_directed_checked (metrics.cpp:84-93): every input entry finite
    // -- checked on the device (bit 2 of the flag), reported before any result
    launch_finite_check(dX.get(), xt, n * p, flag.get(), st.s);
    const size_t plane = static_cast<size_t>(n) * n * dtype_size(out_t);
    const size_t bytes = static_cast<size_t>(nnu) * plane;
    DevBuf<unsigned char> dD(bytes);
    GMDS_CUDA(cudaMemsetAsync(dD.get(), 0, bytes, st.s));
    // A pinned destination is filled row stripe by row stripe while later
    // tiles are still computing (copy stream + one event per stripe).
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, D) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    struct CopySink : RowSink {
      cudaStream_t cs = nullptr;
      std::vector<cudaEvent_t> evs;
      unsigned char* host;
      const unsigned char* dev;
      size_t plane, row_bytes;
      int nnu;
      int64_t prev = 0;
      void rows_done(int64_t rows, cudaStream_t st) override {
        cudaEvent_t ev;
        GMDS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        evs.push_back(ev);
        GMDS_CUDA(cudaEventRecord(ev, st));
        GMDS_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        for (int v = 0; v < nnu; ++v)
          GMDS_CUDA(cudaMemcpyAsync(host + v * plane + prev * row_bytes, dev + v * plane + prev * row_bytes,
                                    (rows - prev) * row_bytes, cudaMemcpyDeviceToHost, cs));
        prev = rows;
      }
      ~CopySink() override {
        if (cs) {
          cudaStreamSynchronize(cs);
          cudaStreamDestroy(cs);
        }
        for (auto e : evs) cudaEventDestroy(e);
      }
    } sink;
    sink.host = static_cast<unsigned char*>(D);
    sink.dev = dD.get();
    sink.plane = plane;
    sink.row_bytes = static_cast<size_t>(n) * dtype_size(out_t);
    sink.nnu = nnu;
    if (pinned) GMDS_CUDA(cudaStreamCreateWithFlags(&sink.cs, cudaStreamNonBlocking));
    run_gini(dX.get(), xt, n, p, nus, nnu, out_t, 0, dD.get(), 0, 1, st.s, flag.get(), nullptr,
             pinned ? &sink : nullptr);
    int hflag = 0;
    GMDS_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
    if (hflag & 4) fail(GMDS_INVALID_INPUT, "gen_gini_directed: non-finite input entry");
    if (hflag & 1) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
    if (pinned && sink.prev == n && !sink.late_writes) {
      GMDS_CUDA(cudaStreamSynchronize(sink.cs));
    } else {
      if (pinned) GMDS_CUDA(cudaStreamSynchronize(sink.cs));
      GMDS_CUDA(cudaMemcpyAsync(D, dD.get(), bytes, cudaMemcpyDeviceToHost, st.s));
      GMDS_CUDA(cudaStreamSynchronize(st.s));
    }
  });
}

gmds_status gmds_pairwise_euclidean_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, double* dD,
                                           int32_t mode, void* stream) {
  return guard([&] {
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    if (mode < 0 || mode > 2) fail(GMDS_INVALID_CONFIG, "pairwise_euclidean: mode must be 0 (auto), 1 (exact), 2 (tc)");
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CallScope scope(st);
    const bool tc = mode == 2 || (mode == 0 && euclid_tc_enabled(n, p));
    if (tc) {
      launch_euclid_tc(dX, xt, n, static_cast<int>(p), dD, st);
    } else {
      GMDS_CUDA(cudaMemsetAsync(dD, 0, sizeof(double) * n * n, st));
      launch_euclid(dX, xt, n, static_cast<int>(p), dD, st);
    }
    GMDS_CUDA(cudaStreamSynchronize(st));
  });
}

gmds_status gmds_pairwise_euclidean(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p, double* D) {
  return guard([&] {
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    require_device();
    Stream st;
    DevBuf<unsigned char> dX = upload_rows(X, xt, lx, n, p, st.s);
    DevBuf<double> dD(static_cast<size_t>(n * n));
    GMDS_CUDA(cudaMemsetAsync(dD.get(), 0, sizeof(double) * n * n, st.s));
    if (euclid_tc_enabled(n, p))
      launch_euclid_tc(dX.get(), xt, n, static_cast<int>(p), dD.get(), st.s);
    else
      launch_euclid(dX.get(), xt, n, static_cast<int>(p), dD.get(), st.s);
    GMDS_CUDA(cudaMemcpyAsync(D, dD.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
    // from_matrix (metrics.cpp:169-191): Euclidean entries are finite for finite
    // X unless a square overflows; reject like the reference.
    for (int64_t k = 0; k < n * n; ++k)
      if (!std::isfinite(D[k])) fail(GMDS_INVALID_INPUT, "DistanceMatrix: non-finite entry");
  });
}

gmds_status gmds_pairwise_gini_device(const void* dX, gmds_dtype xt, int64_t n, int64_t p, const double* nus,
                                      int32_t nnu, gmds_dtype out_t, int32_t packed, void* dD, int32_t shard,
                                      int32_t nshards, void* stream) {
  return guard([&] {
    if (nnu < 1) fail(GMDS_INVALID_CONFIG, "pairwise_matrix: no nu value given");
    for (int v = 0; v < nnu; ++v) check_nu(nus[v]);
    if (n < 2) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 2 rows");
    if (p < 1) fail(GMDS_INVALID_INPUT, "pairwise_matrix: need at least 1 column");
    if (nshards < 1 || shard < 0 || shard >= nshards) fail(GMDS_INVALID_CONFIG, "pairwise_matrix: bad shard");
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CallScope scope(st);
    DevBuf<int> flag(1);
    GMDS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    run_gini(dX, xt, n, p, nus, nnu, out_t, packed, dD, shard, nshards, st, flag.get());
    check_flag(flag.get(), st);
  });
}

}  // extern "C"
