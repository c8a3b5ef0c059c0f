// Caching device allocator behind DevBuf (see common.cuh).
//
// Per device: a list of idle blocks, each with an event recorded on the
// releasing call's stream.  pool_alloc takes the smallest idle block that
// fits (at most 2x the request) whose event has completed, else cudaMalloc;
// on cudaErrorMemoryAllocation it returns every idle block to the driver and
// retries once.  Idle bytes are capped (kCacheCap), oldest blocks first.
#include <exception>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "lib_internal.h"

namespace gmds {

namespace {

constexpr size_t kCacheCap = size_t(8) << 30;  // idle bytes kept per device
constexpr int kMaxDev = 64;

struct Block {
  void* p;
  size_t bytes;
  cudaEvent_t ev;
};

struct DevicePool {
  std::mutex mu;
  std::vector<Block> idle;  // oldest first
  size_t idle_bytes = 0;
};

DevicePool g_pools[kMaxDev];

thread_local cudaStream_t t_stream = nullptr;
thread_local int t_depth = 0;

size_t round_bytes(size_t b) {
  if (b <= (size_t(1) << 20)) {
    size_t r = 512;
    while (r < b) r <<= 1;
    return r;
  }
  const size_t g = size_t(2) << 20;
  return (b + g - 1) / g * g;
}

int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) d = 0;
  return d;
}

void drop(Block& b) {
  if (b.ev) {
    cudaEventSynchronize(b.ev);
    cudaEventDestroy(b.ev);
  }
  cudaFree(b.p);
}

void trim_device(DevicePool& P) {
  std::vector<Block> v;
  {
    std::lock_guard<std::mutex> g(P.mu);
    v.swap(P.idle);
    P.idle_bytes = 0;
  }
  for (auto& b : v) drop(b);
}

}  // namespace

// Stream (lib_internal.h) marks the extent of a library call on this thread.
void call_stream_push(cudaStream_t s, cudaStream_t* prev) {
  *prev = t_stream;
  t_stream = s;
  ++t_depth;
}
void call_stream_pop(cudaStream_t prev) {
  t_stream = prev;
  --t_depth;
}

void* pool_alloc(size_t bytes, size_t* cap) {
  const size_t rb = round_bytes(bytes);
  DevicePool& P = g_pools[current_device()];
  {
    std::lock_guard<std::mutex> g(P.mu);
    int best = -1;
    for (int k = 0; k < static_cast<int>(P.idle.size()); ++k) {
      const Block& b = P.idle[k];
      if (b.bytes < rb || b.bytes > 2 * rb) continue;
      if (best >= 0 && P.idle[best].bytes <= b.bytes) continue;
      if (b.ev && cudaEventQuery(b.ev) != cudaSuccess) {
        cudaGetLastError();  // cudaErrorNotReady: still in use by its stream
        continue;
      }
      best = k;
    }
    if (best >= 0) {
      Block b = P.idle[best];
      P.idle.erase(P.idle.begin() + best);
      P.idle_bytes -= b.bytes;
      if (b.ev) cudaEventDestroy(b.ev);
      *cap = b.bytes;
      return b.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, rb);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    trim_device(P);
    e = cudaMalloc(&p, rb);
  }
  cuda_check(e, "cudaMalloc");
  *cap = rb;
  return p;
}

void pool_free(void* p, size_t cap) {
  if (!p) return;
  // no call stream to order the reuse against, or unwinding with work
  // possibly in flight on other streams: synchronous free
  if (t_depth == 0 || std::uncaught_exceptions() > 0) {
    cudaFree(p);
    return;
  }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(ev, t_stream) != cudaSuccess) {
    cudaGetLastError();
    if (ev) cudaEventDestroy(ev);
    cudaFree(p);
    return;
  }
  DevicePool& P = g_pools[current_device()];
  std::vector<Block> evict;
  {
    std::lock_guard<std::mutex> g(P.mu);
    P.idle.push_back(Block{p, cap, ev});
    P.idle_bytes += cap;
    while (P.idle_bytes > kCacheCap && !P.idle.empty()) {
      evict.push_back(P.idle.front());
      P.idle_bytes -= P.idle.front().bytes;
      P.idle.erase(P.idle.begin());
    }
  }
  for (auto& b : evict) drop(b);
}

void pool_trim() {
  for (auto& P : g_pools) trim_device(P);
}

}  // namespace gmds
