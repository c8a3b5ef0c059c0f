// Shared host/device helpers for libgmds (status mapping, CUDA checks).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <stdexcept>
#include <utility>
#include <string>

#include "gmds.h"

namespace gmds {

// Host-side error carrying a gmds_status; thrown inside the library and
// converted to a status + thread-local message at the C-ABI boundary.
struct Failure : std::runtime_error {
  gmds_status status;
  Failure(gmds_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(gmds_status s, const std::string& msg) { throw Failure(s, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(GMDS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define GMDS_CUDA(call) ::gmds::cuda_check((call), #call)

inline void check_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

void set_last_error(const std::string& msg);

template <typename F>
gmds_status guard(F&& f) {
  try {
    f();
    return GMDS_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return GMDS_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GMDS_ERROR;
  }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (stress loop): a kernel launched with
// launch_pdl may be scheduled while its predecessor in the stream drains; it
// must call pdl_wait() before touching memory (griddepcontrol.wait returns once
// the predecessor grid has completed and its writes are visible).
// GMDS_NO_PDL=1 launches them with ordinary stream order.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// lets the next PDL launch in the stream be scheduled now (its pdl_wait still
// waits for this grid to complete)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = std::getenv("GMDS_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

inline size_t dtype_size(gmds_dtype t) { return t == GMDS_F32 ? 4 : 8; }

// Device memory: a caching pool (pool.cu).  Buffers released while a library
// call is running (a Stream is live on this thread) go back to a per-device
// free list with an event recorded on the call's stream; a later allocation
// reuses a block only once that event has completed.  cudaMalloc/cudaFree on
// every call cost 2-300 ms of host-side stalls at the metric shape (the e2e
// output alone is 3.2 GB).  Buffers released outside a call, or while an
// exception unwinds, are returned with cudaFree.
void* pool_alloc(size_t bytes, size_t* cap);
void pool_free(void* p, size_t cap);
void pool_trim();  // return every idle cached block to the driver

// RAII device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;  // bytes held from the pool
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) {
    o.p = nullptr;
    o.n = 0;
    o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      cap = o.cap;
      o.p = nullptr;
      o.n = 0;
      o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) p = static_cast<T*>(pool_alloc(count * sizeof(T), &cap));
    n = count;
  }
  void release() {
    if (p) pool_free(p, cap);
    p = nullptr;
    n = 0;
    cap = 0;
  }
  T* get() const { return p; }
};

}  // namespace gmds
