// pairwise_matrix, Euclidean branch (metrics.cpp:220-235) on the 5th-generation
// tensor cores: D_ij = sqrt(|x_i|^2 + |x_j|^2 - 2 x_i . x_j) with the
// Gram products from tcgen05.mma (TMA-fed shared-memory operands, fp32
// accumulators in TMEM) plus the rank-1 norm corrections in the epilogue.
//
// Precision.  The reference sums (x_ic - x_jc)^2 in fp64.  Here X is centred first
// (distances are translation invariant; centring removes the |x|^2 ~ x_i . x_j
// cancellation of uncentred data) and each centred value is split into three
// bf16 pieces h + m + l (24 significant bits, like fp32); the six products
// hh, hm, mh, hl, lh, mm are one bf16 GEMM over K = 6p of A = [h m l h h m] and
// B = [h h h m l m], exact products accumulated in fp32.  Norms are fp64.  A pair
// whose d^2 is below kRecompute of |x_i|^2 + |x_j|^2 (near-duplicates, where the
// subtraction cancels) is recomputed exactly in the reference's fp64 order
// (euclid_fix_kernel), so duplicated rows give exactly 0.
//
// Kernel anatomy (one 128 x 128 tile of the upper triangle per CTA, 128 threads):
//   warp 0 / lane 0   TMA producer: 128 x 64 bf16 boxes of A (rows I) and B (rows J),
//                     SWIZZLE_128B, into a kStages ring (full / empty mbarriers)
//   warp 1 / lane 0   MMA issuer: 4 x tcgen05.mma (M 128, N 128, K 16) per stage into
//                     a 128-column fp32 TMEM accumulator; tcgen05.commit frees the
//                     stage and finally signals the epilogue
//   warp 2            TMEM allocation / release
//   warps 0-3         epilogue: tcgen05.ld 32x32b.x32 (thread = row), d^2 in fp64,
//                     sqrt, both triangles written (the mirror coalesced)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "lib_internal.h"

namespace gmds {

namespace {

constexpr int kTileE = 128;     // rows per tile (UMMA M = N = 128)
constexpr int kBK = 64;         // K per stage: 64 bf16 = 128 B rows (one SW128 atom wide)
constexpr int kStagesE = 3;  // 96 KB of operands: two CTAs per SM, one's epilogue under the other's mainloop
constexpr int kStageBytes = 2 * kTileE * kBK * 2;  // A + B boxes
constexpr double kRecompute = 1.0 / 16.0;          // d^2 < this * (|x_i|^2 + |x_j|^2): exact fp64 pair

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}
// K-major, SWIZZLE_128B operand descriptor (8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t a = smem_addr(p);
  uint64_t d = 0;
  d |= (a >> 4) & 0x3FFFull;          // start address
  d |= 1ull << 16;                    // leading byte offset (unused for swizzled K-major)
  d |= (1024ull >> 4) << 32;          // stride byte offset: 8 rows x 128 B
  d |= 1ull << 46;                    // descriptor version (sm_100)
  d |= 2ull << 61;                    // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, both K-major, M = N = 128
constexpr uint32_t kIdesc = (1u << 4)                         // D fp32
                            | (1u << 7) | (1u << 10)          // A, B bf16
                            | ((kTileE >> 3) << 17)           // N
                            | ((kTileE >> 4) << 24);          // M

__device__ __forceinline__ void decode_upper(int64_t t, int64_t T, int64_t& I, int64_t& J) {
  const double b = 2.0 * static_cast<double>(T) + 1.0;
  int64_t i = static_cast<int64_t>((b - sqrt(b * b - 8.0 * static_cast<double>(t))) * 0.5);
  if (i < 0) i = 0;
  auto start = [T](int64_t r) { return r * T - (r * (r - 1)) / 2; };
  while (i > 0 && start(i) > t) --i;
  while (start(i + 1) <= t) ++i;
  I = i;
  J = i + (t - start(i));
}

__global__ void __launch_bounds__(128, 2)
    euclid_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int kblocks,
                     int64_t n, int64_t T, const double* __restrict__ nrm, double* __restrict__ D,
                     int2* __restrict__ fix, int* __restrict__ nfix, int fix_cap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStagesE], empty[kStagesE], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t I, J;
  decode_upper(blockIdx.x, T, I, J);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStagesE;
      if (kb >= kStagesE) mbar_wait(&empty[s], ((kb / kStagesE) - 1) & 1);
      unsigned char* a = smem + s * kStageBytes;
      unsigned char* b = a + kTileE * kBK * 2;
      mbar_expect(&full[s], kStageBytes);
      tma_load_2d(a, &mapA, kb * kBK, static_cast<int>(I * kTileE), &full[s]);
      tma_load_2d(b, &mapB, kb * kBK, static_cast<int>(J * kTileE), &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStagesE;
      mbar_wait(&full[s], (kb / kStagesE) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* a = smem + s * kStageBytes;
      const unsigned char* b = a + kTileE * kBK * 2;
      const uint64_t da = sw128_desc(a), db = sw128_desc(b);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {  // K = 16 bf16 = 32 B per instruction: +2 in 16-B units
        const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da + 2ull * k), "l"(db + 2ull * k), "r"(kIdesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_addr(&done))
                 : "memory");
  }
  __syncwarp();

  // epilogue: thread = row r of tile I (TMEM lane r), 4 x 32 columns
  mbar_wait(&done, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int r = warp * 32 + lane;
  const int64_t i = I * kTileE + r;
  const double ni = (i < n) ? nrm[i] : 0.0;
#pragma unroll 1
  for (int cb = 0; cb < kTileE / 32; ++cb) {
    uint32_t v[32];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cb * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // row i's 32 values: the mirror entries D(j, i) go straight out (consecutive i across the
    // warp: coalesced); D(i, j) is staged in the (now idle) operand ring and written row by
    // row, 32 consecutive doubles per warp store
    double* stage = reinterpret_cast<double*>(smem) + warp * (32 * 33);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int64_t j = J * kTileE + cb * 32 + c;
      double val = 0.0;
      if (i < n && j < n && j > i) {
        const double nj = nrm[j];
        const double g = static_cast<double>(__uint_as_float(v[c]));
        const double d2 = ni + nj - 2.0 * g;
        if (d2 < kRecompute * (ni + nj)) {  // cancellation: exact fp64 pass (euclid_fix_kernel)
          const int slot = atomicAdd(nfix, 1);
          if (slot < fix_cap) fix[slot] = make_int2(static_cast<int>(i), static_cast<int>(j));
        } else {
          val = sqrt(d2);
        }
        D[j * n + i] = val;
      }
      stage[lane * 33 + c] = val;
    }
    __syncwarp();
    const int64_t j = J * kTileE + cb * 32 + lane;
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t row = I * kTileE + warp * 32 + rr;
      if (row < n && j < n && j >= row) D[row * n + j] = stage[rr * 33 + lane];  // j == row: the zero diagonal
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

// centring (column means in fp64, fixed order), the three-piece bf16 split of every centred
// value into A = [h m l h h m] and B = [h h h m l m] (row-major, K = 6 pp, zero padded), and
// fp64 squared norms of the centred rows
template <typename T>
__global__ void colsum_part_kernel(const T* __restrict__ X, int64_t n, int p, int nparts, double* __restrict__ part) {
  // part[b][c] = sum of column c over row chunk b (thread: column c, rows strided by 8 within the chunk)
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  const int64_t r0 = n * blockIdx.y / nparts, r1 = n * (blockIdx.y + 1) / nparts;
  double s = 0.0;
  if (c < p)
    for (int64_t i = r0 + ty; i < r1; i += 8) s += static_cast<double>(X[i * p + c]);
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < p) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k][tx];
    part[static_cast<int64_t>(blockIdx.y) * p + c] = t;
  }
}

__global__ void colmean_finish_kernel(const double* __restrict__ part, int nparts, int64_t n, int p,
                                      double* __restrict__ mean) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[static_cast<int64_t>(b) * p + c];  // fixed order
    mean[c] = s / static_cast<double>(n);
  }
}

template <typename T>
__global__ void split_kernel(const T* __restrict__ X, int64_t n, int p, int pp, const double* __restrict__ mean,
                             __nv_bfloat16* __restrict__ A, __nv_bfloat16* __restrict__ B, double* __restrict__ nrm) {
  const int64_t K6 = 6 * static_cast<int64_t>(pp);
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    double s = 0.0;
    for (int c = threadIdx.x; c < pp; c += blockDim.x) {
      __nv_bfloat16 h = __float2bfloat16(0.f), m = h, l = h;
      if (c < p) {
        const double x = static_cast<double>(X[i * p + c]) - mean[c];
        s += x * x;
        h = __double2bfloat16(x);
        const double r1 = x - static_cast<double>(__bfloat162float(h));
        m = __double2bfloat16(r1);
        l = __double2bfloat16(r1 - static_cast<double>(__bfloat162float(m)));
      }
      __nv_bfloat16* a = A + i * K6;
      __nv_bfloat16* b = B + i * K6;
      a[c] = h, a[pp + c] = m, a[2 * pp + c] = l, a[3 * pp + c] = h, a[4 * pp + c] = h, a[5 * pp + c] = m;
      b[c] = h, b[pp + c] = h, b[2 * pp + c] = h, b[3 * pp + c] = m, b[4 * pp + c] = l, b[5 * pp + c] = m;
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) nrm[i] = red[0];
    __syncthreads();
  }
}

// the reference's own arithmetic for listed pairs: sq += (x_ic - x_jc)^2 in column order,
// sqrt (metrics.cpp:224-231), written to both triangles
template <typename T>
__global__ void euclid_fix_kernel(const T* __restrict__ X, int64_t n, int p, const int2* __restrict__ fix,
                                  const int* __restrict__ nfix, double* __restrict__ D) {
  const int cnt = *nfix;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
    const int64_t i = fix[k].x, j = fix[k].y;
    double sq = 0.0;
    for (int c = 0; c < p; ++c) {
      const double d = static_cast<double>(X[i * p + c]) - static_cast<double>(X[j * p + c]);
      sq = __dadd_rn(sq, __dmul_rn(d, d));
    }
    const double v = sqrt(sq);
    D[i * n + j] = v;
    D[j * n + i] = v;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) fail(GMDS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const void* base, int64_t rows, int64_t K) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  const cuuint32_t box[2] = {kBK, kTileE};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GMDS_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
  return m;
}

template <typename T>
void euclid_tc_t(const T* dX, int64_t n, int p, double* dD, cudaStream_t st) {
  const int pp = static_cast<int>(ceil_div(p, kBK) * kBK);
  const int64_t K6 = 6 * static_cast<int64_t>(pp);
  const int64_t T_ = ceil_div(n, kTileE), rows = T_ * kTileE;
  DevBuf<double> mean(static_cast<size_t>(p)), nrm(static_cast<size_t>(rows));
  DevBuf<__nv_bfloat16> A(static_cast<size_t>(rows * K6)), B(static_cast<size_t>(rows * K6));
  GMDS_CUDA(cudaMemsetAsync(A.get(), 0, A.n * sizeof(__nv_bfloat16), st));
  GMDS_CUDA(cudaMemsetAsync(B.get(), 0, B.n * sizeof(__nv_bfloat16), st));
  const int nparts = 64;
  DevBuf<double> part(static_cast<size_t>(nparts) * p);
  colsum_part_kernel<T><<<dim3(static_cast<unsigned>(ceil_div(p, 32)), nparts), 256, 0, st>>>(dX, n, p, nparts,
                                                                                             part.get());
  colmean_finish_kernel<<<static_cast<unsigned>(ceil_div(p, 128)), 128, 0, st>>>(part.get(), nparts, n, p, mean.get());
  split_kernel<T><<<static_cast<unsigned>(std::min<int64_t>(n, 148 * 16)), 256, 0, st>>>(dX, n, p, pp, mean.get(),
                                                                                         A.get(), B.get(), nrm.get());
  count_launch(3);
  check_launch("euclid split");
  const CUtensorMap ma = make_map(A.get(), rows, K6), mb = make_map(B.get(), rows, K6);
  const int cap = 1 << 22;
  DevBuf<int2> fix(static_cast<size_t>(cap));
  DevBuf<int> nfix(1);
  GMDS_CUDA(cudaMemsetAsync(nfix.get(), 0, sizeof(int), st));
  const size_t smem = static_cast<size_t>(kStagesE) * kStageBytes + 1024;
  GMDS_CUDA(cudaFuncSetAttribute(euclid_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t tiles = T_ * (T_ + 1) / 2;
  euclid_tc_kernel<<<static_cast<unsigned>(tiles), 128, smem, st>>>(ma, mb, static_cast<int>(K6 / kBK), n, T_, nrm.get(),
                                                                  dD, fix.get(), nfix.get(), cap);
  count_launch();
  check_launch("euclid_tc_kernel");
  int hf = 0;
  GMDS_CUDA(cudaMemcpyAsync(&hf, nfix.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  if (hf > cap) {  // too many near-duplicates for the list: the exact kernel does the whole matrix
    launch_euclid(dX, sizeof(T) == 4 ? GMDS_F32 : GMDS_F64, n, p, dD, st);
    return;
  }
  if (hf > 0) {
    euclid_fix_kernel<T><<<static_cast<unsigned>(std::min<int64_t>(ceil_div(hf, 128), 148 * 8)), 128, 0, st>>>(
        dX, n, p, fix.get(), nfix.get(), dD);
    count_launch();
    check_launch("euclid_fix_kernel");
  }
  GMDS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

bool euclid_tc_enabled(int64_t n, int64_t p) {
  const char* e = std::getenv("GMDS_EUCLID");
  if (e && std::string(e) == "exact") return false;
  if (e && std::string(e) == "tc") return n < (int64_t(1) << 31) / kTileE;
  return n >= 512 && n < (int64_t(1) << 24) && p >= 1;
}

void launch_euclid_tc(const void* dX, gmds_dtype xt, int64_t n, int p, double* dD, cudaStream_t st) {
  if (xt == GMDS_F32)
    euclid_tc_t(static_cast<const float*>(dX), n, p, dD, st);
  else
    euclid_tc_t(static_cast<const double*>(dX), n, p, dD, st);
}

}  // namespace gmds
