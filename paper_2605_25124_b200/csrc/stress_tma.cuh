// K3 (fp32 storage): the stress pass with D streamed by TMA bulk copies.
//
// Same contract as stress_pass_kernel (stress_pass.cuh): one pass over the
// packed upper triangle, loss partials at up to kMaxCand configurations, and
// (GRAD) per-row sums of c_ij (y_i - y_j), reduced in a fixed order.
//
// Data movement: every 128x128 block of the packed fp32 image is two
// contiguous 32 KB half-blocks (rows 0-63, 64-127).  One elected thread
// streams them with cp.async.bulk (1-D TMA) into a 2-stage shared-memory
// ring guarded by mbarriers (two CTAs per SM: up to 128 KB in flight) while the
// 256 threads consume the previous stage from shared memory.
//
// Arithmetic diet per pair (kruskal, q = 2): y_j held in registers, 2 FADD,
// FMUL+FFMA, FMNMX, MUFU.RSQ, FMUL, FADD, FFMA (loss), FMUL, 4 FFMA
// (row/column sums).  d2 is clamped to FLT_MIN before rsqrtf so coincident
// points (d2 = 0, hence dy = 0) add exactly 0 without a select; interior
// blocks skip all validity masks.
#pragma once

#include <float.h>

#include <type_traits>

#include "f32x2.cuh"
#include "stress_pass.cuh"

#ifndef GMDS_CSPLIT_DG
#define GMDS_CSPLIT_DG 0
#endif
#ifndef GMDS_CSPLIT_Q2
#define GMDS_CSPLIT_Q2 0
#endif
#ifndef GMDS_TMA_MINB_FUSED
#define GMDS_TMA_MINB_FUSED 2
#endif
#ifndef GMDS_TMA_MINB
// CTAs per SM: 3 for loss passes, 2 for gradient passes (128 registers).  At
// Q >= 3 the gradient passes spill (448 B at Q = 3) yet stay faster than one
// CTA per SM without spills (n = 20000: 24.2 vs 28.5 ms per 50 iterations)
#define GMDS_TMA_MINB(MODE, Q) ((MODE) == 0 ? 3 : ((MODE) == 2 ? GMDS_TMA_MINB_FUSED : 2))
#endif

namespace gmds {

namespace tma_detail {

#ifndef GMDS_TMA_PARTS
#define GMDS_TMA_PARTS 2  // 4 bands of 16 KB measured 13.1 vs 12.9 ms per 50 iterations (more barriers)
#endif
constexpr int kParts = GMDS_TMA_PARTS;  // TMA units per 128x128 block (row bands of kPT / kParts rows)
#ifndef GMDS_TMA_STAGES
#define GMDS_TMA_STAGES GMDS_TMA_PARTS
#endif
constexpr int kStages = GMDS_TMA_STAGES;  // loss passes: one block's bytes in flight (3 CTAs/SM: 192 KB per SM)
constexpr int kStagesGrad = GMDS_TMA_STAGES;  // gradient passes: 64 KB per CTA (3 x 32 KB left one CTA per SM: 288 vs 207 us)
constexpr int kHalfRows = kPT / kParts;        // rows per TMA unit ("half" below: one band)
constexpr int kHalfFloats = kHalfRows * kPT;  // 4096 floats = 16 KB at 4 parts
constexpr int kMR = kHalfRows / kTG;          // micro-tile rows per band (ti*kMR + x)
constexpr int kTmaCand = 2;                   // trial points per loss pass (y_j kept in registers)
// Thread column tj owns columns 4tj..4tj+3 and 64+4tj..64+4tj+3 of a block: each
// 16-byte shared-memory read of a D row by 8 consecutive threads covers 128
// contiguous bytes (no bank conflicts; 8 contiguous columns per thread gave 2-way).
__device__ __forceinline__ int tcol(int tj, int y) { return (y < 4) ? 4 * tj + y : 64 + 4 * tj + (y - 4); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int KIND>
__device__ __forceinline__ void kind_terms(float Dv, float invD, float dist, float inv, float w, float delta,
                                           float& term, float& c) {
  const float e = Dv - dist;
  if constexpr (KIND == kKruskal) {
    term = e * e;
    c = -e * inv;
  } else if constexpr (KIND == kHuber) {
    const float ae = fabsf(e);
    term = (ae <= delta) ? 0.5f * e * e : delta * (ae - 0.5f * delta);
    c = -fminf(fmaxf(e, -delta), delta) * inv;
  } else if constexpr (KIND == kSammon) {
    term = e * e * invD;
    c = -e * invD * inv;
  } else if constexpr (KIND == kSmacof) {
    term = w * e * e;
    c = -2.f * w * e * inv;
  } else {  // kGuttman
    term = w * e * e;
    c = w * Dv * inv;
  }
}

}  // namespace tma_detail

// MODE 0: loss of up to two trial points; 1: loss + gradient at one point;
// 2 (fused): loss of two trial points + gradient at the first (the predicted
// Armijo acceptance, so the next iteration usually needs no gradient pass);
// 3 / 5: loss differences of two / the first trial (configurations Y and the scaled
// gradient); 6 / 7 (the device loop's sub-resolution "tiny" phase): 3 / 5 plus the
// gradient at the first trial point, from the same per-pair quantities (y_i - y_j -
// s_0 (g_i - g_j) and the trial distance the difference needs anyway: no extra MUFU) --
// one pass per tiny iteration instead of a difference pass and a gradient pass.
// Shared memory of one pass, all of it carved from the dynamic allocation (ring first), so one
// kernel can hold several modes' bodies (stress_tma_multi_kernel) without adding up static arrays.
template <int Q, int MODE>
constexpr size_t tma_smem_bytes() {
  constexpr bool DG = (MODE == 6 || MODE == 7);
  constexpr bool GRAD = (MODE == 1 || MODE == 2 || DG);
  constexpr int NCM = (MODE == 1) ? 1 : tma_detail::kTmaCand;
  constexpr int NS = GRAD ? tma_detail::kStagesGrad : tma_detail::kStages;
  return static_cast<size_t>(NS) * tma_detail::kHalfFloats * 4 + 128 /* barriers */ +
         (kThreads / 32) * kMaxCand * 8 /* sLoss */ + static_cast<size_t>(NCM) * kPT * Q * 4 /* sYi */ +
         static_cast<size_t>(2) * NCM * Q * kPT * 4 /* sYj */ + (GRAD ? static_cast<size_t>(Q) * kTG * kPT * 4 : 16);
}

template <int Q, int MODE, int KIND>
__device__ __forceinline__ void stress_tma_body(const PassArgs& a, unsigned char* dyn) {
  using namespace tma_detail;
  constexpr bool DG = (MODE == 6 || MODE == 7);      // difference + gradient at the first trial point
  constexpr bool DIFF = (MODE == 3 || MODE == 5 || DG);  // loss differences: configurations are Y and the gradient
  constexpr int NT = (MODE == 5 || MODE == 7) ? 1 : 2;   // trial steps of a difference pass (5, 7: the first only)
  constexpr bool GRAD = (MODE == 1 || MODE == 2 || DG);  // gradient accumulation (configuration 0 / DG: trial 0)
  constexpr int NCM = (MODE == 1) ? 1 : kTmaCand;
  // Q >= 3: a thread's 8 columns are processed as two groups of 4 (columns 4tj..4tj+3, then
  // 64+4tj..) per band, so only one group's coordinates and column sums are live at a time
  // (the full 8-column tile needs > 128 registers at Q = 3 and spilled 328-944 B per thread)
  // (GMDS_CSPLIT_DG / GMDS_CSPLIT_Q2: the same split for the q <= 2 difference + gradient passes /
  // for every q <= 2 loss and gradient mode -- all of them, so their loss sums stay bit-identical)
  constexpr bool CSPLIT = (Q >= 3) || (DG && GMDS_CSPLIT_DG) || (!DIFF && GMDS_CSPLIT_Q2);
  constexpr int NCH = CSPLIT ? 2 : 1;        // column groups per band
  constexpr int NYY = (kMT / 2) / NCH;       // column pairs (y, y+1) per group
  constexpr int NY = 2 * NYY;                // columns per group
  constexpr int NS = GRAD ? kStagesGrad : kStages;
  float* ring = reinterpret_cast<float*>(dyn);  // [NS][kHalfFloats]: half h lives in stage h % NS
  unsigned char* sp = dyn + static_cast<size_t>(NS) * kHalfFloats * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp);  // [NS]
  sp += 128;
  double (*sLoss)[kMaxCand] = reinterpret_cast<double (*)[kMaxCand]>(sp);  // [kThreads / 32][kMaxCand]
  sp += (kThreads / 32) * kMaxCand * 8;
  float (*sYi)[kPT][Q] = reinterpret_cast<float (*)[kPT][Q]>(sp);  // [NCM][kPT][Q]
  sp += static_cast<size_t>(NCM) * kPT * Q * 4;
  // [block parity][cand][k][column]: one coordinate of consecutive columns is contiguous, so a
  // thread's column pairs (y, y+1) arrive as one 16-byte load per 4 columns (no register moves
  // to form the FFMA2 operand pairs); double-buffered
  float (*sYj)[NCM][Q][kPT] = reinterpret_cast<float (*)[NCM][Q][kPT]>(sp);  // [2][NCM][Q][kPT]
  sp += static_cast<size_t>(2) * NCM * Q * kPT * 4;
  float* sRed = reinterpret_cast<float*>(sp);  // [Q kTG kPT] (GRAD): column partials of one block, all k at once

  if (a.halt && *a.halt) return;
  // device loop: the one-point pass (MODE 1: a solo pass at cand0, or the gradient pass at Y after a
  // slot-1 acceptance, GdState::fix) or the two-trial fused pass
  const double* y0p = a.Y[0];
  if constexpr (MODE == 1 || MODE == 2) {
    if (a.gds) {
      const bool one = a.gds->solo != 0 || a.gds->fix != 0;
      if (one != (MODE == 1)) return;
      if (MODE == 1 && a.gds->fix != 0) y0p = a.Y[2];
    }
  }
  // configuration c's coordinates (a.Y[c] stays a constant-bank read; no local array)
  auto Yof = [&](int c) { return (MODE == 1) ? y0p : a.Y[c]; };
  if constexpr (DG) {  // device loop: run only in the tiny phase, in the matching width
    if (a.gds && (a.gds->tiny == 0 || a.gds->stop != 0 || (a.gds->single != 0) != (NT == 1))) return;
  } else if constexpr (DIFF) {  // device loop: run only for a pending decision, in the matching width
    if (a.gds && (a.gds->pending == 0 || a.gds->stop != 0 || (a.gds->single != 0) != (NT == 1))) return;
  }
  const int tid = threadIdx.x;
  const int ti = tid / kTG, tj = tid % kTG;
  const int64_t chunk = blockIdx.x;
  const int64_t I = a.chunk_I[chunk];
  const int64_t J0 = a.chunk_J0[chunk];
  const int64_t J1 = min(J0 + a.chunk_len, a.nb);
  const int nblocks = static_cast<int>(J1 - J0);
  const int nhalves = kParts * nblocks;
  const int nc = (MODE == 1) ? 1 : (MODE >= 2 ? NCM : a.ncand);  // fused / difference passes: all configurations
  const float* __restrict__ D = static_cast<const float*>(a.D);
  const float* __restrict__ W = static_cast<const float*>(a.W);
  const float delta = static_cast<float>(a.huber_delta);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int h) {
    const int64_t J = J0 + h / kParts;
    const float* src = D + blk_index(I, J, a.nb) * (kPT * kPT) + (h % kParts) * kHalfFloats;
    uint64_t* bar = &bars[h % NS];
    mbar_expect_tx(bar, kHalfFloats * 4);
    bulk_g2s(ring + (h % NS) * kHalfFloats, src, kHalfFloats * 4, bar);
  };
  if (tid == 0)
    for (int h = 0; h < min(NS, nhalves); ++h) issue(h);

  if constexpr (Q == 2) {  // one 16-byte load per (candidate, row)
    const int r = tid & (kPT - 1);
    const int64_t i = I * kPT + r;
    for (int c = tid >> 7; c < NCM; c += 2) {
      const double2 v = (c < nc && i < a.n) ? reinterpret_cast<const double2*>(Yof(c))[i] : make_double2(0.0, 0.0);
      *reinterpret_cast<float2*>(&sYi[c][r][0]) = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    }
  } else {
    for (int e = tid; e < nc * kPT * Q; e += kThreads) {
      const int c = e / (kPT * Q), r = (e / Q) % kPT, k = e % Q;
      const int64_t i = I * kPT + r;
      sYi[c][r][k] = (i < a.n) ? static_cast<float>(Yof(c)[i * Q + k]) : 0.f;
    }
  }
  double lossacc[NCM];
#pragma unroll
  for (int c = 0; c < NCM; ++c) lossacc[c] = 0.0;
  double diffacc[DIFF ? 3 : 1] = {};  // DIFF: sum dE_0, sum dE_1, sum e_0^2
  float ds0 = static_cast<float>(a.dstep[0]), ds1 = static_cast<float>(a.dstep[1]);
  if (DIFF && a.gds) {  // device loop: the trial steps of the pending decision (slot order)
    const double st = a.gds->step;
    ds0 = static_cast<float>(a.gds->pred == 0 ? st : 0.5 * st);
    ds1 = static_cast<float>(a.gds->pred == 0 ? 0.5 * st : st);
  }
  // GRAD: this thread's 8 rows (4 per half) accumulate over every block of the
  // chunk in registers and are reduced across the 16 tj-threads once per chunk
  float rowsum[GRAD ? kParts : 1][GRAD ? kMR : 1][Q];
  if constexpr (GRAD) {
#pragma unroll
    for (int hh = 0; hh < kParts; ++hh)
#pragma unroll
      for (int x = 0; x < kMR; ++x)
#pragma unroll
        for (int k = 0; k < Q; ++k) rowsum[hh][x][k] = 0.f;
  }
  // this thread's 8 columns as (y, y+1) pairs, loaded once per block
  constexpr int NCMR = NCM;
  float2 yj2[NCMR][NYY][Q];
  // Q = 2: thread (c = tid / 128, r = tid % 128) stages point r of candidate c
  // as one 16-byte load, prefetched a block ahead into registers
  const int sc = tid >> 7, sr = tid & (kPT - 1);
  constexpr int NSC = (NCM + 1) / 2;  // configurations staged per thread (thread c stages c, c + 2)
  auto col_load = [&](int64_t J, int c) {
    const int64_t j = J * kPT + sr;
    return (c < nc && j < a.n) ? reinterpret_cast<const double2*>(Yof(c))[j] : make_double2(0.0, 0.0);
  };
  double2 ycol[NSC];
#pragma unroll
  for (int u = 0; u < NSC; ++u) ycol[u] = make_double2(0.0, 0.0);
  if constexpr (Q == 2)
#pragma unroll
    for (int u = 0; u < NSC; ++u) ycol[u] = col_load(J0, sc + 2 * u);

  // Barriers per block: one after the column coordinates are staged (their
  // buffer alternates, so no barrier is needed before writing it), one per
  // half to free its stage -- the second also publishes the column partials.
  for (int b = 0; b < nblocks; ++b) {
    const int64_t J = J0 + b;
    const int yb = b & 1;
    if constexpr (Q == 2) {
#pragma unroll
      for (int u = 0; u < NSC; ++u) {
        const int c = sc + 2 * u;
        if (c < NCM)
        {
          sYj[yb][c][0][sr] = static_cast<float>(ycol[u].x);
          sYj[yb][c][1][sr] = static_cast<float>(ycol[u].y);
        }
        if (b + 1 < nblocks) ycol[u] = col_load(J + 1, c);
      }
    } else {
      for (int e = tid; e < nc * kPT * Q; e += kThreads) {
        const int c = e / (kPT * Q), r = (e / Q) % kPT, k = e % Q;
        const int64_t j = J * kPT + r;
        sYj[yb][c][k][r] = (j < a.n) ? static_cast<float>(Yof(c)[j * Q + k]) : 0.f;
      }
    }
    __syncthreads();
    float2 colacc2[GRAD ? NYY : 1][Q];  // column sums of columns (y, y+1)
    auto load_cols = [&](int ch) {  // this group's column coordinates (and zeroed column sums)
#pragma unroll
      for (int c = 0; c < NCMR; ++c)
#pragma unroll
        for (int k = 0; k < Q; ++k) {  // columns 4tj..4tj+3 and 64+4tj..64+4tj+3: 16-byte loads
          if constexpr (!CSPLIT) {
            const float4 lo = (c < nc) ? *reinterpret_cast<const float4*>(&sYj[yb][c][k][4 * tj])
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 hi = (c < nc) ? *reinterpret_cast<const float4*>(&sYj[yb][c][k][64 + 4 * tj])
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            yj2[c][0][k] = make_float2(lo.x, lo.y);
            yj2[c][1][k] = make_float2(lo.z, lo.w);
            yj2[c][NYY - 2][k] = make_float2(hi.x, hi.y);
            yj2[c][NYY - 1][k] = make_float2(hi.z, hi.w);
          } else {
            const float4 v = (c < nc) ? *reinterpret_cast<const float4*>(&sYj[yb][c][k][64 * ch + 4 * tj])
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
            yj2[c][0][k] = make_float2(v.x, v.y);
            yj2[c][1][k] = make_float2(v.z, v.w);
          }
        }
      if constexpr (GRAD) {
#pragma unroll
        for (int y = 0; y < NYY; ++y)
#pragma unroll
          for (int k = 0; k < Q; ++k) colacc2[y][k] = make_float2(0.f, 0.f);
      }
    };
    if constexpr (!CSPLIT) load_cols(0);
    const int64_t blk = blk_index(I, J, a.nb);
    const bool edge = (I == J) || (J * kPT + kPT > a.n);
#pragma unroll
    for (int half = 0; half < kParts; ++half) {
      const int h = kParts * b + half;
      const int stage = h % NS;
      mbar_wait(&bars[stage], static_cast<uint32_t>((h / NS) & 1));
      const float* Ds = ring + stage * kHalfFloats;
      const float* Wb = W ? W + blk * (kPT * kPT) + half * kHalfFloats : nullptr;
      float2 lhalf[NCM];  // loss of this half, two fp32 lanes per candidate (widened once per half)
#pragma unroll
      for (int c = 0; c < NCM; ++c) lhalf[c] = make_float2(0.f, 0.f);
      float dhalf[3] = {0.f, 0.f, 0.f};  // DIFF: this half's sums
      // the row loop, instantiated per block kind (edge / packed / generic) so the
      // interior-block version is a branch-free, fully unrolled loop over the rows
      auto row_loop = [&](auto mode_tag, auto ch_tag) {
      constexpr int MODE_ROWS = decltype(mode_tag)::value;  // 0 packed, 1 edge, 2 generic
      constexpr int CH = decltype(ch_tag)::value;           // column group (CSPLIT), else 0
      constexpr int Y0 = CSPLIT ? 4 * CH : 0;               // first column slot (tcol) of the group
#pragma unroll
      for (int x = 0; x < kMR; ++x) {
        const int rloc = ti * kMR + x;           // row within the half
        const int ri = half * kHalfRows + rloc;  // row within the block
        const float4 v0 = *reinterpret_cast<const float4*>(Ds + rloc * kPT + 64 * CH + 4 * tj);
        float4 v1 = v0;
        if constexpr (!CSPLIT) v1 = *reinterpret_cast<const float4*>(Ds + rloc * kPT + 64 + 4 * tj);
        float dv[NY];
        dv[0] = v0.x, dv[1] = v0.y, dv[2] = v0.z, dv[3] = v0.w;
        if constexpr (!CSPLIT) dv[NY - 4] = v1.x, dv[NY - 3] = v1.y, dv[NY - 2] = v1.z, dv[NY - 1] = v1.w;
        float wv[NY];
#pragma unroll
        for (int y = 0; y < NY; ++y) wv[y] = Wb ? Wb[rloc * kPT + tcol(tj, Y0 + y)] : 1.f;
        float yi[NCM][Q];
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
          if constexpr (Q == 2) {
            const float2 t = (c < nc) ? *reinterpret_cast<const float2*>(&sYi[c][ri][0]) : make_float2(0.f, 0.f);
            yi[c][0] = t.x;
            yi[c][1] = t.y;
          } else {
#pragma unroll
            for (int k = 0; k < Q; ++k) yi[c][k] = (c < nc) ? sYi[c][ri][k] : 0.f;
          }
        }
        // interior blocks: no masks at all; edge blocks (diagonal / last column block) mask per pair
        auto pairs = [&](auto edge_tag) {
          constexpr bool EDGE = decltype(edge_tag)::value;
#pragma unroll
          for (int y = 0; y < NY; ++y) {
            const int rj = tcol(tj, Y0 + y);
            bool keep = true;
            if constexpr (EDGE) keep = (J * kPT + rj < a.n) && (I != J || ri < rj);
            const float Dv = dv[y];
            const float invD = (KIND == kSammon) ? 1.f / fmaxf(Dv, FLT_MIN) : 0.f;
#pragma unroll
            for (int c = 0; c < NCMR; ++c) {
              if (c >= nc) break;
              float dy[Q];
              float d2 = 0.f;
#pragma unroll
              for (int k = 0; k < Q; ++k) {
                dy[k] = yi[c][k] - ((y & 1) ? yj2[c][y / 2][k].y : yj2[c][y / 2][k].x);
                d2 = fmaf(dy[k], dy[k], d2);
              }
              const float inv = rsqrtf(fmaxf(d2, FLT_MIN));
              const float dist = d2 * inv;
              float term, cc;
              kind_terms<KIND>(Dv, invD, dist, inv, wv[y], delta, term, cc);
              if constexpr (EDGE) {
                term = keep ? term : 0.f;
                cc = keep ? cc : 0.f;
              }
              lhalf[c].x += term;
              if constexpr (GRAD) {
                if (c != 0) continue;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                  rowsum[half][x][k] = fmaf(cc, dy[k], rowsum[half][x][k]);
                  float& ca = (y & 1) ? colacc2[y / 2][k].y : colacc2[y / 2][k].x;
                  ca = fmaf(-cc, dy[k], ca);
                }
              }
            }
          }
        };
        // DIFF (e^2 kinds, unweighted): per pair, with dy = y_i - y_j and dg = g_i - g_j,
        // a_t = |dy - s_t dg|^2 - |dy|^2 = s_t (s_t |dg|^2 - 2 <dy, dg>) is formed from the
        // small quantities, dist_t - dist_0 = a_t / (dist_t + dist_0) and
        // e_t^2 - e_0^2 = (dist_t - dist_0) (dist_t - dist_0 - 2 e_0): the loss changes
        // keep fp32's relative precision however small the step (the direct e_t^2 would
        // lose them below one ulp of e).
        auto pairs_diff = [&]() {
#pragma unroll
          for (int y = 0; y < NY; ++y) {
            const int rj = tcol(tj, Y0 + y);
            bool keep = true;
            if (edge) keep = (J * kPT + rj < a.n) && (I != J || ri < rj);
            float dy[Q], dg[Q];
            float d0 = FLT_MIN, pp = 0.f, qq = 0.f;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              dy[k] = yi[0][k] - ((y & 1) ? yj2[0][y / 2][k].y : yj2[0][y / 2][k].x);
              dg[k] = yi[1][k] - ((y & 1) ? yj2[1][y / 2][k].y : yj2[1][y / 2][k].x);
              d0 = fmaf(dy[k], dy[k], d0);
              pp = fmaf(dy[k], dg[k], pp);
              qq = fmaf(dg[k], dg[k], qq);
            }
            const float dist0 = d0 * rsqrt_mufu(d0);
            const float e0 = dv[y] - dist0;
            float t0 = 0.f, t1 = 0.f;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const float st = t ? ds1 : ds0;
              const float at = st * fmaf(st, qq, -2.f * pp);
              const float dt2 = fmaxf(d0 + at, FLT_MIN);
              const float rt = rsqrt_mufu(dt2);
              const float distt = dt2 * rt;
              const float dd = at / (distt + dist0);  // dist_t - dist_0
              const float de = dd * (dd - 2.f * e0);  // e_t^2 - e_0^2
              if (t) t1 = de; else t0 = de;
              if constexpr (DG) {
                if (t == 0) {  // kruskal gradient at y - s_0 g: c = -(D - dist_0') / dist_0'
                  const float cc = keep ? -(dv[y] - distt) * rt : 0.f;
#pragma unroll
                  for (int k = 0; k < Q; ++k) {
                    const float dyt = fmaf(-st, dg[k], dy[k]);
                    rowsum[half][x][k] = fmaf(cc, dyt, rowsum[half][x][k]);
                    float& ca = (y & 1) ? colacc2[y / 2][k].y : colacc2[y / 2][k].x;
                    ca = fmaf(-cc, dyt, ca);
                  }
                }
              }
            }
            if (keep) {
              dhalf[0] += t0;
              dhalf[1] += t1;
              dhalf[2] = fmaf(e0, e0, dhalf[2]);
            }
          }
        };
        // DIFF on interior blocks: the same on column pairs (y, y+1) with packed fp32 math
        auto pairs_diff_packed = [&]() {
          float2 dvp[NYY];
          dvp[0] = make_float2(v0.x, v0.y), dvp[1] = make_float2(v0.z, v0.w);
          if constexpr (!CSPLIT) dvp[NYY - 2] = make_float2(v1.x, v1.y), dvp[NYY - 1] = make_float2(v1.z, v1.w);
          float2 yY[Q], yG[Q];
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            yY[k] = make_float2(yi[0][k], yi[0][k]);
            yG[k] = make_float2(yi[1][k], yi[1][k]);
          }
          const float2 s0v = make_float2(ds0, ds0), s1v = make_float2(ds1, ds1);
          const float2 m2 = make_float2(-2.f, -2.f);
          float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0;
          float2 racc[DG ? Q : 1];  // DG: this row's gradient sums at the first trial point
#pragma unroll
          for (int k = 0; k < (DG ? Q : 1); ++k) racc[k] = make_float2(0.f, 0.f);
          const float2 ms0v = make_float2(-ds0, -ds0);
#pragma unroll
          for (int yy = 0; yy < NYY; ++yy) {
            float2 d0 = make_float2(FLT_MIN, FLT_MIN), pp = make_float2(0.f, 0.f), qq = pp;
            float2 dyv[Q], dgv[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              const float2 dy = f2sub(yY[k], yj2[0][yy][k]);
              const float2 dg = f2sub(yG[k], yj2[1][yy][k]);
              dyv[k] = dy;
              dgv[k] = dg;
              d0 = f2fma(dy, dy, d0);
              pp = f2fma(dy, dg, pp);
              qq = f2fma(dg, dg, qq);
            }
            const float2 dist0 = f2mul(d0, make_float2(rsqrt_mufu(d0.x), rsqrt_mufu(d0.y)));
            const float2 e0 = f2sub(dvp[yy], dist0);
            a2 = f2fma(e0, e0, a2);
            const float2 m2p = f2mul(pp, m2);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const float2 sv = t ? s1v : s0v;
              const float2 at = f2mul(sv, f2fma(sv, qq, m2p));
              float2 dt2 = f2add(d0, at);
              dt2.x = fmaxf(dt2.x, FLT_MIN);
              dt2.y = fmaxf(dt2.y, FLT_MIN);
              const float2 rt = make_float2(rsqrt_mufu(dt2.x), rsqrt_mufu(dt2.y));
              const float2 distt = f2mul(dt2, rt);
              const float2 den = f2add(distt, dist0);
              const float2 dd = f2mul(at, make_float2(rcp_mufu(den.x), rcp_mufu(den.y)));
              const float2 de = f2mul(dd, f2fma(e0, m2, dd));
              if (t) a1 = f2add(a1, de); else a0 = f2add(a0, de);
              if constexpr (DG) {
                if (t == 0) {  // kruskal gradient at y - s_0 g (pairs_packed's conventions: u = e / dist)
                  const float2 u = f2mul(f2sub(dvp[yy], distt), rt);
#pragma unroll
                  for (int k = 0; k < Q; ++k) {
                    const float2 dyt = f2fma(ms0v, dgv[k], dyv[k]);
                    racc[k] = f2fma(u, dyt, racc[k]);
                    colacc2[yy][k] = f2fma(u, dyt, colacc2[yy][k]);
                  }
                }
              }
            }
          }
          if constexpr (DG) {
#pragma unroll
            for (int k = 0; k < Q; ++k) rowsum[half][x][k] += -(racc[k].x + racc[k].y);
          }
          dhalf[0] += a0.x + a0.y;
          dhalf[1] += a1.x + a1.y;
          dhalf[2] += a2.x + a2.y;
        };
        // Kruskal / Guttman, interior, unweighted: two pairs (y, y+1) per
        // FADD2 / FMUL2 / FFMA2, bare MUFU.RSQ on d2 seeded with FLT_MIN (so no
        // clamp: coincident points give dy = 0 and add exactly 0)
        auto pairs_packed = [&]() {
          constexpr bool KR = (KIND == kKruskal);
          float2 dvp[NYY];
          dvp[0] = make_float2(v0.x, v0.y), dvp[1] = make_float2(v0.z, v0.w);
          if constexpr (!CSPLIT) dvp[NYY - 2] = make_float2(v1.x, v1.y), dvp[NYY - 1] = make_float2(v1.z, v1.w);
#pragma unroll
          for (int c = 0; c < NCMR; ++c) {
            if (c >= nc) break;
            float2 yi2[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) yi2[k] = make_float2(yi[c][k], yi[c][k]);
            float2 lacc = lhalf[c];
            float2 racc[Q];  // this row's gradient sums over columns (y, y+1)
#pragma unroll
            for (int k = 0; k < Q; ++k) racc[k] = make_float2(0.f, 0.f);
#pragma unroll
            for (int yy = 0; yy < NYY; ++yy) {
              float2 dy2[Q];
              float2 d2 = make_float2(FLT_MIN, FLT_MIN);
#pragma unroll
              for (int k = 0; k < Q; ++k) {
                dy2[k] = f2sub(yi2[k], yj2[c][yy][k]);
                d2 = f2fma(dy2[k], dy2[k], d2);
              }
              const float2 inv = make_float2(rsqrt_mufu(d2.x), rsqrt_mufu(d2.y));
              const float2 dist = f2mul(d2, inv);
              const float2 e = f2sub(dvp[yy], dist);
              lacc = f2fma(e, e, lacc);  // kruskal and guttman: term = e^2
              if constexpr (GRAD) {
                if (c != 0) continue;
                // row += c dy, column -= c dy with kruskal c = -e/dist = -u,
                // guttman c = D/dist = u
                const float2 u = KR ? f2mul(e, inv) : f2mul(dvp[yy], inv);
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                  racc[k] = f2fma(u, dy2[k], racc[k]);
                  if constexpr (KR)
                    colacc2[yy][k] = f2fma(u, dy2[k], colacc2[yy][k]);
                  else
                    colacc2[yy][k] = f2sub(colacc2[yy][k], f2mul(u, dy2[k]));
                }
              }
            }
            lhalf[c] = lacc;
            if constexpr (GRAD) {
              if (c == 0) {
#pragma unroll
                for (int k = 0; k < Q; ++k)  // row += c dy: kruskal c = -u, guttman c = u
                  rowsum[half][x][k] += KR ? -(racc[k].x + racc[k].y) : (racc[k].x + racc[k].y);
              }
            }
          }
        };
        if constexpr (DIFF) {
          if constexpr (MODE_ROWS == 0) pairs_diff_packed(); else pairs_diff();
        }
        else if constexpr (MODE_ROWS == 1)
          pairs(std::true_type{});
        else if constexpr (MODE_ROWS == 0)
          pairs_packed();
        else
          pairs(std::false_type{});
      }
      };
      auto group = [&](auto ch_tag) {
        constexpr int CH = decltype(ch_tag)::value;
        if constexpr (CSPLIT) load_cols(CH);
        if (edge)
          row_loop(std::integral_constant<int, 1>{}, ch_tag);
        else if ((KIND == kKruskal || KIND == kGuttman) && !Wb)
          row_loop(std::integral_constant<int, 0>{}, ch_tag);
        else
          row_loop(std::integral_constant<int, 2>{}, ch_tag);
        if constexpr (CSPLIT && GRAD) {  // this group's column sums of the band -> sRed (each cell one thread's)
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            float4* dst = reinterpret_cast<float4*>(sRed + (k * kTG + ti) * kPT + 64 * CH + 4 * tj);
            float4 v = make_float4(colacc2[0][k].x, colacc2[0][k].y, colacc2[1][k].x, colacc2[1][k].y);
            if (half != 0) {
              const float4 o = *dst;
              v.x += o.x, v.y += o.y, v.z += o.z, v.w += o.w;
            }
            *dst = v;
          }
        }
      };
      group(std::integral_constant<int, 0>{});
      if constexpr (CSPLIT) group(std::integral_constant<int, 1>{});
#pragma unroll
      for (int c = 0; c < NCM; ++c) lossacc[c] += static_cast<double>(lhalf[c].x) + static_cast<double>(lhalf[c].y);
      if constexpr (DIFF) {
#pragma unroll
        for (int c = 0; c < 3; ++c) diffacc[c] += static_cast<double>(dhalf[c]);
      }
      if constexpr (GRAD && !CSPLIT) {
        if (half == kParts - 1) {
#pragma unroll
          for (int k = 0; k < Q; ++k) {  // columns 4tj..+3 and 64+4tj..+3: two 16-byte stores
            float* dst = sRed + (k * kTG + ti) * kPT;
            *reinterpret_cast<float4*>(dst + 4 * tj) =
                make_float4(colacc2[0][k].x, colacc2[0][k].y, colacc2[1][k].x, colacc2[1][k].y);
            *reinterpret_cast<float4*>(dst + 64 + 4 * tj) =
                make_float4(colacc2[2][k].x, colacc2[2][k].y, colacc2[3][k].x, colacc2[3][k].y);
          }
        }
      }
      __syncthreads();  // stage `half` is free (and, after half 1, the column partials are in sRed)
      if (tid == 0 && h + NS < nhalves) issue(h + NS);
    }
    if constexpr (GRAD) {  // column partials of block J: 16 ti-threads per column, fixed order
      for (int e = tid; e < kPT * Q; e += kThreads) {
        const int col = e % kPT, k = e / kPT;  // a warp reads 32 consecutive columns of one k
        float s = 0.f;
#pragma unroll
        for (int t = 0; t < kTG; ++t) s += sRed[(k * kTG + t) * kPT + col];
        reinterpret_cast<float*>(a.colpart)[(blk * kPT + col) * Q + k] = s;  // fp32 partials (exact as summed)
      }
    }
  }
  if constexpr (GRAD) {  // row partials of the chunk: xor-trees over the 16 tj-threads of each row
#pragma unroll
    for (int hh = 0; hh < kParts; ++hh)
#pragma unroll
      for (int x = 0; x < kMR; ++x)
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          float v = rowsum[hh][x][k];
#pragma unroll
          for (int m = 8; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
          if (tj == 0) reinterpret_cast<float*>(a.rowpart)[(chunk * kPT + hh * kHalfRows + ti * kMR + x) * Q + k] = v;
        }
  }
#pragma unroll
  for (int c = 0; c < NCM; ++c) {
    double v = lossacc[c];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((tid & 31) == 0) sLoss[tid >> 5][c] = v;
  }
  if constexpr (DIFF) {
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v = diffacc[c];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
      if ((tid & 31) == 0) sLoss[tid >> 5][c] = v;
    }
    __syncthreads();
    if (tid == 0) {  // slots: raw at Y - s0 g, raw at Y - s1 g, raw at Y (slot 0 as a trial pass leaves it)
      double sd[3] = {0.0, 0.0, 0.0};
      for (int w = 0; w < kThreads / 32; ++w)
        for (int c = 0; c < 3; ++c) sd[c] += sLoss[w][c];
      a.losspart[chunk * kMaxCand + 0] = sd[2] + sd[0];
      a.losspart[chunk * kMaxCand + 1] = sd[2] + (NT == 2 ? sd[1] : 0.0);  // single: Y (never accepted)
      a.losspart[chunk * kMaxCand + 2] = sd[2];
    }
    return;
  }
  __syncthreads();
  if (tid < nc) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += sLoss[w][tid];
    a.losspart[chunk * kMaxCand + tid] = s;
  }
}

template <int Q, int MODE, int KIND>
__global__ void __launch_bounds__(kThreads, GMDS_TMA_MINB(MODE, Q)) stress_tma_kernel(PassArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char dyn[];
  stress_tma_body<Q, MODE, KIND>(a, dyn);
}

// Device loop, kruskal, q <= 3: the passes a unit of the enqueued chain may need, behind two
// three launches instead of six (each skipped pass used to cost an empty launch): WHICH 0 = the
// difference pass of a pending decision (MODE 3, or 5 when single), WHICH 1 = the unit's main
// pass -- two-trial fused (2) or one-point (1: solo / fix), WHICH 2 = the tiny phase's
// difference + gradient pass (6 / 7; with the main pass in one kernel the fused body spilled
// 388 B at q = 2).  The GdState the passes' own guards read selects the body.
template <int Q, int WHICH>
__global__ void __launch_bounds__(kThreads, 2) stress_tma_multi_kernel(PassArgs a, PassArgs d) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char dyn[];
  const GdState* g = a.gds;
  if (g->stop != 0) return;
  if constexpr (WHICH == 0) {
    if (g->pending == 0) return;
    if (g->single != 0) stress_tma_body<Q, 5, kKruskal>(d, dyn);
    else stress_tma_body<Q, 3, kKruskal>(d, dyn);
  } else if constexpr (WHICH == 1) {
    if (g->tiny != 0) return;
    if (g->solo != 0 || g->fix != 0) stress_tma_body<Q, 1, kKruskal>(a, dyn);
    else stress_tma_body<Q, 2, kKruskal>(a, dyn);
  } else {
    if (g->tiny == 0) return;
    if (g->single != 0) stress_tma_body<Q, 7, kKruskal>(d, dyn);
    else stress_tma_body<Q, 6, kKruskal>(d, dyn);
  }
}

template <int Q>
constexpr size_t tma_multi_smem() {
  size_t m = tma_smem_bytes<Q, 1>();
  if (tma_smem_bytes<Q, 2>() > m) m = tma_smem_bytes<Q, 2>();
  if (tma_smem_bytes<Q, 3>() > m) m = tma_smem_bytes<Q, 3>();
  if (tma_smem_bytes<Q, 6>() > m) m = tma_smem_bytes<Q, 6>();
  return m;
}

#define GMDS_TMA_KIND(QQ, KK)                                                                              \
  case KK:                                                                                                 \
    GMDS_CUDA(cudaFuncSetAttribute(stress_tma_kernel<QQ, MODE, KK>,                                        \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,                            \
                                   static_cast<int>(tma_smem_bytes<QQ, MODE>())));                         \
    launch_pdl(stress_tma_kernel<QQ, MODE, KK>, dim3(g), dim3(kThreads), tma_smem_bytes<QQ, MODE>(), st, a); \
    break;
#define GMDS_TMA_Q(QQ)                                                                                    \
  case QQ:                                                                                                \
    switch (a.kind) {                                                                                     \
      GMDS_TMA_KIND(QQ, kKruskal) GMDS_TMA_KIND(QQ, kHuber) GMDS_TMA_KIND(QQ, kSammon)                    \
      GMDS_TMA_KIND(QQ, kSmacof) GMDS_TMA_KIND(QQ, kGuttman)                                              \
      default: fail(GMDS_ERROR, "stress pass: bad kind");                                                 \
    }                                                                                                     \
    break;
#define GMDS_TMA_SWITCH                                                                                   \
    const unsigned g = static_cast<unsigned>(a.nchunks);                                                  \
    switch (Q) {                                                                                          \
      GMDS_TMA_Q(1) GMDS_TMA_Q(2) GMDS_TMA_Q(3) GMDS_TMA_Q(4)                                             \
      default: fail(GMDS_ERROR, "stress pass: unsupported padded dimension");                             \
    }
#define GMDS_INSTANTIATE_TMA_DIFF                                                                         \
  void launch_pass_diff_f32(const PassArgs& a, int Q, cudaStream_t st) {                                  \
    constexpr int MODE = 3;                                                                               \
    GMDS_TMA_SWITCH                                                                                       \
    count_launch();                                                                                       \
    check_launch("stress_tma_kernel (difference)");                                                       \
  }
#define GMDS_INSTANTIATE_TMA_DIFF1                                                                        \
  void launch_pass_diff1_f32(const PassArgs& a, int Q, cudaStream_t st) {                                 \
    constexpr int MODE = 5;                                                                               \
    GMDS_TMA_SWITCH                                                                                       \
    count_launch();                                                                                       \
    check_launch("stress_tma_kernel (difference, first trial)");                                          \
  }
#define GMDS_TMA_DG_Q(QQ)                                                                                 \
  case QQ:                                                                                                \
    GMDS_CUDA(cudaFuncSetAttribute(stress_tma_kernel<QQ, MODE, kKruskal>,                                  \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,                            \
                                   static_cast<int>(tma_smem_bytes<QQ, MODE>())));                         \
    launch_pdl(stress_tma_kernel<QQ, MODE, kKruskal>, dim3(g), dim3(kThreads), tma_smem_bytes<QQ, MODE>(), st, a); \
    break;
#define GMDS_INSTANTIATE_TMA_DG                                                                           \
  void launch_pass_diffgrad_f32(const PassArgs& a, int Q, bool single, cudaStream_t st) {                 \
    if (a.kind != kKruskal) fail(GMDS_ERROR, "difference + gradient pass: kruskal only");                 \
    const unsigned g = static_cast<unsigned>(a.nchunks);                                                  \
    if (single) {                                                                                         \
      constexpr int MODE = 7;                                                                             \
      switch (Q) {                                                                                        \
        GMDS_TMA_DG_Q(1) GMDS_TMA_DG_Q(2) GMDS_TMA_DG_Q(3)                                                \
        default: fail(GMDS_ERROR, "difference + gradient pass: q <= 3");                                  \
      }                                                                                                   \
    } else {                                                                                              \
      constexpr int MODE = 6;                                                                             \
      switch (Q) {                                                                                        \
        GMDS_TMA_DG_Q(1) GMDS_TMA_DG_Q(2) GMDS_TMA_DG_Q(3)                                                \
        default: fail(GMDS_ERROR, "difference + gradient pass: q <= 3");                                  \
      }                                                                                                   \
    }                                                                                                     \
    count_launch();                                                                                       \
    check_launch("stress_tma_kernel (difference + gradient)");                                            \
  }
#define GMDS_TMA_MULTI_Q(QQ)                                                                              \
  case QQ:                                                                                                \
    if (which == 0) {                                                                                     \
      GMDS_CUDA(cudaFuncSetAttribute(stress_tma_multi_kernel<QQ, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     static_cast<int>(tma_multi_smem<QQ>())));                            \
      launch_pdl(stress_tma_multi_kernel<QQ, 0>, dim3(g), dim3(kThreads), tma_multi_smem<QQ>(), st, a, d); \
    } else if (which == 2) {                                                                              \
      GMDS_CUDA(cudaFuncSetAttribute(stress_tma_multi_kernel<QQ, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     static_cast<int>(tma_multi_smem<QQ>())));                            \
      launch_pdl(stress_tma_multi_kernel<QQ, 2>, dim3(g), dim3(kThreads), tma_multi_smem<QQ>(), st, a, d); \
    } else {                                                                                              \
      GMDS_CUDA(cudaFuncSetAttribute(stress_tma_multi_kernel<QQ, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     static_cast<int>(tma_multi_smem<QQ>())));                            \
      launch_pdl(stress_tma_multi_kernel<QQ, 1>, dim3(g), dim3(kThreads), tma_multi_smem<QQ>(), st, a, d); \
    }                                                                                                     \
    break;
#define GMDS_INSTANTIATE_TMA_MULTI                                                                        \
  void launch_pass_multi_f32(const PassArgs& a, const PassArgs& d, int Q, int which, cudaStream_t st) {   \
    if (a.kind != kKruskal || !a.gds) fail(GMDS_ERROR, "multi pass: kruskal device loop only");           \
    const unsigned g = static_cast<unsigned>(a.nchunks);                                                  \
    switch (Q) {                                                                                          \
      GMDS_TMA_MULTI_Q(1) GMDS_TMA_MULTI_Q(2) GMDS_TMA_MULTI_Q(3)                                         \
      default: fail(GMDS_ERROR, "multi pass: q <= 3");                                                    \
    }                                                                                                     \
    count_launch();                                                                                       \
    check_launch("stress_tma_multi_kernel");                                                              \
  }
#define GMDS_INSTANTIATE_TMA_FUSED                                                                        \
  void launch_pass_fused_f32(const PassArgs& a, int Q, cudaStream_t st) {                                 \
    constexpr int MODE = 2;                                                                               \
    GMDS_TMA_SWITCH                                                                                       \
    count_launch();                                                                                       \
    check_launch("stress_tma_kernel (fused)");                                                            \
  }
#define GMDS_INSTANTIATE_TMA_SOLO                                                                         \
  void launch_pass_solo_f32(const PassArgs& a, int Q, cudaStream_t st) {                                  \
    constexpr int MODE = 1;                                                                               \
    GMDS_TMA_SWITCH                                                                                       \
    count_launch();                                                                                       \
    check_launch("stress_tma_kernel (solo)");                                                             \
  }
#define GMDS_INSTANTIATE_TMA(GR)                                                                          \
  template <>                                                                                             \
  void launch_pass_td<float, GR>(const PassArgs& a, int Q, cudaStream_t st) {                              \
    constexpr int MODE = GR ? 1 : 0;                                                                      \
    const unsigned g = static_cast<unsigned>(a.nchunks);                                                  \
    switch (Q) {                                                                                          \
      GMDS_TMA_Q(1) GMDS_TMA_Q(2) GMDS_TMA_Q(3) GMDS_TMA_Q(4)                                             \
      default: fail(GMDS_ERROR, "stress pass: unsupported padded dimension");                             \
    }                                                                                                     \
  }

}  // namespace gmds
