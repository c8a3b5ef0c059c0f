// Stress-pass launch interface (host side).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "gmds.h"

namespace gmds {

enum PassKind { kKruskal = 0, kHuber = 1, kSammon = 2, kSmacof = 3, kGuttman = 4 };
constexpr int kMaxCand = 4;
constexpr int kTmaCands = 2;  // trial points of an fp32 (TMA) pass

struct PassArgs {
  const void* D;            // packed image (storage dtype)
  const void* W;            // packed weights image or nullptr
  int64_t n, nb;            // rows, ceil(n / kPT)
  const double* Y[kMaxCand];  // n x Q row-major (padded), one per candidate
  int ncand;
  int kind;
  double huber_delta;
  const int64_t* chunk_I;   // [nchunks]
  const int64_t* chunk_J0;  // [nchunks]
  int64_t chunk_len;
  int64_t nchunks;
  double* rowpart;          // [nchunks][kPT][Q]  (rows kernel: [n][q] final; TMA passes: fp32 partials)
  double* colpart;          // [nblk][kPT][Q]     (TMA passes: fp32 partials)
  double* losspart;         // [nchunks][kMaxCand] (rows kernel: [n][kMaxCand])
  int64_t cand_stride_row;  // elements between candidates' rowpart images (fused trial passes)
  int64_t cand_stride_col;  // elements between candidates' colpart images
  const int* halt;          // device flag: nonzero -> the pass is a no-op (device-resident loops)
  double dstep[2];          // difference passes: trial steps (Y[0] = Y, Y[1] = scaled gradient)
  const struct GdState* gds;  // difference passes in the device loop: run only if gds->pending, steps from it
};

// Device-resident gradient descent state (double-buffered by iteration parity)
struct GdState {
  double f, step;
  double t0, t1, gsq;  // the last decided pass: raw trial losses (slot order), |g|^2
  int it, pred, stop, stalled;  // stop: 0 running, 1 finished, 2 iteration handed to the host
  int ndiff;                    // difference passes run so far (pass accounting)
  int pending;                  // 1: the fused pass's trial losses were below fp32 resolution; a
                                // difference pass follows and gd_step phase 1 decides on it
  int tiny;                     // 1: the last change was far below resolution -- the next iteration
                                // runs the gradient pass only, and its decision defers directly
  int halt_fused, halt_grad;    // halt flags of the next fused pass / gradient-only pass
  int single;                   // the pending decision's difference pass evaluates the first trial only
  int solo;                     // the next trial pass evaluates slot 0 only (loss + gradient at cand0): the
                                // full step was accepted with a resolved margin last time (pred == 0), so
                                // the half step's loss would go unread; a miss hands the iteration to the host
  int solo_miss;                // stop == 2 after a solo pass: t1 (the loss at cand1) was not evaluated
  int streak;                   // consecutive full-step acceptances on resolved sums (solo needs 2)
  // Decisions the predicted slot does not cover, kept on the device (one extra unit of the
  // enqueued chain each, no host round trip):
  int fix;                      // the trial in slot 1 was accepted: Y moved there, the next pass is the
                                // gradient pass at Y (MODE 1), and the gd_step after it forms the trials
  int rt;                       // neither trial was accepted: the trials were re-formed at step / 4 and
                                // step / 8 (natural slot order, embed.cpp:242-250's further halvings) and
                                // the next decision tests those (no fp32 re-evaluation, as on the host)
  int halv;                     // halvings spent on this iteration (the reference allows 60)
  int nextra;                   // passes run for these units (pass accounting)
  int init;                     // with fix: the pass at Y is the fit's first -- its loss is f(Y0), history[it]
};

struct Steps {
  double v[kMaxCand];
  int n;
};

// fp32 storage: could the Armijo decision on fp32 sums differ from the reference's fp64
// one (embed.cpp:242-250)?  The trials are tested in the reference's order (step, then
// step / 2) and the first accepted wins, so the decision is unresolved when a TESTED
// trial's loss lies within `tol` of its threshold f - 1e-4 s |g|^2 (f_step, f_half: the
// losses at step and step / 2).  Host and device use the same rounding (no FMA).
#if defined(__CUDACC__)
__host__ __device__
#endif
inline bool armijo_unresolved(double f, double step, double gsq, double f_step, double f_half, double tol) {
  for (int c = 0; c < 2; ++c) {
#if defined(__CUDA_ARCH__)
    const double sc = c == 0 ? step : __dmul_rn(step, 0.5);
    const double thr = __dsub_rn(f, __dmul_rn(__dmul_rn(1e-4, sc), gsq));
    const double fc = c == 0 ? f_step : f_half;
    if (fabs(__dsub_rn(fc, thr)) <= tol) return true;
#else
    const double sc = c == 0 ? step : step * 0.5;
    const double thr = f - 1e-4 * sc * gsq;
    const double fc = c == 0 ? f_step : f_half;
    if (std::fabs(fc - thr) <= tol) return true;
#endif
    if (fc <= thr) return false;  // accepted: later trials are not tested
  }
  return false;
}

void launch_stress_pass(const PassArgs& a, int q, bool grad, gmds_dtype storage, cudaStream_t st);
// gpart (reduce_rows_scratch(nb, q) doubles): the two-level reduction; nullptr: one-level
void launch_reduce_rows(const double* rowpart, const double* colpart, const int64_t* strip_first, int64_t n,
                        int64_t nb, int q, double* out, cudaStream_t st, double* gpart = nullptr,
                        const int* halt = nullptr, bool f32parts = false, const double* losspart = nullptr,
                        int64_t nparts = 0, int lstride = 0, double* sums = nullptr);
void launch_gd_step(GdState* st2, int par, const double* losspart, int64_t nparts, int stride, const double* sqprev,
                    int nsq, double* sqnext, int kind, double sum_sq, double sum, double* Y, double* cand0,
                    double* cand1, double* gnext, const double* gpart, int Q, double* graw, int64_t m,
                    double* history, int max_iters, double rel_tol, const double* pre, double precise_rel,
                    int phase, cudaStream_t st, const double* xred = nullptr, const double* dsum = nullptr,
                    bool tiny_ok = false, bool solo_ok = false, bool ondev = false);
// row-sharded device loop: gradient groups -> xred[0, nQ), the pass's trial-loss sums -> xred[nQ, nQ + 2)
void launch_shard_collect(const double* gpart, int64_t n, int Q, const double* losspart, int64_t nparts, int stride,
                          double* xred, const int* halt, cudaStream_t st);
size_t reduce_rows_scratch(int64_t nb, int q);
void launch_sum_parts(const double* part, int64_t count, int stride, int m, double* out, cudaStream_t st);
// fp32 storage, q <= 4: losses at a.Y[0], a.Y[1] and the gradient partials at a.Y[0] in one pass
void launch_pass_fused_f32(const PassArgs& a, int Q, cudaStream_t st);
// device loop: loss + gradient at a.Y[0] only; runs when a.gds->solo (the fused pass then exits)
void launch_pass_solo_f32(const PassArgs& a, int Q, cudaStream_t st);
// fp32 storage, fp64 arithmetic: loss of up to kMaxCand points
void launch_pass_precise(const PassArgs& a, int Q, cudaStream_t st);
// fp32 storage, e^2 kinds: losspart slots (sum of e_t^2 - e_0^2 at Y - s_t g for t = 0, 1; sum e_0^2 at Y)
void launch_pass_diff_f32(const PassArgs& a, int Q, cudaStream_t st);
// the same for the first trial only (slot 1 then holds the loss at Y; device loop, tiny mode)
void launch_pass_diff1_f32(const PassArgs& a, int Q, cudaStream_t st);
// kruskal, device loop's tiny phase: the difference pass (both trials, or the first when single)
// plus the raw gradient at a.Y[2] (the first trial point) -- runs only when a.gds->tiny
void launch_pass_diffgrad_f32(const PassArgs& a, int Q, bool single, cudaStream_t st);
// kruskal device loop, q <= 3: one launch for whichever pass the GdState (a.gds) asks for --
// which 0: the pending decision's difference pass (d: its arguments); which 1: the unit's main
// pass (a: the fused / one-point arguments, d: the difference + gradient pass's)
void launch_pass_multi_f32(const PassArgs& a, const PassArgs& d, int Q, int which, cudaStream_t st);
constexpr int kSqBlocks = 148;
void launch_scale_sqnorm(double* g, int64_t m, double scale, double* out, double* part, cudaStream_t st);
// raw loss (from the pass partials) -> scale -> g *= scale, trial points T0/T1, |g|^2 block partials;
// returns the number of partials written to sqpart (<= kSqBlocks)
int launch_finish_grad(const double* losspart, int64_t nparts, int stride, int kind, double sum_sq, double sum,
                       double* g, const double* Y, int64_t m, double s0, double s1, double* T0, double* T1,
                       double* sqpart, double* raw_out, cudaStream_t st, const double* raw_in = nullptr);
void launch_axpy_cand(const double* Y, const double* G, int64_t m, const Steps& s, double* const* outs,
                      cudaStream_t st);
void launch_scale(const double* in, int64_t m, double divisor, double* out, cudaStream_t st);
// out (n x Q) = V^+ (n x n, symmetric) times bz (n x Q); Q <= 4
void launch_vpinv_apply(const double* Vp, const double* bz, int64_t n, int Q, double* out, cudaStream_t st);

}  // namespace gmds
