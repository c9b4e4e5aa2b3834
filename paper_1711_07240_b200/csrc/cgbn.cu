// cgbn.cu — sm_100a kernels and the C ABI (include/cgbn.h) of the CGBN hot path.
// One translation unit: cgbn_common.cuh (geometry, vector I/O), cgbn_ops.cuh (fp64
// arithmetic, finishers, reduction ops), cgbn_reduce.cuh (reduction kernels),
// cgbn_ew.cuh (finalize + elementwise kernels), cgbn_tma.cuh / cgbn_fused.cuh (opt-in
// variants), cgbn_p2p.cuh (one-shot NVLink exchange), cgbn_host.cuh (planning and
// launches); the C ABI is below.
//
// The path is HBM-bandwidth bound (no contraction; tensor cores do not apply). Each BN
// direction is a per-channel reduction followed by an elementwise pass:
//
//  * reduction kernels (statistics; backward sums) stream a channel's "stream" -- its N
//    planes of HW elements, C*HW apart in NCHW -- with 16-byte loads (4 fp32 or 8
//    bf16 / fp16 values; masked covers for odd planes), several independent loads in
//    flight per thread, an incremental address cursor, and fp64 accumulation per element.
//    Work decompositions, chosen per shape:
//      cluster-team (k_reduce_ct, NCHW default): a thread-block cluster of KC CTAs owns
//        whole channels; in each CTA a team of 2^TL threads streams its rank's share of
//        one channel, warp partials meet in shared memory and the KC CTA partials are
//        folded over DSMEM in rank order (tools/flatlab.cu measured the decomposition);
//      rows (k_reduce_rows + k_fold_rows, NHWC and (N, C)): threads own 4 adjacent
//        channels and walk rows with contiguous loads; row-block partials are folded
//        one warp per channel;
//      flat / team: fallbacks (channel counts too small for clusters to fill the GPU;
//        NHWC with C % 4 != 0).
//    The thread that completes a channel also *finishes* it: for a single-rank group
//    (G == 1) it computes mean/var/inv_std (resp. dgamma/dbeta), updates the running
//    statistics and writes the channel's affine coefficients into a table in the
//    workspace; for G > 1 it writes the rank partial that the group exchanges, and a
//    small finalize kernel folds the G partials (ascending rank order) into the same
//    table after the exchange.
//  * elementwise kernels (normalise, dx) are a memory-order grid-stride sweep over the
//    whole tensor in 16-byte units (coalesced for every layout), run from the end of the
//    tensor for L2 reuse, looking up each element's channel coefficients in the table.
//  * every kernel uses programmatic dependent launch (pdl_wait / pdl_trigger).
//
// Every reduction folds in a fixed order, so results are bitwise run-to-run
// reproducible without float atomics, and all ranks of a group compute identical
// statistics from the identical gathered partials.
//
// Reference being replaced (file:line under /root/reference/pkg/src/bigbatch):
//   channel_sum / sequential_sum_rows      tensor.py:121-153   -> reduce kernels, StatsOp
//   _train_forward finalise                batchnorm.py:121-138 -> finalize_fwd_channel
//   channel_affine (x_hat, y)              batchnorm.py:139-140, tensor.py:156-170 -> k_ew_affine
//   bn_update_running                      batchnorm.py:239-252 (in finalize_fwd_channel)
//   _backward_core sums                    batchnorm.py:198-201 -> reduce kernels, BwdOp
//   _backward_core dgamma/dbeta, dx        batchnorm.py:203-209 -> finalize_bwd_channel, k_ew_dx
//   allreduce_sum root fold                collectives.py:293-295 (ascending-rank fold in
//                                          k_finalize_* / merge_fwd_partials)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <utility>

#include "cgbn.h"
#include "cgbn_slots.cuh"

// The library is built from this file three times, once per activation dtype
// (-DCGBN_TU_ACT=0 fp32, 1 bf16, 2 fp16), so the per-dtype kernel families compile in
// parallel. Each unit exports its dtype's entry points with a suffix (cgbn_fwd_stats_a1,
// ...); unit 0 also exports the dtype-independent entry points and the public names,
// which route on the dtype bits of `layout` (include/cgbn.h).
#ifndef CGBN_TU_ACT
#define CGBN_TU_ACT 0
#endif
#define CGBN_CAT2(a, b) a##b
#define CGBN_CAT(a, b) CGBN_CAT2(a, b)
#define CGBN_FN(name) CGBN_CAT(name, CGBN_CAT(_a, CGBN_TU_ACT))

namespace {
#if CGBN_TU_ACT == 1
using TuAct = __nv_bfloat16;
#elif CGBN_TU_ACT == 2
using TuAct = __half;
#else
using TuAct = float;
#endif
}  // namespace

#define CGBN_ROUTED(act)                                                                   \
  do {                                                                                     \
    if ((act) != CGBN_TU_ACT)                                                              \
      return set_error(CGBN_ERR_INVALID, "internal: activation dtype %d routed to unit %d", \
                       (int)(act), CGBN_TU_ACT);                                           \
  } while (0)

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kTeamMaxLv = 2048;  // channels up to this many units use team kernels
constexpr int64_t kMinElemsPerCta = 2048;
constexpr int kMaxCtasPerSm = 8;  // 2048 threads / 256
// Workspace head: 65536 per-channel tickets (fixed size: independent of C), then 64
// reserved words (kept so the workspace layout and size stay those of ABI v6).
constexpr size_t kTicketWords = 65536;
constexpr size_t kTicketBytes = (kTicketWords + 64) * sizeof(unsigned);

}  // namespace

#include "cgbn_common.cuh"
#include "cgbn_ops.cuh"
#include "cgbn_reduce.cuh"
#include "cgbn_ew.cuh"
#include "cgbn_onchip.cuh"
#include "cgbn_p2p.cuh"
#include "cgbn_host.cuh"

#if CGBN_TU_ACT == 0
// The one thread-local error message behind cgbn_last_error(), shared by every unit
// (set_error forwards here; cgbn_conv.cu too).
namespace {
thread_local std::string g_last_error;
}
int cgbn_internal_set_error(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
#endif

namespace {
// A rank's partial through the on-chip kernel (statistics only) when the layer is
// on-chip eligible, so it is bitwise the partial the single-rank path reduces: the
// group-of-identical-shards invariant (test_batchnorm.py:252-262) and the bitwise match
// of every exchange transport hold. Returns 1 if launched, 0 if not eligible, < 0 error.
int onchip_stats(bool bwd, int act, bool relu, int64_t N, int64_t C, int64_t HW, int layout,
                 uintptr_t align, const void* x, const void* dy, const double* saved,
                 const float* gamma, const float* beta, double* partial,
                 const p2p::Push* push, cudaStream_t st) {
  onchip::Args oa;
  memset(&oa, 0, sizeof(oa));
  oa.x = x;
  oa.dy = dy;
  oa.partial = partial;
  if (push) oa.push = *push;
  oa.B.saved = saved;
  oa.B.gamma = gamma;
  oa.B.beta = beta;
  oa.B.relu = relu ? 1 : 0;
  oa.B.C = (uint32_t)C;
  oa.F.C = (uint32_t)C;
  return bwd ? try_onchip<true>(act, relu, N, C, HW, layout, align, oa, st)
             : try_onchip<false>(act, false, N, C, HW, layout, align, oa, st);
}
}  // namespace

// ==================================================================================
// C ABI

extern "C" {

int CGBN_FN(cgbn_fwd_stats)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   double* partial, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && partial, "cgbn_fwd_stats: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int oc = onchip_stats(false, act, false, N, C, HW, layout, (uintptr_t)x, x, nullptr,
                              nullptr, nullptr, nullptr, partial, nullptr, st);
  if (oc < 0) return -oc;
  if (oc == 0) CGBN_TRY(dispatch_stats(pl, x, true, kPartial, partial, nullptr, nullptr, w, st));
  return check_launch("cgbn_fwd_stats");
}

int CGBN_FN(cgbn_channel_sum)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                     double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && sum, "cgbn_channel_sum: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CGBN_TRY(dispatch_stats(pl, x, false, kRawSums, sum, sum_sq, nullptr, w, st));
  return check_launch("cgbn_channel_sum");
}

int CGBN_FN(cgbn_centered_sumsq)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* sum, const double* count, double* out, void* ws,
                        size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && sum && count && out, "cgbn_centered_sumsq: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CGBN_TRY(dispatch_stats(pl, x, false, kSumSq, out, nullptr, nullptr, w, st, sum, count));
  return check_launch("cgbn_centered_sumsq");
}

int CGBN_FN(cgbn_fwd_normalize_sums)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                            const double* sum, const double* sq, const double* count,
                            int centered, const float* gamma, const float* beta, double eps,
                            double momentum, float* running_mean, float* running_var,
                            double* saved, int relu, void* y, unsigned* status, void* ws,
                            size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  CGBN_REQUIRE(sum && sq && count, "cgbn_fwd_normalize_sums: NULL pointer");
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  launch_pdl(k_finalize_sums, chan_blocks(C), true, st, sum, sq, count, centered ? 1 : 0, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st, true, w.T1);
  return check_launch("cgbn_fwd_normalize_sums");
}

int CGBN_FN(cgbn_fwd_normalize)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                       const double* const* partials, int G, const float* gamma,
                       const float* beta, double eps, double momentum, float* running_mean,
                       float* running_var, double* saved, int relu, void* y, unsigned* status,
                       void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  Parts parts;
  CGBN_TRY(fill_parts(&parts, partials, G));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  launch_pdl(k_finalize_fwd, chan_blocks(C), true, st, parts, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st, true, w.T1);
  return check_launch("cgbn_fwd_normalize");
}

int CGBN_FN(cgbn_fwd_train_local)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                         const float* gamma, const float* beta, double eps, double momentum,
                         float* running_mean, float* running_var, double* saved, int relu,
                         void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  const void* eptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, eptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  // single launch with the activation held on chip when the layer fits (cgbn_onchip.cuh)
  onchip::Args oa;
  oa.trace = nullptr;
  oa.partial = nullptr;
  oa.push.G = 0;
  oa.x = x;
  oa.dy = nullptr;
  oa.out = y;
  oa.F = F;
  oa.F.P = oa.F.Q = nullptr;
  oa.F.T1 = nullptr;
  const int oc = try_onchip<false>(act, relu != 0, N, C, HW, layout,
                                   (uintptr_t)x | (uintptr_t)y, oa, st);
  if (oc < 0) return -oc;
  if (oc == 1) return check_launch("cgbn_fwd_train_local");
  CGBN_TRY(dispatch_stats(pl, x, true, kLocalFinal, nullptr, nullptr, &F, w, st));
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st, true, w.T1);
  return check_launch("cgbn_fwd_train_local");
}

int CGBN_FN(cgbn_fwd_eval)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                  const float* gamma, const float* beta, const float* running_mean,
                  const float* running_var, double eps, int relu, void* y, void* ws,
                  size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && y && gamma && beta && running_mean && running_var,
               "cgbn_fwd_eval: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_coef_eval<<<chan_blocks(C), 256, 0, st>>>(gamma, beta, running_mean, running_var, eps, w.P,
                                              w.Q, (uint32_t)C);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st);  // (fp64 tables only)
  return check_launch("cgbn_fwd_eval");
}

int CGBN_FN(cgbn_xhat)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
              const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && saved && xhat, "cgbn_xhat: NULL pointer");
  const void* ptrs[] = {x, xhat};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_coef_xhat<<<chan_blocks(C), 256, 0, st>>>(saved, w.P, w.Q, (uint32_t)C);
  launch_ew_affine(ep, false, x, xhat, w.P, w.Q, st);
  return check_launch("cgbn_xhat");
}

int CGBN_FN(cgbn_channel_affine)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* scale, const double* shift, void* out, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && scale && shift && out, "cgbn_channel_affine: NULL pointer");
  const void* ptrs[] = {x, out};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  // no PDL: the previous kernel on the stream may be the caller's producer of x
  launch_ew_affine(ep, false, x, out, scale, shift, reinterpret_cast<cudaStream_t>(stream), false);
  return check_launch("cgbn_channel_affine");
}

int CGBN_FN(cgbn_bwd_reduce)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                    int layout, const double* saved, const float* gamma, const float* beta,
                    int relu, double* partial, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && partial, "cgbn_bwd_reduce: NULL pointer");
  CGBN_REQUIRE(!relu || (gamma && beta), "cgbn_bwd_reduce: relu needs gamma and beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 2, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int oc = onchip_stats(true, act, relu != 0, N, C, HW, layout,
                              (uintptr_t)dy | (uintptr_t)x, x, dy, saved, gamma, beta, partial,
                              nullptr, st);
  if (oc < 0) return -oc;
  if (oc == 0)
    CGBN_TRY(dispatch_bwd_reduce(pl, dy, x, saved, gamma, beta, relu != 0, kPartial, partial,
                                 nullptr, w, st));
  return check_launch("cgbn_bwd_reduce");
}

int CGBN_FN(cgbn_bwd_dx)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                const double* const* partials, int G, const double* saved, const float* gamma,
                const float* beta, double eps, int relu, void* dx, float* dgamma,
                float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_dx: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_dx: relu needs beta");
  const void* ptrs[] = {dy, x, dx};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 3, &ep));
  Parts parts;
  CGBN_TRY(fill_parts(&parts, partials, G));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const BwdFinal F =
      make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  launch_pdl(k_finalize_bwd, chan_blocks(C), true, st, parts, F);
  launch_ew_dx(ep, relu != 0, dy, x, dx, w, st);
  return check_launch("cgbn_bwd_dx");
}

int CGBN_FN(cgbn_bwd_local)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                   int layout, const double* saved, const float* gamma, const float* beta,
                   double eps, int relu, void* dx, float* dgamma, float* dbeta,
                   unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_local: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_local: relu needs beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 2, &pl));
  const void* eptrs[] = {dy, x, dx};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, eptrs, 3, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const BwdFinal F =
      make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  onchip::Args oa;
  oa.trace = nullptr;
  oa.partial = nullptr;
  oa.push.G = 0;
  oa.x = x;
  oa.dy = dy;
  oa.out = dx;
  oa.B = F;
  oa.B.A = oa.B.B = oa.B.Cc = oa.B.P = oa.B.Q = nullptr;
  oa.B.T1 = nullptr;
  oa.B.T2 = nullptr;
  const int oc = try_onchip<true>(act, relu != 0, N, C, HW, layout,
                                  (uintptr_t)dy | (uintptr_t)x | (uintptr_t)dx, oa, st);
  if (oc < 0) return -oc;
  if (oc == 1) return check_launch("cgbn_bwd_local");
  CGBN_TRY(dispatch_bwd_reduce(pl, dy, x, saved, gamma, beta, relu != 0, kLocalFinal, nullptr,
                               &F, w, st));
  launch_ew_dx(ep, relu != 0, dy, x, dx, w, st);
  return check_launch("cgbn_bwd_local");
}

// Debug hook (not in include/cgbn.h): record per-CTA phase timestamps of this unit's
// on-chip launches into a device buffer of 8 u64 per CTA (NULL: off). tools/onchip_trace.py.
int CGBN_FN(cgbn_debug_onchip_trace)(void* dev_buf) {
  g_onchip_trace = static_cast<unsigned long long*>(dev_buf);
  return CGBN_OK;
}

// Whether the *_local / statistics entry points run this layer on chip by themselves.
int CGBN_FN(cgbn_onchip_selected)(int64_t N, int64_t C, int64_t HW, int layout, int backward) {
  int act = 0;
  if (split_fmt(&layout, &act)) return 0;
  return (backward ? onchip_supported<true>(act, false, N, C, HW, layout, true)
                   : onchip_supported<false>(act, false, N, C, HW, layout, true))
             ? 1
             : 0;
}

// The single-launch on-chip passes (cgbn_onchip.cuh) on request: the *_local entry points
// pick them by themselves whenever a layer fits; these force them (error if not eligible).
int CGBN_FN(cgbn_fused_supported)(int64_t N, int64_t C, int64_t HW, int layout, int backward) {
  int act = 0;
  if (split_fmt(&layout, &act)) return 0;
  return (backward ? onchip_supported<true>(act, false, N, C, HW, layout, false)
                   : onchip_supported<false>(act, false, N, C, HW, layout, false))
             ? 1
             : 0;
}

int CGBN_FN(cgbn_fwd_fused)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                            const float* gamma, const float* beta, double eps, double momentum,
                            float* running_mean, float* running_var, double* saved, int relu,
                            void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  CGBN_TRY(validate_shape(N, C, HW, layout));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  onchip::Args oa;
  oa.trace = nullptr;
  oa.partial = nullptr;
  oa.push.G = 0;
  oa.x = x;
  oa.dy = nullptr;
  oa.out = y;
  oa.F = make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  oa.F.P = oa.F.Q = nullptr;  // the coefficients stay in shared memory
  oa.F.T1 = nullptr;
  const int oc = try_onchip<false>(act, relu != 0, N, C, HW, layout,
                                   (uintptr_t)x | (uintptr_t)y, oa,
                                   reinterpret_cast<cudaStream_t>(stream), false);
  if (oc < 0) return -oc;
  if (oc == 0) return set_error(CGBN_ERR_UNSUPPORTED, "cgbn_fwd_fused: layer does not fit on chip");
  return check_launch("cgbn_fwd_fused");
}

int CGBN_FN(cgbn_bwd_fused)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                            int layout, const double* saved, const float* gamma,
                            const float* beta, double eps, int relu, void* dx, float* dgamma,
                            float* dbeta, unsigned* status, void* ws, size_t ws_bytes,
                            void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_fused: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_fused: relu needs beta");
  CGBN_TRY(validate_shape(N, C, HW, layout));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  onchip::Args oa;
  oa.trace = nullptr;
  oa.partial = nullptr;
  oa.push.G = 0;
  oa.x = x;
  oa.dy = dy;
  oa.out = dx;
  oa.B = make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  oa.B.A = oa.B.B = oa.B.Cc = oa.B.P = oa.B.Q = nullptr;
  oa.B.T1 = nullptr;
  oa.B.T2 = nullptr;
  const int oc = try_onchip<true>(act, relu != 0, N, C, HW, layout,
                                  (uintptr_t)dy | (uintptr_t)x | (uintptr_t)dx, oa,
                                  reinterpret_cast<cudaStream_t>(stream), false);
  if (oc < 0) return -oc;
  if (oc == 0) return set_error(CGBN_ERR_UNSUPPORTED, "cgbn_bwd_fused: layer does not fit on chip");
  return check_launch("cgbn_bwd_fused");
}


// ---- fused exchange (SURVEY 8(e) backend 3): the reductions' finishers push the rank's
// partial into every region and the last one publishes; the finalize kernel waits.

}  // extern "C"

namespace {
int make_push(p2p::Push* P, int rank, int G, void* const* regions, int64_t max_len,
              int64_t need, int64_t C) {
  if (G < 1 || G > p2p::kMaxPush)
    return set_error(CGBN_ERR_INVALID, "fused exchange: group size %d outside [1, %d]", G,
                     p2p::kMaxPush);
  if (rank < 0 || rank >= G) return set_error(CGBN_ERR_INVALID, "rank %d outside [0, %d)", rank, G);
  if (!regions) return set_error(CGBN_ERR_INVALID, "regions array is NULL");
  if (need > max_len)
    return set_error(CGBN_ERR_INVALID, "partial of %lld values exceeds max_len %lld",
                     (long long)need, (long long)max_len);
  for (int q = 0; q < G; ++q) {
    if (!regions[q]) return set_error(CGBN_ERR_INVALID, "regions[%d] is NULL", q);
    P->base[q] = static_cast<char*>(regions[q]);
  }
  for (int q = G; q < p2p::kMaxPush; ++q) P->base[q] = nullptr;
  P->rank = rank;
  P->G = G;
  P->max_len = max_len;
  P->nfinish = (unsigned)C;
  return CGBN_OK;
}

int make_pull(p2p::Pull* P, void* region, int G, int64_t max_len, int64_t need,
              unsigned* status, double timeout_s) {
  if (G < 1 || G > p2p::kMaxPeers)
    return set_error(CGBN_ERR_INVALID, "group size %d outside [1, %d]", G, p2p::kMaxPeers);
  if (!region) return set_error(CGBN_ERR_INVALID, "region is NULL");
  if (need > max_len)
    return set_error(CGBN_ERR_INVALID, "partial of %lld values exceeds max_len %lld",
                     (long long)need, (long long)max_len);
  if (!(timeout_s > 0.0)) return set_error(CGBN_ERR_INVALID, "timeout must be positive");
  P->own = static_cast<char*>(region);
  P->G = G;
  P->max_len = max_len;
  P->status = status;
  P->timeout_ns = (uint64_t)(timeout_s * 1e9);
  return CGBN_OK;
}

struct PushScope {  // the push applies to the reductions dispatched while it is alive
  explicit PushScope(const p2p::Push* p) { g_push = p; }
  ~PushScope() { g_push = nullptr; }
};
}  // namespace

extern "C" {

int CGBN_FN(cgbn_fwd_stats_p2p)(const void* x, int64_t N, int64_t C, int64_t HW, int layout, int rank,
                       int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes,
                       void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x, "cgbn_fwd_stats_p2p: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  p2p::Push push;
  CGBN_TRY(make_push(&push, rank, G, regions, max_len, 2 * C + 1, C));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int oc = onchip_stats(false, act, false, N, C, HW, layout, (uintptr_t)x, x, nullptr,
                              nullptr, nullptr, nullptr, nullptr, &push, st);
  if (oc < 0) return -oc;
  if (oc == 1) return check_launch("cgbn_fwd_stats_p2p");
  PushScope scope(&push);
  CGBN_TRY(dispatch_stats(pl, x, true, kPartial, nullptr, nullptr, nullptr, w, st));
  return check_launch("cgbn_fwd_stats_p2p");
}

int CGBN_FN(cgbn_fwd_normalize_p2p)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                           void* region, int G, int64_t max_len, double timeout_s,
                           const float* gamma, const float* beta, double eps, double momentum,
                           float* running_mean, float* running_var, double* saved, int relu,
                           void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  p2p::Pull pull;
  CGBN_TRY(make_pull(&pull, region, G, max_len, 2 * C + 1, status, timeout_s));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  launch_pdl(k_finalize_fwd_p2p, chan_blocks(C), true, st, pull, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st, true, w.T1);
  return check_launch("cgbn_fwd_normalize_p2p");
}

int CGBN_FN(cgbn_bwd_reduce_p2p)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                        int layout, const double* saved, const float* gamma, const float* beta,
                        int relu, int rank, int G, void* const* regions, int64_t max_len,
                        void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved, "cgbn_bwd_reduce_p2p: NULL pointer");
  CGBN_REQUIRE(!relu || (gamma && beta), "cgbn_bwd_reduce_p2p: relu needs gamma and beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 2, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  p2p::Push push;
  CGBN_TRY(make_push(&push, rank, G, regions, max_len, 2 * C, C));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int oc = onchip_stats(true, act, relu != 0, N, C, HW, layout,
                              (uintptr_t)dy | (uintptr_t)x, x, dy, saved, gamma, beta, nullptr,
                              &push, st);
  if (oc < 0) return -oc;
  if (oc == 1) return check_launch("cgbn_bwd_reduce_p2p");
  PushScope scope(&push);
  CGBN_TRY(dispatch_bwd_reduce(pl, dy, x, saved, gamma, beta, relu != 0, kPartial, nullptr,
                               nullptr, w, st));
  return check_launch("cgbn_bwd_reduce_p2p");
}

int CGBN_FN(cgbn_bwd_dx_p2p)(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                    void* region, int G, int64_t max_len, double timeout_s, const double* saved,
                    const float* gamma, const float* beta, double eps, int relu, void* dx,
                    float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes,
                    void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_dx_p2p: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_dx_p2p: relu needs beta");
  const void* ptrs[] = {dy, x, dx};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 3, &ep));
  p2p::Pull pull;
  CGBN_TRY(make_pull(&pull, region, G, max_len, 2 * C, status, timeout_s));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const BwdFinal F =
      make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  launch_pdl(k_finalize_bwd_p2p, chan_blocks(C), true, st, pull, F);
  launch_ew_dx(ep, relu != 0, dy, x, dx, w, st);
  return check_launch("cgbn_bwd_dx_p2p");
}

// ---- producer fusion, single-rank group: the conv's statistics slots -> coefficients in
// one kernel (merge + the forward finisher), then the elementwise pass.
}  // extern "C"

namespace {
__global__ void __launch_bounds__(1024) k_finalize_slots(const void* slot_ws, FwdFinal F) {
  __shared__ double sn[32][32], sa[32][32], sb[32][32];
  pdl_wait();  // the slot table comes from the conv kernel
  const cgbn_slots::Header h = *static_cast<const cgbn_slots::Header*>(slot_ws);
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double n, mean, M2;
  cgbn_slots::merge(cgbn_slots::table(slot_ws), h.cout, h.mtiles, h.grid, h.nslots, c, sn, sa,
                    sb, n, mean, M2);
  pdl_trigger();
  if ((threadIdx.x >> 5) == 0 && c < (int)F.C) {
    double P, Q;
    finalize_fwd_channel(F, (uint32_t)c, n, mean, M2, true, P, Q);
  }
}
}  // namespace

extern "C" {

int CGBN_FN(cgbn_fwd_normalize_slots)(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                             const void* slot_ws, const float* gamma, const float* beta,
                             double eps, double momentum, float* running_mean,
                             float* running_var, double* saved, int relu, void* y,
                             unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  CGBN_REQUIRE(slot_ws, "cgbn_fwd_normalize_slots: NULL slot table");
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((C + 31) / 32));
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_finalize_slots, slot_ws, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st, true, w.T1);
  return check_launch("cgbn_fwd_normalize_slots");
}


// ---- unit 0: dtype-independent entry points
#if CGBN_TU_ACT == 0

int cgbn_abi_version(void) { return CGBN_ABI_VERSION; }

#define CGBN_STR2(x) #x
#define CGBN_STR(x) CGBN_STR2(x)
const char* cgbn_build_info(void) {
  return "cgbn sm_100a; nvcc " CGBN_STR(__CUDACC_VER_MAJOR__) "." CGBN_STR(__CUDACC_VER_MINOR__)
         "; on-chip single-launch passes (cluster DSMEM, bulk copies) for layers that fit, "
         "else cluster-team / row reductions (fp64) + memory-order elementwise; PDL; fp32 / "
         "bf16 / fp16 activations";
}

const char* cgbn_last_error(void) { return g_last_error.c_str(); }

int cgbn_num_sms(void) { return num_sms_cached(); }

size_t cgbn_workspace_bytes(int64_t N, int64_t C, int64_t HW, int layout) {
  int act = 0;
  if (split_fmt(&layout, &act)) return 0;
  if (validate_shape(N, C, HW, layout)) return 0;
  return ws_bytes_for(N, C, HW, layout, num_sms_cached());
}

size_t cgbn_p2p_region_bytes(int G, int64_t max_len) {
  if (G < 1 || G > CGBN_MAX_GROUP || max_len < 1) return 0;
  return p2p::region_bytes(G, max_len);
}

int cgbn_p2p_alloc(size_t bytes, void** region, void* ipc_handle) {
  CGBN_REQUIRE(region && ipc_handle && bytes > 0, "cgbn_p2p_alloc: bad argument");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_alloc: cudaMalloc: %s", cudaGetErrorString(e));
  e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess)
    e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(ipc_handle), p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_alloc: %s", cudaGetErrorString(e));
  }
  *region = p;
  return CGBN_OK;
}

int cgbn_p2p_open(const void* ipc_handle, void** region) {
  CGBN_REQUIRE(region && ipc_handle, "cgbn_p2p_open: NULL pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(region, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_open: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

int cgbn_p2p_close(void* region) {
  const cudaError_t e = cudaIpcCloseMemHandle(region);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_close: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

int cgbn_p2p_free(void* region) {
  const cudaError_t e = cudaFree(region);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_free: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

}  // extern "C"

namespace {
int fill_peers(p2p::Peers* P, void* const* regions, int G) {
  if (G < 1 || G > p2p::kMaxPeers)
    return set_error(CGBN_ERR_INVALID, "group size %d outside [1, %d]", G, p2p::kMaxPeers);
  if (!regions) return set_error(CGBN_ERR_INVALID, "regions array is NULL");
  for (int q = 0; q < G; ++q) {
    if (!regions[q]) return set_error(CGBN_ERR_INVALID, "regions[%d] is NULL", q);
    P->base[q] = static_cast<char*>(regions[q]);
  }
  for (int q = G; q < p2p::kMaxPeers; ++q) P->base[q] = nullptr;
  return CGBN_OK;
}
}  // namespace

extern "C" {

int cgbn_p2p_exchange(const double* vec, int64_t n, int rank, int G, void* const* regions,
                      int64_t max_len, double* out, unsigned* status, double timeout_s,
                      void* stream) {
  CGBN_REQUIRE(vec && out, "cgbn_p2p_exchange: NULL pointer");
  CGBN_REQUIRE(n >= 1 && n <= max_len, "cgbn_p2p_exchange: n=%lld outside [1, %lld]",
               (long long)n, (long long)max_len);
  CGBN_REQUIRE(rank >= 0 && rank < G, "cgbn_p2p_exchange: rank %d outside [0, %d)", rank, G);
  CGBN_REQUIRE(timeout_s > 0.0, "cgbn_p2p_exchange: timeout must be positive");
  p2p::Peers peers;
  CGBN_TRY(fill_peers(&peers, regions, G));
  launch_pdl(p2p::k_p2p_exchange, 1u, true, reinterpret_cast<cudaStream_t>(stream), vec, n, rank,
             G, peers, max_len, out, status, (uint64_t)(timeout_s * 1e9));
  return check_launch("cgbn_p2p_exchange");
}

int cgbn_p2p_emulate(const double* vecs, int64_t n, int G, void* const* regions, int64_t max_len,
                     double* outs, unsigned* status, double timeout_s, int skip, void* stream) {
  CGBN_REQUIRE(vecs && outs, "cgbn_p2p_emulate: NULL pointer");
  CGBN_REQUIRE(n >= 1 && n <= max_len, "cgbn_p2p_emulate: n outside [1, max_len]");
  CGBN_REQUIRE(timeout_s > 0.0, "cgbn_p2p_emulate: timeout must be positive");
  p2p::Peers peers;
  CGBN_TRY(fill_peers(&peers, regions, G));
  // cooperative launch: the G rank-CTAs are guaranteed co-resident while they wait on
  // each other (the single-GPU stand-in for G processes)
  const uint64_t tns = (uint64_t)(timeout_s * 1e9);
  void* args[] = {(void*)&vecs, (void*)&n,      (void*)&G,      (void*)&peers, (void*)&max_len,
                  (void*)&outs, (void*)&status, (void*)&tns,    (void*)&skip};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)p2p::k_p2p_emulate, dim3(G),
                                                    dim3(p2p::kThreadsP2P), args, 0,
                                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_emulate: %s", cudaGetErrorString(e));
  return check_launch("cgbn_p2p_emulate");
}

int cgbn_fold_sum(const void* const* vectors, int G, int64_t n, int dtype, void* out,
                  void* stream) {
  CGBN_REQUIRE(vectors && out, "cgbn_fold_sum: NULL pointer");
  CGBN_REQUIRE(n >= 1, "cgbn_fold_sum: n must be >= 1");
  CGBN_REQUIRE(dtype == CGBN_DTYPE_F32 || dtype == CGBN_DTYPE_F64, "unknown dtype %d", dtype);
  Parts P;
  CGBN_TRY(fill_parts(&P, reinterpret_cast<const double* const*>(vectors), G));
  const int threads = 256;
  int64_t blocks = ceil_div(n, threads);
  if (blocks > (int64_t)num_sms_cached() * 8) blocks = (int64_t)num_sms_cached() * 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == CGBN_DTYPE_F64)
    k_fold_sum<double><<<(unsigned)blocks, threads, 0, st>>>(P, n, reinterpret_cast<double*>(out));
  else
    k_fold_sum<float><<<(unsigned)blocks, threads, 0, st>>>(P, n, reinterpret_cast<float*>(out));
  return check_launch("cgbn_fold_sum");
}


// Public names: route on the activation dtype in bits 4..7 of `layout` (an unknown
// dtype goes to unit 0, which reports it).
int cgbn_fwd_stats_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* partial, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_stats_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* partial, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_stats(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* partial, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_stats_a1(x, N, C, HW, layout, partial, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_stats_a2(x, N, C, HW, layout, partial, ws, ws_bytes, stream);
    default: return cgbn_fwd_stats_a0(x, N, C, HW, layout, partial, ws, ws_bytes, stream);
  }
}

int cgbn_channel_sum_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream);
int cgbn_channel_sum_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream);
int cgbn_channel_sum(const void* x, int64_t N, int64_t C, int64_t HW, int layout, double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_channel_sum_a1(x, N, C, HW, layout, sum, sum_sq, ws, ws_bytes, stream);
    case 2: return cgbn_channel_sum_a2(x, N, C, HW, layout, sum, sum_sq, ws, ws_bytes, stream);
    default: return cgbn_channel_sum_a0(x, N, C, HW, layout, sum, sum_sq, ws, ws_bytes, stream);
  }
}

int cgbn_centered_sumsq_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* count, double* out, void* ws, size_t ws_bytes, void* stream);
int cgbn_centered_sumsq_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* count, double* out, void* ws, size_t ws_bytes, void* stream);
int cgbn_centered_sumsq(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* count, double* out, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_centered_sumsq_a1(x, N, C, HW, layout, sum, count, out, ws, ws_bytes, stream);
    case 2: return cgbn_centered_sumsq_a2(x, N, C, HW, layout, sum, count, out, ws, ws_bytes, stream);
    default: return cgbn_centered_sumsq_a0(x, N, C, HW, layout, sum, count, out, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_normalize_sums_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* sq, const double* count, int centered, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_sums_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* sq, const double* count, int centered, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_sums(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* sum, const double* sq, const double* count, int centered, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_normalize_sums_a1(x, N, C, HW, layout, sum, sq, count, centered, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_normalize_sums_a2(x, N, C, HW, layout, sum, sq, count, centered, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_normalize_sums_a0(x, N, C, HW, layout, sum, sq, count, centered, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_normalize_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_normalize_a1(x, N, C, HW, layout, partials, G, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_normalize_a2(x, N, C, HW, layout, partials, G, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_normalize_a0(x, N, C, HW, layout, partials, G, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_train_local_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_train_local_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_train_local(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_train_local_a1(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_train_local_a2(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_train_local_a0(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_eval_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, const float* running_mean, const float* running_var, double eps, int relu, void* y, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_eval_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, const float* running_mean, const float* running_var, double eps, int relu, void* y, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_eval(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, const float* running_mean, const float* running_var, double eps, int relu, void* y, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_eval_a1(x, N, C, HW, layout, gamma, beta, running_mean, running_var, eps, relu, y, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_eval_a2(x, N, C, HW, layout, gamma, beta, running_mean, running_var, eps, relu, y, ws, ws_bytes, stream);
    default: return cgbn_fwd_eval_a0(x, N, C, HW, layout, gamma, beta, running_mean, running_var, eps, relu, y, ws, ws_bytes, stream);
  }
}

int cgbn_xhat_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream);
int cgbn_xhat_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream);
int cgbn_xhat(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_xhat_a1(x, N, C, HW, layout, saved, xhat, ws, ws_bytes, stream);
    case 2: return cgbn_xhat_a2(x, N, C, HW, layout, saved, xhat, ws, ws_bytes, stream);
    default: return cgbn_xhat_a0(x, N, C, HW, layout, saved, xhat, ws, ws_bytes, stream);
  }
}

int cgbn_channel_affine_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* scale, const double* shift, void* out, void* stream);
int cgbn_channel_affine_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* scale, const double* shift, void* out, void* stream);
int cgbn_channel_affine(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* scale, const double* shift, void* out, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_channel_affine_a1(x, N, C, HW, layout, scale, shift, out, stream);
    case 2: return cgbn_channel_affine_a2(x, N, C, HW, layout, scale, shift, out, stream);
    default: return cgbn_channel_affine_a0(x, N, C, HW, layout, scale, shift, out, stream);
  }
}

int cgbn_bwd_reduce_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, double* partial, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_reduce_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, double* partial, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_reduce(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, double* partial, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_reduce_a1(dy, x, N, C, HW, layout, saved, gamma, beta, relu, partial, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_reduce_a2(dy, x, N, C, HW, layout, saved, gamma, beta, relu, partial, ws, ws_bytes, stream);
    default: return cgbn_bwd_reduce_a0(dy, x, N, C, HW, layout, saved, gamma, beta, relu, partial, ws, ws_bytes, stream);
  }
}

int cgbn_bwd_dx_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_dx_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_dx(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* const* partials, int G, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_dx_a1(dy, x, N, C, HW, layout, partials, G, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_dx_a2(dy, x, N, C, HW, layout, partials, G, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    default: return cgbn_bwd_dx_a0(dy, x, N, C, HW, layout, partials, G, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
  }
}

int cgbn_bwd_local_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_local_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_local(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_local_a1(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_local_a2(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    default: return cgbn_bwd_local_a0(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
  }
}

int cgbn_onchip_selected_a1(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_onchip_selected_a2(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_onchip_selected(int64_t N, int64_t C, int64_t HW, int layout, int backward) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_onchip_selected_a1(N, C, HW, layout, backward);
    case 2: return cgbn_onchip_selected_a2(N, C, HW, layout, backward);
    default: return cgbn_onchip_selected_a0(N, C, HW, layout, backward);
  }
}

int cgbn_fused_supported_a1(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_fused_supported_a2(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_fused_supported(int64_t N, int64_t C, int64_t HW, int layout, int backward) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fused_supported_a1(N, C, HW, layout, backward);
    case 2: return cgbn_fused_supported_a2(N, C, HW, layout, backward);
    default: return cgbn_fused_supported_a0(N, C, HW, layout, backward);
  }
}

int cgbn_fwd_fused_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_fused_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_fused(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_fused_a1(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_fused_a2(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_fused_a0(x, N, C, HW, layout, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

int cgbn_bwd_fused_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_fused_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_fused(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_fused_a1(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_fused_a2(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    default: return cgbn_bwd_fused_a0(dy, x, N, C, HW, layout, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_stats_p2p_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_stats_p2p_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_stats_p2p(const void* x, int64_t N, int64_t C, int64_t HW, int layout, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_stats_p2p_a1(x, N, C, HW, layout, rank, G, regions, max_len, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_stats_p2p_a2(x, N, C, HW, layout, rank, G, regions, max_len, ws, ws_bytes, stream);
    default: return cgbn_fwd_stats_p2p_a0(x, N, C, HW, layout, rank, G, regions, max_len, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_normalize_p2p_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_p2p_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_p2p(const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_normalize_p2p_a1(x, N, C, HW, layout, region, G, max_len, timeout_s, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_normalize_p2p_a2(x, N, C, HW, layout, region, G, max_len, timeout_s, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_normalize_p2p_a0(x, N, C, HW, layout, region, G, max_len, timeout_s, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

int cgbn_bwd_reduce_p2p_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_reduce_p2p_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_reduce_p2p(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, const double* saved, const float* gamma, const float* beta, int relu, int rank, int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_reduce_p2p_a1(dy, x, N, C, HW, layout, saved, gamma, beta, relu, rank, G, regions, max_len, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_reduce_p2p_a2(dy, x, N, C, HW, layout, saved, gamma, beta, relu, rank, G, regions, max_len, ws, ws_bytes, stream);
    default: return cgbn_bwd_reduce_p2p_a0(dy, x, N, C, HW, layout, saved, gamma, beta, relu, rank, G, regions, max_len, ws, ws_bytes, stream);
  }
}

int cgbn_bwd_dx_p2p_a1(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_dx_p2p_a2(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_dx_p2p(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout, void* region, int G, int64_t max_len, double timeout_s, const double* saved, const float* gamma, const float* beta, double eps, int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_bwd_dx_p2p_a1(dy, x, N, C, HW, layout, region, G, max_len, timeout_s, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    case 2: return cgbn_bwd_dx_p2p_a2(dy, x, N, C, HW, layout, region, G, max_len, timeout_s, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
    default: return cgbn_bwd_dx_p2p_a0(dy, x, N, C, HW, layout, region, G, max_len, timeout_s, saved, gamma, beta, eps, relu, dx, dgamma, dbeta, status, ws, ws_bytes, stream);
  }
}

int cgbn_fwd_normalize_slots_a1(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const void* slot_ws, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_slots_a2(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const void* slot_ws, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_fwd_normalize_slots(const void* x, int64_t N, int64_t C, int64_t HW, int layout, const void* slot_ws, const float* gamma, const float* beta, double eps, double momentum, float* running_mean, float* running_var, double* saved, int relu, void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  switch ((layout >> 4) & 0xF) {
    case 1: return cgbn_fwd_normalize_slots_a1(x, N, C, HW, layout, slot_ws, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    case 2: return cgbn_fwd_normalize_slots_a2(x, N, C, HW, layout, slot_ws, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
    default: return cgbn_fwd_normalize_slots_a0(x, N, C, HW, layout, slot_ws, gamma, beta, eps, momentum, running_mean, running_var, saved, relu, y, status, ws, ws_bytes, stream);
  }
}

#endif  // CGBN_TU_ACT == 0

}  // extern "C"
