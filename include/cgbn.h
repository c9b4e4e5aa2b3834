/*
 * cgbn.h — C ABI of the B200-native Cross-GPU Batch Normalization (CGBN) hot path.
 *
 * This is the drop-in boundary for the reference's CGBN operator
 * (`bigbatch.batchnorm`, /root/reference/pkg/src/bigbatch/batchnorm.py). The reference
 * has no native code: its hot path is NumPy (channel_sum / channel_affine in tensor.py)
 * glued by the `reduce_vec` seam that is bound to `allreduce_sum` over the BN sub-group
 * (batchnorm.py:115-144, 169-185, 188-236). Every entry point below replaces one piece
 * of that path; the per-function comment names the reference lines it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types. All device pointers are CUDA device
 *    memory on the device current to the calling thread. `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream). Every call is asynchronous
 *    (stream-ordered) and performs no allocation and no host synchronisation.
 *  - Activations are contiguous fp32 (the reference's f32 path), bf16 or fp16; statistics,
 *    coefficients and every reduction are fp64, outputs are rounded once to the
 *    activation type. `layout` is CGBN_LAYOUT_NCHW (x[N][C][HW]; a 2-D (N, C) tensor is
 *    NCHW with HW == 1) or CGBN_LAYOUT_NHWC (x[N][HW][C]), OR'd with the activation
 *    dtype CGBN_ACT_F32 (0, default) / CGBN_ACT_BF16 / CGBN_ACT_F16. gamma, beta and the
 *    running statistics stay fp32 for every activation dtype.
 *  - Statistics travel between kernels and ranks as fp64 "partials":
 *      forward  partial (2C+1 doubles): [mean_r (C) | M2_r (C) | count_r (1)]
 *      backward partial (2C   doubles): [sum dy (C) | sum dy*(x-mean) (C)]
 *    The forward partial is the reference's packed [sum, sum_sq, m] vector
 *    (batchnorm.py:120) re-expressed as (mean, centred M2, count) so that the merge is
 *    cancellation-free; the backward partial is the reference's [sum dy, sum dy*x_hat]
 *    (batchnorm.py:198-202) with the 1/std factor applied after the reduction.
 *  - A group of G ranks exchanges partials (NCCL all-gather, the host rendezvous of the
 *    threaded DeviceGroup, or the one-shot P2P path) and each consumer kernel folds the
 *    G partials in ascending rank order, exactly like the reference's star all-reduce
 *    (collectives.py:293-295); every rank therefore computes bitwise-identical
 *    statistics.
 *  - Return value: 0 (CGBN_OK) or a CGBN_ERR_* code; cgbn_last_error() returns a
 *    thread-local message for the last failing call. Data-dependent errors found on the
 *    device (non-finite statistics, total count < 2) are OR-ed into the caller-provided
 *    device status word (CGBN_STATUS_* bits) and checked by the host at sync points.
 */
#ifndef CGBN_H_
#define CGBN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGBN_ABI_VERSION 7

#define CGBN_LAYOUT_NCHW 0
#define CGBN_LAYOUT_NHWC 1

/* Activation dtype, OR'd into `layout` (bf16 / fp16 activations with
 * fp32 parameters and fp64 statistics). */
#define CGBN_ACT_F32 0x00
#define CGBN_ACT_BF16 0x10
#define CGBN_ACT_F16 0x20

#define CGBN_MAX_GROUP 64

#define CGBN_OK 0
#define CGBN_ERR_INVALID 1 /* bad argument (shape, alignment, group size, ws too small) */
#define CGBN_ERR_CUDA 2    /* CUDA launch / runtime error */
#define CGBN_ERR_UNSUPPORTED 3 /* fused entry point: shape/layout not eligible (use split) */

#define CGBN_STATUS_NONFINITE 1u  /* NaN/Inf reached the statistics (tensor.py:59-60) */
#define CGBN_STATUS_SMALL_COUNT 2u /* total count < 2 (batchnorm.py:133-137) */
#define CGBN_STATUS_EXCHANGE_TIMEOUT 4u /* a P2P exchange peer did not arrive in time */

#define CGBN_DTYPE_F32 0
#define CGBN_DTYPE_F64 1

/* ABI version (CGBN_ABI_VERSION) and build info. */
int cgbn_abi_version(void);
const char* cgbn_build_info(void);

/* Thread-local message describing the last non-zero return of any cgbn_* call. */
const char* cgbn_last_error(void);

/* Number of SMs of the current device (cached per device). */
int cgbn_num_sms(void);

/* Bytes of zero-initialised workspace every kernel entry point below needs for this
 * shape (depends on C only). It holds per-channel arrival tickets, per-CTA partial
 * slots and the per-channel coefficient table that connects a reduction to the
 * elementwise pass that follows it; the kernels leave the tickets at zero on exit, so
 * one zeroed buffer per stream can be reused by every later call on that stream
 * (calls on one stream are ordered; concurrent streams need separate workspaces). */
size_t cgbn_workspace_bytes(int64_t N, int64_t C, int64_t HW, int layout);

/* Forward, step 1: this rank's per-channel partial statistics.
 * Replaces channel_sum(x, with_sum_sq) (tensor.py:143-153; the _channels_last_rows +
 * sequential_sum_rows pair, tensor.py:121-140) as called from _train_forward
 * (batchnorm.py:118) — one read of x, deterministic fixed-order cross-CTA fold.
 * Writes `partial` (2C+1 doubles). */
int cgbn_fwd_stats(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   double* partial, void* ws, size_t ws_bytes, void* stream);

/* Forward, step 2 (G ranks): fold the G gathered partials (ascending rank order),
 * finalise mean/var/inv_std, update the running statistics in place, and write
 * y = gamma * (x - mean) * inv_std + beta (optionally ReLU'd). Two launches: a per-channel
 * finalize kernel that writes the coefficient table into `ws`, then a memory-order
 * elementwise pass over the whole tensor.
 * Replaces _train_forward's post-reduction half (batchnorm.py:121-143): mu/var
 * (:122-124, :128-132), the m < 2 check (:133-137), inv_std (:138), the two
 * channel_affine calls (:139-140, tensor.py:156-170) and bn_update_running
 * (batchnorm.py:239-252).
 *  partials : host array of G device pointers, partials[r] = rank r's forward partial.
 *  saved    : out, 3C+1 doubles [mean (C) | var (C) | inv_std (C) | total_count (1)];
 *             the backward reads it (it replaces BNForwardCache.mu/var/total_count —
 *             x_hat is recomputed from x instead of being stored, batchnorm.py:142).
 *  running_mean/var may be NULL (no update). momentum in [0, 1]. */
int cgbn_fwd_normalize(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                       const double* const* partials, int G,
                       const float* gamma, const float* beta, double eps, double momentum,
                       float* running_mean, float* running_var, double* saved, int relu,
                       void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);

/* Single-rank training forward (G == 1: bn_forward_local, batchnorm.py:147-157, or a BN
 * group of one): the statistics kernel's last CTA per channel finalises the channel
 * directly (no partial, no exchange), then the elementwise pass. Two launches. Same
 * outputs and contract as cgbn_fwd_stats + cgbn_fwd_normalize with G == 1. */
int cgbn_fwd_train_local(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                         const float* gamma, const float* beta, double eps, double momentum,
                         float* running_mean, float* running_var, double* saved, int relu,
                         void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);

/* Eval-mode forward: y = gamma * (x - running_mean) / sqrt(running_var + eps) + beta.
 * Replaces bn_forward_local(mode="eval") (batchnorm.py:158-166); no collective and the
 * running statistics are left untouched. */
int cgbn_fwd_eval(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                  const float* gamma, const float* beta, const float* running_mean,
                  const float* running_var, double eps, int relu, void* y, void* ws,
                  size_t ws_bytes, void* stream);

/* Backward, step 1: this rank's partial [sum g, sum g*(x-mean)] with g = dy (times the
 * ReLU mask recomputed from x when relu != 0). Replaces the two sequential_sum_rows
 * calls of _backward_core (batchnorm.py:198-201). Writes `partial` (2C doubles). */
int cgbn_bwd_reduce(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                    int layout, const double* saved, const float* gamma, const float* beta,
                    int relu, double* partial, void* ws, size_t ws_bytes, void* stream);

/* Backward, step 2 (G ranks): fold the G gathered backward partials (ascending rank
 * order) into the BN-group sums dbeta = sum g, dgamma = sum g*x_hat (identical on every
 * rank, as in batchnorm.py:203) and write dx = gamma/sqrt(var+eps)*(g - dbeta/m -
 * x_hat*dgamma/m) (batchnorm.py:204-209). As in the reference, `eps` is the backward
 * state's eps while x_hat keeps the forward's normalisation. dgamma/dbeta (C floats
 * each) may be NULL. Two launches (finalize, memory-order elementwise). */
int cgbn_bwd_dx(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                const double* const* partials, int G, const double* saved,
                const float* gamma, const float* beta, double eps, int relu, void* dx,
                float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes,
                void* stream);

/* Single-rank backward (G == 1: bn_backward_local, batchnorm.py:213-218, or a BN group
 * of one): reduce kernel that finalises each channel, then the elementwise dx pass.
 * Same outputs as cgbn_bwd_reduce + cgbn_bwd_dx with G == 1. */
int cgbn_bwd_local(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                   int layout, const double* saved, const float* gamma, const float* beta,
                   double eps, int relu, void* dx, float* dgamma, float* dbeta,
                   unsigned* status, void* ws, size_t ws_bytes, void* stream);

/* x_hat = (x - mean) * inv_std from a saved forward context (the reference caches
 * x_hat in BNForwardCache, batchnorm.py:142; here it is recomputed on demand). */
int cgbn_xhat(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
              const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream);

/* One-shot P2P exchange of the statistics partial over NVLink / NVSwitch (
 * the alternative to the NCCL all-gather; replaces the star gather of
 * collectives.py:224-252). Each rank of a BN group allocates one region of
 * cgbn_p2p_region_bytes(G, max_len) bytes (cgbn_p2p_alloc, zeroed; returns the
 * 64-byte CUDA IPC handle), shares the handles, and opens its peers' regions
 * (cgbn_p2p_open). cgbn_p2p_exchange is one single-CTA kernel: it pushes `vec` (n <=
 * max_len doubles) into every region, publishes an epoch flag (release, system scope),
 * waits for every peer's flag (acquire; after timeout_s it sets
 * CGBN_STATUS_EXCHANGE_TIMEOUT and continues instead of hanging) and writes the G rows
 * in rank order to out[G * n]. Every rank of the group must issue the same sequence of
 * exchanges. regions[q] is rank q's region as mapped in this process.
 *
 * cgbn_p2p_emulate runs the same per-rank routine as a cooperative launch of G CTAs on
 * one GPU (CTA b = rank b, regions all local): the protocol check used by the tests.
 * skip >= 0 makes that rank sit the exchange out. */
size_t cgbn_p2p_region_bytes(int G, int64_t max_len);
int cgbn_p2p_alloc(size_t bytes, void** region, void* ipc_handle);
int cgbn_p2p_open(const void* ipc_handle, void** region);
int cgbn_p2p_close(void* region);
int cgbn_p2p_free(void* region);
int cgbn_p2p_exchange(const double* vec, int64_t n, int rank, int G, void* const* regions,
                      int64_t max_len, double* out, unsigned* status, double timeout_s,
                      void* stream);
int cgbn_p2p_emulate(const double* vecs, int64_t n, int G, void* const* regions, int64_t max_len,
                     double* outs, unsigned* status, double timeout_s, int skip, void* stream);

/* The P2P exchange fused into the kernels on either side of it (SURVEY 8(e) backend 3:
 * "the same fused into the K1/K4a tail"); no exchange kernel of its own. Same regions and
 * protocol as cgbn_p2p_exchange (the region layout carries a finisher counter for this):
 *  - cgbn_fwd_stats_p2p / cgbn_bwd_reduce_p2p: the statistics reduction whose channel
 *    finishers write the rank's partial straight into row `rank` of every region of the
 *    group (the epoch parity comes from the own region's counter); the last finisher
 *    advances the epoch and publishes the rank's flag in every region (release, system
 *    scope). Replaces cgbn_fwd_stats / cgbn_bwd_reduce + cgbn_p2p_exchange.
 *  - cgbn_fwd_normalize_p2p / cgbn_bwd_dx_p2p: the finalize kernel first waits for every
 *    rank's flag of the current epoch in the own region (acquire; timeout_s ->
 *    CGBN_STATUS_EXCHANGE_TIMEOUT in *status), folds the G rows read there in ascending
 *    rank order, then the elementwise pass. Same outputs as cgbn_fwd_normalize /
 *    cgbn_bwd_dx on the gathered partials (bitwise).
 * G <= 8 (one NVSwitch box) for the fused variant. */
int cgbn_fwd_stats_p2p(const void* x, int64_t N, int64_t C, int64_t HW, int layout, int rank,
                       int G, void* const* regions, int64_t max_len, void* ws, size_t ws_bytes,
                       void* stream);
int cgbn_fwd_normalize_p2p(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                           void* region, int G, int64_t max_len, double timeout_s,
                           const float* gamma, const float* beta, double eps, double momentum,
                           float* running_mean, float* running_var, double* saved, int relu,
                           void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_reduce_p2p(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                        int layout, const double* saved, const float* gamma, const float* beta,
                        int relu, int rank, int G, void* const* regions, int64_t max_len,
                        void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_dx_p2p(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                    void* region, int G, int64_t max_len, double timeout_s, const double* saved,
                    const float* gamma, const float* beta, double eps, int relu, void* dx,
                    float* dgamma, float* dbeta, unsigned* status, void* ws, size_t ws_bytes,
                    void* stream);

/* Ascending-rank fold of G device vectors of n elements (dtype CGBN_DTYPE_F32/F64):
 * out = v[0] + v[1] + ... + v[G-1], evaluated left to right. This is the arithmetic of
 * the reference's allreduce_sum at the root (collectives.py:293-295); the transport
 * (gathering the G vectors) is done by the caller. */
int cgbn_fold_sum(const void* const* vectors, int G, int64_t n, int dtype, void* out,
                  void* stream);

/* Per-channel sums of an activation (sum and optional sum of squares, fp64 out).
 * Device counterpart of the reference's channel_sum (tensor.py:143-153). sum_sq may be
 * NULL. ws as for cgbn_fwd_stats. */
int cgbn_channel_sum(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                     double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream);

/* Reference-literal forward statistics (bigbatch's own algorithm, selected with
 * set_forward_exchange("reference")). Two-pass (the reference
 * default, batchnorm.py:125-132): cgbn_channel_sum -> exchange [sum | m] ->
 * cgbn_centered_sumsq -> exchange -> cgbn_fwd_normalize_sums(centered = 1). One-pass
 * (batchnorm.py:119-124): cgbn_channel_sum with sum_sq -> exchange [sum | sum_sq | m] ->
 * cgbn_fwd_normalize_sums(centered = 0).
 *
 * cgbn_centered_sumsq: out[c] = sum over this rank's elements of (x - mean_c)^2 in fp64,
 * with mean_c = sum[c] / count[0] from the group-folded first exchange
 * (batchnorm.py:128-129). */
int cgbn_centered_sumsq(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* sum, const double* count, double* out, void* ws,
                        size_t ws_bytes, void* stream);

/* Normalise from group sums: mean = sum[c] / m, var = sq[c] / m (centered != 0) or
 * max(sq[c] / m - mean^2, 0) (centered == 0), m = count[0]; then what
 * cgbn_fwd_normalize does after its fold (batchnorm.py:121-124, 131-141). */
int cgbn_fwd_normalize_sums(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                            const double* sum, const double* sq, const double* count,
                            int centered, const float* gamma, const float* beta, double eps,
                            double momentum, float* running_mean, float* running_var,
                            double* saved, int relu, void* y, unsigned* status, void* ws,
                            size_t ws_bytes, void* stream);

/* Per-channel affine map out = scale[c] * x + shift[c] (fp64 coefficients, device
 * arrays of C doubles). Device counterpart of the reference's channel_affine
 * (tensor.py:156-170). */
int cgbn_channel_affine(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* scale, const double* shift, void* out, void* stream);

/* Single-launch on-chip forward / backward for a single-rank group (G == 1:
 * bn_forward_local / bn_backward_local, or a BN group of one). One kernel per direction
 * (cgbn_onchip.cuh): a thread-block cluster owns whole channels; its CTAs bulk-copy
 * (cp.async.bulk) their image runs of those channels into shared memory, reduce them,
 * fold the CTA partials over DSMEM and write the elementwise result from shared memory,
 * so x (and dy) cross HBM once (forward 8 B/elem instead of 12, backward 12 instead of
 * 20) with no grid barrier. Same outputs and contracts as cgbn_fwd_stats +
 * cgbn_fwd_normalize (resp. cgbn_bwd_reduce + cgbn_bwd_dx) with G == 1; NCHW, any
 * activation dtype.
 * cgbn_fwd_train_local / cgbn_bwd_local (and cgbn_fwd_stats / cgbn_bwd_reduce, in a
 * statistics-only mode) choose this kernel by themselves for layers below a footprint
 * cap measured in-step (cgbn_onchip_selected() reports that choice); cgbn_*_fused force
 * it for any layer that fits in one resident wave and return CGBN_ERR_UNSUPPORTED
 * otherwise, which cgbn_fused_supported() answers without launching (backward != 0:
 * the backward variant). */
int cgbn_onchip_selected(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_fused_supported(int64_t N, int64_t C, int64_t HW, int layout, int backward);
int cgbn_fwd_fused(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   const float* gamma, const float* beta, double eps, double momentum,
                   float* running_mean, float* running_var, double* saved, int relu, void* y,
                   unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_bwd_fused(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   const double* saved, const float* gamma, const float* beta, double eps,
                   int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws,
                   size_t ws_bytes, void* stream);

/* Producer fusion (ABI v7). The layer that feeds a BN in the
 * reference model is a GEMM-shaped convolution (model.py:235-242, out = cols @ W^T + b)
 * whose output _train_forward immediately re-reads for its statistics (batchnorm.py:118,
 * channel_sum, tensor.py:143-153). cgbn_conv1x1_stats computes the pointwise (1x1) case
 *     z[n][co][p] = sum_ci w[co][ci] * x[n][ci][p] + bias[co]          (NCHW, p = h*W + w)
 * on the tcgen05 tensor cores (bf16 x and w, fp32 accumulation, z stored as fp32 or bf16
 * per out_dtype = CGBN_ACT_F32 / CGBN_ACT_BF16) and, in the same kernel's epilogue, this
 * rank's forward partial of z as stored (2C+1 doubles, [mean | M2 | count], C = Cout) —
 * the vector cgbn_fwd_stats(z) would produce, so the exchange and cgbn_fwd_normalize
 * follow unchanged and the BN forward no longer reads z for its statistics.
 *  bias     : Cout floats or NULL.
 *  ws       : cgbn_conv1x1_ws_bytes(N, Cin, Cout, HW) bytes, 16-byte aligned: the per-CTA
 *             statistics slot table and the split-K partials; the LAST 16 KB of the
 *             ws_bytes passed are the split-K tickets (ABI v7), which must be zero before
 *             the first call on a buffer (allocate it zero-filled) and are left zero by
 *             every call, so one buffer serves layers of any shape.
 *  partial  : may be NULL: the fold is skipped and the slot table stays in ws for
 *             cgbn_fwd_normalize_slots (below).
 * Two launches (the conv, then a per-channel fold of the tile partials). Returns
 * CGBN_ERR_UNSUPPORTED when H*W or Cin is not a multiple of 8 (TMA row strides).
 * cgbn_conv1x1 is the same convolution without the statistics (the unfused producer); its
 * ws (same size and contract) may be NULL, which only forgoes split-K.
 * Split-K: layers with fewer 128-pixel tiles than SMs cut each tile's k-steps into up to 4
 * ranges on as many CTAs; the last range's CTA adds the others' fp32 partials in range
 * order (deterministic) before the epilogue. */
size_t cgbn_conv1x1_ws_bytes(int64_t N, int64_t Cin, int64_t Cout, int64_t HW);
/* Single-rank groups (bn_forward_local, or a BN group of one): call the *_stats entry
 * point with partial = NULL, which leaves the statistics slot table in ws (a 32-byte
 * header written by the conv kernel, then the per-CTA slots), and pass that ws here as
 * slot_ws: one kernel merges the slots straight into the coefficients (no partial, no
 * fold launch), then the elementwise pass — the same outputs and contract as
 * cgbn_fwd_normalize with G == 1. */
int cgbn_fwd_normalize_slots(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                             const void* slot_ws, const float* gamma, const float* beta,
                             double eps, double momentum, float* running_mean,
                             float* running_var, double* saved, int relu, void* y,
                             unsigned* status, void* ws, size_t ws_bytes, void* stream);
int cgbn_conv1x1(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                 int64_t Cout, int64_t HW, int out_dtype, void* z, void* ws, size_t ws_bytes,
                 void* stream);
int cgbn_conv1x1_stats(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                       int64_t Cout, int64_t HW, int out_dtype, void* z, double* partial,
                       void* ws, size_t ws_bytes, void* stream);

/* The producer on channels-last activations (x, z NHWC = [N][H][W][C], the layout
 * detector training uses and the BN's native NHWC kernels read): ksize 1 or 3 (zero
 * padding 1 for 3x3 — the reference model's conv layer, model.py:235-242), stride 1 or
 * 2, any H and W; z is [N][Ho][Wo][Cout] with Ho = (H + 2 pad - ksize) / stride + 1. The
 * 3x3 and strided cases are an implicit GEMM on TMA im2col loads (taps x Cin/64 k-steps;
 * the hardware walks the output pixels, shifts each window by the tap and zero-fills
 * outside the image). w: bf16 [Cout][Cin] (ksize 1) or [Cout][9][Cin] with tap =
 * 3 * ky + kx (OHWI: torch's channels_last (Cout, Cin, 3, 3) weight as it lies in memory;
 * ABI v7 — v6 took [9][Cout][Cin]). Cin and Cout must be
 * multiples of 8. Statistics contract as cgbn_conv1x1_stats; ws: cgbn_conv_nhwc_ws_bytes
 * bytes. */
size_t cgbn_conv_nhwc_ws_bytes(int64_t N, int64_t Cin, int64_t Cout, int64_t H, int64_t W,
                               int ksize, int stride);
int cgbn_conv_nhwc(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                   int64_t Cout, int64_t H, int64_t W, int ksize, int stride, int out_dtype,
                   void* z, void* ws, size_t ws_bytes, void* stream);
int cgbn_conv_nhwc_stats(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                         int64_t Cout, int64_t H, int64_t W, int ksize, int stride, int out_dtype,
                         void* z, double* partial, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CGBN_H_ */
