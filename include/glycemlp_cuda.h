/*
 * glycemlp_cuda.h -- C ABI of libglycemlp_cuda.so, the B200 (sm_100a)
 * replacement for the glycemlp training hot path.
 *
 * Reference boundary (all paths relative to /root/reference/pkg/src/glycemlp):
 *   backend.run_train_segment(w_ih2d, w_ho2d, feats2d, targets, epochs, lr, kind)
 *                                                         backend.py:208-234
 *   kernels.train_segment_seq / train_segment_par        kernels.py:264-349
 *   kernels.eval_counts(w_ih2d, w_ho2d, feats2d, labels) kernels.py:352-375
 *   trainer._confusion                                    trainer.py:94-97
 *
 * Conventions
 *   - Weight layout is the reference's (network.py:84-90): w_ih is
 *     hidden x (input+1) row-major with the bias in the trailing slot, w_ho is
 *     outputs x (hidden+1). Both are float32 and updated IN PLACE.
 *   - Return 0 on success, a negative GLX_ERR_* code otherwise; the message
 *     is in glx_last_error() (thread-local). Codes map onto the reference's
 *     exception types (errors.py:16-25).
 *   - "host" entry points take host pointers, copy in, run, copy out and
 *     synchronise (the reference's synchronous in-place contract).
 *   - "device" entry points take device pointers owned by the caller and a
 *     cudaStream_t (NULL = legacy default stream); they are asynchronous.
 *   - numerics: GLX_FP32 (packed-FP32 FMA, fast sigmoid; within 1e-4
 *     max(1,|w|)-relative of the reference) or GLX_REF64 (the reference's
 *     f64 op order, f32 stores).
 */
#ifndef GLYCEMLP_CUDA_H
#define GLYCEMLP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLX_OK 0
#define GLX_ERR_SHAPE (-1)   /* ShapeError       (errors.py:20) */
#define GLX_ERR_INVALID (-2) /* ValidationError  (errors.py:16) */
#define GLX_ERR_NUMERIC (-3) /* NumericError     (errors.py:24) */
#define GLX_ERR_CUDA (-4)    /* RuntimeError: CUDA / NCCL failure */
#define GLX_ERR_NOMEM (-5)   /* MemoryError */
#define GLX_ERR_RACE (-6)    /* RuntimeError: a debug run's pipeline check failed (backend.py:130-132) */

#define GLX_FP32 0
#define GLX_REF64 1

#define GLX_FLAG_CACHE_INPUTS 1 /* host API: keep feats/targets resident keyed by host pointer */
/* host API, full batch: check the tcgen05 epoch kernels' pipelines every epoch (tile
 * hand-off stamps and per-tile visit counts; GLX_ERR_RACE on a violation) -- the
 * device analogue of the reference's debug=True instrumentation (backend.py:122-133,
 * 237-284). Costs one host sync per epoch. */
#define GLX_FLAG_DEBUG 2

const char* glx_last_error(void);
int glx_version(void);
int glx_device_count(void);
int glx_sm_count(int device);

/* ------------------------------------------------------------------ host API */

/* Drop-in for backend.run_train_segment (backend.py:208-234) /
 * kernels.train_segment_seq|par (kernels.py:264-349): `epochs` passes of
 * per-instance online SGD in dataset order, weights updated in place.
 * feats: rows x input_dim f32, targets: rows f32 in {0,1}. */
int glx_run_train_segment(float* w_ih, float* w_ho, const float* feats, const float* targets, int64_t rows,
                          int32_t input_dim, int32_t hidden_dim, int64_t epochs, double lr, int32_t numerics,
                          int32_t device, int32_t flags);

/* Full-batch gradient descent: every
 * epoch computes the mean gradient over all rows at the epoch-start weights
 * and applies W <- W - lr * grad. FP32 numerics. stats_hist (host, may be
 * NULL) receives 5 doubles per epoch: loss sum, tp, tn, fp, fn at the
 * epoch-start weights. */
int glx_run_train_segment_batch(float* w_ih, float* w_ho, const float* feats, const float* targets, int64_t rows,
                                int32_t input_dim, int32_t hidden_dim, int64_t epochs, double lr,
                                double* stats_hist, int32_t device, int32_t flags);

/* One trainer checkpoint in one call (replacing the
 * segment + 2x eval_counts + weights_finite sequence of trainer.py:152-163):
 * train `epochs` (mode 0 online SGD as glx_run_train_segment, 1 full batch
 * as glx_run_train_segment_batch), then on the device, on the same stream and
 * without a weight round trip: the finiteness test of the new weights and the
 * exact (reference-order f64) confusion counts of the train rows (labels =
 * their u8 labels; the rows are already resident) and of the test rows.
 * counts8 = train (tp, tn, fp, fn) then test (tp, tn, fp, fn); loss2 = the two
 * loss sums; finite = 1 iff every weight is finite; train_seconds = the call's
 * wall time minus the evaluation's device time. The weights are copied back
 * as by the segment calls. With GLX_FLAG_CACHE_INPUTS the train and test rows
 * stay resident across checkpoint calls (keyed on the host pointers). */
int glx_run_train_segment_eval(float* w_ih, float* w_ho, const float* feats, const float* targets,
                               const uint8_t* labels, int64_t rows, const float* test_feats,
                               const uint8_t* test_labels, int64_t test_rows, int32_t input_dim, int32_t hidden_dim,
                               int64_t epochs, double lr, int32_t numerics, int32_t mode, int32_t device,
                               int32_t flags, int64_t* counts8, double* loss2, int32_t* finite, double* train_seconds);

/* Drop-in for kernels.eval_counts (kernels.py:352-375) plus the loss sum.
 * counts4 = (tp, tn, fp, fn) for output_dim 1, (correct, wrong, 0, 0) for
 * output_dim > 1 (argmax). labels: rows u8. */
int glx_eval_counts(const float* w_ih, const float* w_ho, const float* feats, const uint8_t* labels, int64_t rows,
                    int32_t input_dim, int32_t hidden_dim, int32_t output_dim, int32_t numerics, int64_t* counts4,
                    double* loss_sum, int32_t device, int32_t flags);

/* Drop the resident-input cache of GLX_FLAG_CACHE_INPUTS (all devices). */
void glx_cache_clear(void);

/* ---------------------------------------------------------------- device API */

/* Online SGD on device buffers (single network). X: N x D, T: N. Any D and H:
 * D <= 63 and H <= 512 run the register-tiled kernels, wider networks the
 * any-shape engine (weights in global memory; fails with GLX_ERR_INVALID when
 * 2D + H floats of row and activations exceed its ~200 KB of shared memory). */
int glx_train_online(float* w_ih, float* w_ho, const float* X, const float* T, int64_t N, int32_t D, int32_t H,
                     int64_t epochs, double lr, int32_t numerics, void* stream);

/* n_nets independent online networks on one dataset (config 3): network n
 * owns w_pool[w_off[n] ...] = [w_ih (H_n x (D+1)) | w_ho (H_n + 1)].
 * H_per_net and w_off are HOST arrays; w_pool, X, T are device pointers. */
int glx_train_sweep(int64_t n_nets, const int32_t* H_per_net, const int64_t* w_off, float* w_pool, const float* X,
                    const float* T, int64_t N, int32_t D, int64_t epochs, double lr, int32_t numerics, void* stream);

/* Packed row layout of the streaming kernels: row r at Xp + r*ld with
 * ld = glx_packed_ld(D), holding [x_0..x_{D-1}, 1.0, target, 0...]. */
int32_t glx_packed_ld(int32_t D);
int glx_pack_rows(const float* X, const float* T, const uint8_t* labels, int64_t N, int32_t D, float* Xp,
                  void* stream);
/* The same packing with the reference's min-max normalisation applied to the
 * features on the way (dataset.py:383-392; see glx_minmax_apply). */
int glx_pack_rows_minmax(const float* X, const float* T, const uint8_t* labels, int64_t N, int32_t D,
                         const float* col_min, const float* col_max, float* Xp, void* stream);

/* Min-max normalisation, replacing dataset.normalize_fit / normalize_apply
 * (dataset.py:369-392). glx_minmax_fit: col_min/col_max (device float[D]) =
 * per-column min and max of the N x D row-major f32 rows (exact). glx_minmax_apply:
 * Y = X scaled as f32((x - min) / (max - min)) with IEEE f32 ops, constant
 * columns -> 0, clamped to [-0.5, 1.5]; Y may alias X. Inputs are finite
 * (NaN propagation of numpy's min/max is not reproduced). */
int glx_minmax_fit(const float* X, int64_t N, int32_t D, float* col_min, float* col_max, void* stream);

/* Benchmark rows on the device (replacing dataset.synthetic_matrix's host
 * generation, dataset.py:260-289): numpy's PCG64 stream
 * reproduced bit for bit by jump-ahead. state/inc = the 128-bit PCG64 state
 * and increment of default_rng(seed) (bit_generator.state), split hi/lo.
 * glx_pcg64_uniform_f32: out[i] = the i-th float32 draw (Generator.random(
 * dtype=float32)) counted from 64-bit output first_output (two floats per
 * output, low half first). glx_pcg64_coin: labels[r] = 1 iff the float64 draw
 * of output first_output + r is < 0.5 (Generator.random() < 0.5).
 * glx_planted_score: score[r] = sum_q f64(X[r, pick[q]]) * coef[q] (device
 * pick/coef); glx_label_ge: labels[r] = score[r] >= *threshold (device). */
int glx_pcg64_uniform_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first_output,
                          int64_t n_floats, float* out, void* stream);
int glx_pcg64_coin(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first_output,
                   int64_t n, uint8_t* labels, void* stream);
int glx_planted_score(const float* X, int64_t N, int32_t D, const int32_t* pick, const double* coef, int32_t k,
                      double* score, void* stream);
int glx_label_ge(const double* score, int64_t N, const double* threshold, uint8_t* labels, void* stream);
int glx_minmax_apply(const float* X, int64_t N, int32_t D, const float* col_min, const float* col_max, float* Y,
                     void* stream);

/* Full-batch GD on packed rows. stats_hist: device double[5*epochs] or NULL.
 * nonfinite: device int32 set to 1 if any updated weight is non-finite. */
int glx_train_batch(float* w_ih, float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H, int64_t epochs,
                    double lr, double* stats_hist, int32_t* nonfinite, void* stream);

/* Which full-batch epoch kernel glx_train_batch / glx_batch_grad run for this
 * shape: 3 = tcgen05 rows-on-lanes kernel (24 <= H <= 64, D <= 33, from 2^17
 * rows), 2 = tcgen05 units-on-lanes kernel (24 <= H <= 256, D <= 33), 1 =
 * three-role FP32 kernel, 0 = two-role FP32 kernel (D <= 127, H <= 512), 4 =
 * the any-shape FP32 engine (tiled GEMM-shaped kernels, glx_generic.cu), -1 =
 * invalid arguments. Selection only (no device work); GLX_BATCH_KERNEL=3 / =2 cap the choice
 * at 1 / 0, =tc / =rt force a tcgen05 kernel. No reference counterpart (diagnostic). */
int glx_batch_kernel_kind(int64_t N, int32_t D, int32_t H);

/* Data-parallel split of one epoch (config 4): glx_batch_grad writes this
 * rank's gradient SUM over its N rows (not divided by N) into grad (device
 * double[glx_batch_grad_len]), laid out as [dW1 (H(D+1)) | dW2 (H+1) | loss,
 * tp, tn, fp, fn]; after an all-reduce(sum) across ranks, glx_batch_apply
 * performs W <- f32(f64(W) - lr_over_n * grad) with n the global row count. */
int64_t glx_batch_grad_len(int32_t D, int32_t H);
int glx_batch_grad(const float* w_ih, const float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H,
                   double* grad, void* stream);
int glx_batch_apply(float* w_ih, float* w_ho, const double* grad, int32_t D, int32_t H, double lr_over_n,
                    int32_t* nonfinite, void* stream);

/* ------------------------------------------------ data-parallel data plane
 * SURVEY.md 8(b) (glx_dp_init) and 8(e): the per-epoch gradient exchange of the
 * data-parallel batch configurations (C2/C4 across GPUs) over NCCL, owned by
 * this library (no reference counterpart: the reference has no multi-process
 * or multi-GPU path). One communicator per rank (one process
 * per GPU). glx_dp_unique_id fills the 128-byte ncclUniqueId on one rank; the
 * caller ships it to the others by any channel; every rank then calls
 * glx_dp_init (ncclCommInitRank, collective: all ranks must call it).
 * glx_dp_allreduce_f64: in-place all-reduce of n doubles (op 0 sum, 1 max) on
 * `stream`. glx_dp_train_batch: `epochs` full-batch epochs over this rank's N
 * packed rows (glx_packed_ld layout) with the global row count N_total; every
 * epoch = the epoch kernel, the f64 gradient sum, ncclAllReduce(sum) of the
 * P + 5 doubles, and the update W <- f32(f64(W) - lr/N_total * grad) applied
 * identically on every rank; captured once into a CUDA graph and replayed
 * (GLX_DP_GRAPH=0: eager). N may be 0 (the rank still joins the all-reduce).
 * stats_hist (device, may be NULL): 5 doubles per epoch, loss, tp, tn, fp, fn
 * over ALL ranks' rows at the epoch-start weights. Collective: all ranks call
 * it with the same D, H, epochs, lr, N_total.
 * glx_dp_run_train_segment_batch: the same from host buffers (the rank's
 * shard), with glx_run_train_segment_batch's copy-in/copy-out contract. */
int glx_dp_unique_id(uint8_t* id128);
int glx_dp_init(int32_t device, int32_t nranks, int32_t rank, const uint8_t* id128, void** comm);
int glx_dp_finalize(void* comm);
int glx_dp_allreduce_f64(void* comm, double* buf, int64_t n, int32_t op, void* stream);
int glx_dp_train_batch(void* comm, float* w_ih, float* w_ho, const float* Xp, int64_t N, int64_t N_total, int32_t D,
                       int32_t H, int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream);
int glx_dp_run_train_segment_batch(void* comm, float* w_ih, float* w_ho, const float* feats, const float* targets,
                                   int64_t rows, int64_t rows_total, int32_t input_dim, int32_t hidden_dim,
                                   int64_t epochs, double lr, double* stats_hist, int32_t flags);

/* Evaluation on device buffers; results land in device memory
 * (counts4: uint64[4] accumulated, so zero it first; loss: double[1]). */
int glx_eval(const float* w_ih, const float* w_ho, const float* X, const uint8_t* labels, int64_t N, int32_t D,
             int32_t H, int32_t K, uint64_t* counts4, double* loss, void* stream);
/* Fast FP32 evaluation on packed rows (fused streaming forward);
 * stats: device double[5] = loss, tp, tn, fp, fn. */
int glx_eval_packed(const float* w_ih, const float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H,
                    double* stats, void* stream);

/* tcgen05 tensor-core GEMM used by the wide configuration:
 * D[M x N] = A[M x K] . B[N x K]^T with bf16 row-major A, B (device) and f32
 * accumulation in TMEM. epilogue 0 writes D as f32 (row stride ldd); epilogue 1
 * writes bf16 sigmoid(D + bias[col]) to d_bf16. K % 64 == 0, N % 32 == 0. */
int glx_tc_gemm_bf16(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epilogue, float* d_f32,
                     void* d_bf16, const float* bias, int32_t ldd, void* stream);

/* Wide configuration: 1024 inputs -> 1024 hidden -> 16
 * sigmoid outputs, full-batch GD with every large contraction on tcgen05
 * (BF16 operands, FP32 accumulation in TMEM). glx_wide_make_data fills the
 * device buffers Xb (N x 1024 bf16, U[0,1)), XT (1025 x N bf16: [X,1]^T in
 * the K-blocked layout [N/64][1025][64], element (i, r) at
 * ((r/64)*1025 + i)*64 + r%64) and labels (N u8 class ids in [0,16));
 * N % 64 == 0.
 * glx_wide_train runs `epochs` epochs on f32 master weights in the reference
 * layout (w_ih 1024 x 1025, w_ho 16 x 1025); stats_hist (device, may be NULL)
 * gets [loss, correct, wrong] per epoch at the epoch-start weights. */
int glx_wide_make_data(int64_t N, uint64_t seed, void* Xb, void* XT, uint8_t* labels, void* stream);
/* Rows [row0, row0 + N) of the same data set (a data-parallel shard). */
int glx_wide_make_shard(int64_t row0, int64_t N, uint64_t seed, void* Xb, void* XT, uint8_t* labels, void* stream);
/* Data-parallel split of one wide epoch (SURVEY.md 8(e) for C5): glx_wide_grad
 * writes the f64 gradient SUM over this shard's rows at the current weights
 * into grad[0, P) (reference layout: w_ih then w_ho, P = 1,066,000) and
 * [loss, correct, wrong] into grad[P, P+3); after an all-reduce of the
 * glx_wide_grad_len() doubles, glx_wide_apply performs
 * W <- f32(f64(W) - lr_over_n * grad) identically on every rank. */
int64_t glx_wide_grad_len(void);
int glx_wide_grad(const float* w_ih, const float* w_ho, const void* Xb, const void* XT, const uint8_t* labels,
                  int64_t N, double* grad, void* stream);
int glx_wide_apply(float* w_ih, float* w_ho, const double* grad, double lr_over_n, int32_t* nonfinite, void* stream);
int glx_wide_train(float* w_ih, float* w_ho, const void* Xb, const void* XT, const uint8_t* labels, int64_t N,
                   int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream);

/* The wide configuration with f32 rows on tcgen05 kind::tf32 (f32 storage of H and
 * the deltas; SURVEY.md C5 "evaluated against the FP32 tolerance"): X f32 [N][1024]
 * U[0,1) and [X,1]^T f32 K-blocked [N/32][1025][32] (element (i, r) at
 * ((r/32)*1025 + i)*32 + r%32), labels as glx_wide_make_data; N % 32 == 0. The
 * gradient and training calls mirror glx_wide_grad / glx_wide_train (the update is
 * glx_wide_apply). */
int glx_wide_make_shard_tf32(int64_t row0, int64_t N, uint64_t seed, float* X, float* XT, uint8_t* labels,
                             void* stream);
int glx_wide_grad_tf32(const float* w_ih, const float* w_ho, const float* X, const float* XT, const uint8_t* labels,
                       int64_t N, double* grad, void* stream);
int glx_wide_train_tf32(float* w_ih, float* w_ho, const float* X, const float* XT, const uint8_t* labels, int64_t N,
                        int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream);

/* ---------------------------------------------------- per-instance API */
/* network.forward (network.py:128-135) for N rows, the reference's f64 order:
 * hidden (device, N x H f32) and out (device, N x K f32) activations. */
int glx_forward(const float* w_ih, const float* w_ho, const float* X, int64_t N, int32_t D, int32_t H, int32_t K,
                float* hidden, float* out, void* stream);
/* Layer-level API (backend.py:73-205, kernels.py:163-257), device buffers, the
 * reference's f64 order. glx_layer_forward: out[r][j] = _activation of neuron j
 * (W: n x (m+1) f32, bias last) on input row r of X (N x m). glx_layer_backward:
 * deltas[j] = (err[j] a_j)(1 - a_j), grads[j] = deltas[j] [x, 1] (n x (m+1) f64).
 * glx_backprop_error: err_prev[i] = sum_j W[j][i] deltas[j], 16-blocked over j. */
int glx_layer_forward(const float* W, const float* X, int64_t N, int32_t m, int32_t n, float* out, void* stream);
int glx_layer_backward(const float* x, const float* acts, const double* err, int32_t n, int32_t m, double* deltas,
                       double* grads, void* stream);
int glx_backprop_error(const float* W, const double* deltas, int32_t n, int32_t m, double* err_prev, void* stream);
/* network.loss_gradients (network.py:144-165) for one row, one output, from its
 * forward activations: g_ih (H x (D+1) f64) and g_ho (H+1 f64), device. */
int glx_instance_gradients(const float* w_ho, const float* x, const float* hidden, const float* out, double target,
                           int32_t D, int32_t H, double* g_ih, double* g_ho, void* stream);

/* ------------------------------------------------------------ diagnostics */
/* Number of CUDA kernels this library has launched (for launch accounting). */
uint64_t glx_launch_count(void);
/* Per-launch timing of the streaming epoch kernel (batch_epoch_kernel): when
 * enabled, an event pair is recorded on the launching stream around every
 * launch; glx_profile_read synchronises, returns the summed kernel time and
 * launch count since the last read, and resets. */
/* Debug instrumentation of the layer-level API (backend.py:122-133, 237-284).
 * write_counts (device int32[N*n] / [n], zeroed by the caller): every output
 * slot adds 1 when written; the caller requires all ones. glx_forward_pair_debug:
 * `workers` warps write the hidden activations and stamp each slot; after the
 * layer barrier the output pass checks every stamp (status: device int32, 0 = ok,
 * 1 + j = hidden slot j read before it was written; stamps: device int32[H],
 * zeroed by the caller). */
int glx_layer_forward_checked(const float* W, const float* X, int64_t N, int32_t m, int32_t n, float* out,
                              int32_t* write_counts, void* stream);
int glx_layer_backward_checked(const float* x, const float* acts, const double* err, int32_t n, int32_t m,
                               double* deltas, double* grads, int32_t* write_counts, void* stream);
int glx_forward_pair_debug(const float* w_ih, const float* w_ho, const float* x, int32_t D, int32_t H, int32_t K,
                           float* hidden, float* out, int32_t* stamps, int32_t* status, int32_t workers,
                           void* stream);

/* Process-wide debug switch: every full-batch training call (host and device API)
 * runs the GLX_FLAG_DEBUG pipeline checks, as does glx_batch_grad. */
void glx_set_debug(int32_t on);

void glx_profile_enable(int32_t on);
int glx_profile_read(double* total_ms, int64_t* launches);
/* FFMA2 throughput microbenchmark on `device`: returns TFLOP/s. */
int glx_fp32_peak(int32_t device, int32_t iters, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* GLYCEMLP_CUDA_H */
