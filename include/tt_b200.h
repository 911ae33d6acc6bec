/*
 * tt_b200.h -- C ABI of libtt_b200.so, the B200 (sm_100a) hot path of the
 * tensortune cost model (arXiv 2304.05430 reproduction).
 *
 * The reference (/root/reference/pkg/src/tensortune) is pure Python; its
 * "plugin API" for this path is the duck-typed estimator / metric / sampling
 * functions listed beside each entry point below.  The Python host package
 * paper_2304_05430_b200 binds these symbols with ctypes and exposes the
 * reference's own names; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - plain pointers + sizes, no C++ or torch types;
 *  - "d_" pointers are device memory, "h_" pointers host memory;
 *  - every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    unless stated; buffers are caller-owned; the workspace of a call must
 *    not be shared with a concurrently running call;
 *  - return value: TT_OK or an error code; tt_last_error() gives a
 *    thread-local message.  No exceptions cross the ABI.
 *  - *_f32 entry points compute in float32 (the production path), *_f64 in
 *    float64 (the parity/debug build of the same kernels).
 */
#ifndef TT_B200_H
#define TT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_OK 0
#define TT_EINVAL 1        /* bad argument (shape, size, unsupported width) */
#define TT_ENONFINITE 2    /* reserved: non-finite data detected host-side */
#define TT_ECUDA 3         /* CUDA runtime error (launch, co-residency, ...) */

#define TT_LOSS_MSE 0      /* tuner.py:373-375, mlp.py:105-108 */
#define TT_LOSS_RANK 1     /* mlp.py:25-35 (pairwise logistic) */

#define TT_MODE_TRAIN 0    /* forward + backward + Adam for every minibatch */
#define TT_MODE_GRAD 1     /* one minibatch: forward + backward, write gradient */

typedef void *tt_stream_t;

int tt_abi_version(void);
const char *tt_last_error(void);

/* ------------------------------------------------------------------ PCA --
 * replaces metrics.py:46-58 pairwise_comparison_accuracy (called per task by
 * models.py:384-419 per_task_metrics and tuner.py:486-496 _grouped_pca).
 * Tasks are CSR segments of (y, s); d_correct[t] receives the exact number
 * of pairs i<j of task t with sign(y_i-y_j) == sign(s_i-s_j).  The caller
 * zero-fills nothing: the call overwrites d_correct.  h_offsets is a HOST
 * array (n_tasks+1) -- it is needed to plan the pair tiles. */
size_t tt_pca_workspace_bytes(const int64_t *h_offsets, int32_t n_tasks);
int tt_pca_counts(const double *d_y, const double *d_s, const int64_t *h_offsets,
                  int32_t n_tasks, int64_t *d_correct, void *d_ws, size_t ws_bytes,
                  tt_stream_t stream);

/* replaces metrics.py:61-75 top_k_score: per task, d_pick[t] = max y over the
 * min(k, n_t) best scores (stable: ties broken by lower index), d_best[t] =
 * max y.  top_k_score = d_pick / d_best (computed by the caller). */
int tt_topk(const double *d_y, const double *d_s, const int64_t *d_offsets, int32_t n_tasks,
            int32_t k, double *d_pick, double *d_best, tt_stream_t stream);

/* ------------------------------------------------------------ rank loss --
 * replaces estimators/mlp.py:25-35 ranking_grad, one segment per minibatch;
 * max_seg bounds the longest segment (sizes shared memory). */
int tt_rank_loss_f32(const float *d_y, const float *d_s, const int64_t *d_offsets,
                     int32_t n_segs, int32_t max_seg, float *d_loss, float *d_grad,
                     tt_stream_t stream);
int tt_rank_loss_f64(const double *d_y, const double *d_s, const int64_t *d_offsets,
                     int32_t n_segs, int32_t max_seg, double *d_loss, double *d_grad,
                     tt_stream_t stream);

/* ----------------------------------------------------------------- Adam --
 * replaces estimators/optim.py:33-46 Adam.step on a flat parameter vector.
 * corr1 = 1 - b1^t, corr2 = 1 - b2^t (t = step counter after increment).
 * d_mask (uint8 per element, may be NULL) selects trainable entries. */
int tt_adam_step_f32(float *d_param, const float *d_grad, float *d_m, float *d_v, int64_t n,
                     const uint8_t *d_mask, double lr, double b1, double b2, double eps,
                     double corr1, double corr2, tt_stream_t stream);
int tt_adam_step_f64(double *d_param, const double *d_grad, double *d_m, double *d_v, int64_t n,
                     const uint8_t *d_mask, double lr, double b1, double b2, double eps,
                     double corr1, double corr2, tt_stream_t stream);

/* ---------------------------------------------------- attention tuner --
 * replaces estimators/tuner.py RecurrentAttentionTuner._forward/_backward/
 * loss_and_gradients/_train/predict (tuner.py:227-476).
 *
 * Parameters: one flat vector, tensors in the reference's dict order
 * (tuner.py:194-210), each row-major:
 *   for l < layers, for dir in (fw, bw): Wx[d_in][4H], Wh[H][4H], b[4H]
 *   attn_Wq, attn_Wk, attn_Wv, attn_Wo [2H][2H], attn_bq[2H], attn_bo[2H],
 *   head_W1[2H+C][64], head_b1[64], head_W2[64][1], head_b2[1]
 * with d_in = step_width for l == 0 else 2H.  hidden in {4, 8, 16, 32}.
 * Programs: CSR -- d_steps (total_rows x step_width), d_row_offsets (n+1,
 * int64), d_ctx (n x ctx_len); every program has 1..max_steps rows. */
int64_t tt_tuner_param_count(int32_t layers, int32_t hidden, int32_t step_width,
                             int32_t ctx_len);
size_t tt_tuner_predict_workspace_bytes(int32_t f64, int32_t layers, int32_t hidden,
                                        int32_t max_steps);
int tt_tuner_predict_f32(const float *d_params, const float *d_steps,
                         const int64_t *d_row_offsets, const float *d_ctx, int64_t n,
                         int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                         int32_t step_width, int32_t ctx_len, int32_t max_steps,
                         float *d_yhat, void *d_ws, size_t ws_bytes, tt_stream_t stream);
int tt_tuner_predict_f64(const double *d_params, const double *d_steps,
                         const int64_t *d_row_offsets, const double *d_ctx, int64_t n,
                         int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                         int32_t step_width, int32_t ctx_len, int32_t max_steps,
                         double *d_yhat, void *d_ws, size_t ws_bytes, tt_stream_t stream);

/* Tensor-core scoring (tcgen05 kind::tf32, csrc/tt_tuner_tc.cu): the same
 * forward as tt_tuner_predict_f32 with every dense layer (LSTM gates, Wq,
 * Wk, Wv, Wo, W1) as a 128-program GEMM tile; tf32 operands, fp32
 * accumulation and activations ("tf32" precision mode, its own tolerance).
 * Requires hidden = 32, heads in {1, 2}, step_width <= 32, ctx_len <= 64;
 * TT_EINVAL otherwise.  d_ws: tt_tuner_predict_tf32_workspace_bytes(max_steps). */
size_t tt_tuner_predict_tf32_workspace_bytes(int32_t max_steps);
int tt_tuner_predict_tf32(const float *d_params, const float *d_steps,
                          const int64_t *d_row_offsets, const float *d_ctx, int64_t n,
                          int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                          int32_t step_width, int32_t ctx_len, int32_t max_steps,
                          float *d_yhat, void *d_ws, size_t ws_bytes, tt_stream_t stream);

/* fp32-accurate tensor-core scoring (csrc/tt_tuner_x3.cu): the biLSTM stack
 * as split-precision tcgen05 GEMMs (x.w = x_hi.w_hi + x_lo.w_hi + x_hi.w_lo,
 * fp32 accumulation; MUFU ex2/rcp activations), then attention + head in
 * fp32 on the CUDA cores (K and V never formed, online softmax).  Same
 * signature and outputs as tt_tuner_predict_f32 (within its fp32 tolerance);
 * a program's score does not depend on the batch it is scored in.
 * tt_tuner_f32tc_eligible says whether the shapes are covered (hidden = 32,
 * step_width <= 32).  The workspace depends on n (launches of up to 4 tiles of
 * 128 programs per SM; small calls need little). */
size_t tt_tuner_predict_f32tc_workspace_bytes(int32_t layers, int32_t hidden, int32_t max_steps, int64_t n);
int tt_tuner_f32tc_eligible(int32_t layers, int32_t hidden, int32_t heads, int32_t step_width,
                            int32_t max_steps);
int tt_tuner_predict_f32tc(const float *d_params, const float *d_steps,
                           const int64_t *d_row_offsets, const float *d_ctx, int64_t n,
                           int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                           int32_t step_width, int32_t ctx_len, int32_t max_steps,
                           float *d_yhat, void *d_ws, size_t ws_bytes, tt_stream_t stream);

/* Training (tuner.py:427-466) / gradients (tuner.py:364-376).
 * d_order lists sample indices; minibatch k is d_order[k*B, min((k+1)*B, n_order)).
 * TT_MODE_TRAIN: every minibatch runs forward, loss, backward, a deterministic
 *   fixed-order gradient reduction and the fused Adam update; d_corr holds
 *   (1-b1^t, 1-b2^t) per minibatch; d_step_loss[k] receives the loss; on a
 *   non-finite loss d_status[0] = k and the kernel stops before updating.
 * TT_MODE_GRAD: exactly one minibatch (B = n_order); d_grad_out receives the
 *   full gradient (param_count) and d_step_loss[0] the loss; no update.
 * d_trainable: uint8 per parameter element or NULL (all trainable). */
size_t tt_tuner_train_workspace_bytes(int32_t f64, int32_t layers, int32_t hidden,
                                      int32_t step_width, int32_t ctx_len, int32_t max_steps,
                                      int32_t batch_size);
int tt_tuner_train_f32(float *d_params, float *d_m, float *d_v, const float *d_steps,
                       const int64_t *d_row_offsets, const float *d_ctx, const float *d_y,
                       const int32_t *d_order, int64_t n_order, int32_t batch_size,
                       int32_t loss_kind, int32_t mode, double lr, double b1, double b2,
                       double eps, const double *d_corr, const uint8_t *d_trainable,
                       int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                       int32_t step_width, int32_t ctx_len, int32_t max_steps,
                       float *d_step_loss, float *d_grad_out, int32_t *d_status, void *d_ws,
                       size_t ws_bytes, tt_stream_t stream);
int tt_tuner_train_f64(double *d_params, double *d_m, double *d_v, const double *d_steps,
                       const int64_t *d_row_offsets, const double *d_ctx, const double *d_y,
                       const int32_t *d_order, int64_t n_order, int32_t batch_size,
                       int32_t loss_kind, int32_t mode, double lr, double b1, double b2,
                       double eps, const double *d_corr, const uint8_t *d_trainable,
                       int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                       int32_t step_width, int32_t ctx_len, int32_t max_steps,
                       double *d_step_loss, double *d_grad_out, int32_t *d_status, void *d_ws,
                       size_t ws_bytes, tt_stream_t stream);

/* Heads-only fine-tuning (transfer.py fine_tune with trainable = the
 * attention + head groups, tuner.py:397-425): the recurrent stack is frozen,
 * so its last-layer outputs S are computed once per call and training steps
 * run only attention, head, loss and their gradients.
 *   tt_tuner_lstm_outputs_f32: tt_tuner_predict_f32 that also writes S in the
 *     CSR row layout, d_s_out [sum T][2 * hidden] (same workspace).
 *   tt_tuner_train_heads_f32: tt_tuner_train_f32 (mode TRAIN) reading S from
 *     d_s_cache; the recurrent parameters and their moments are left
 *     untouched whatever d_trainable says.  Latency-path kernel only
 *     (hidden 32, batch <= 2048): TT_EINVAL otherwise. */
int tt_tuner_lstm_outputs_f32(const float *d_params, const float *d_steps,
                              const int64_t *d_row_offsets, const float *d_ctx, int64_t n,
                              int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                              int32_t step_width, int32_t ctx_len, int32_t max_steps,
                              float *d_s_out, float *d_yhat, void *d_ws, size_t ws_bytes,
                              tt_stream_t stream);
int tt_tuner_train_heads_f32(float *d_params, float *d_m, float *d_v, const float *d_steps,
                             const int64_t *d_row_offsets, const float *d_ctx, const float *d_y,
                             const int32_t *d_order, int64_t n_order, int32_t batch_size,
                             int32_t loss_kind, double lr, double b1, double b2, double eps,
                             const double *d_corr, const uint8_t *d_trainable, int32_t layers,
                             int32_t hidden, int32_t heads, int32_t unroll, int32_t step_width,
                             int32_t ctx_len, int32_t max_steps, const float *d_s_cache,
                             float *d_step_loss, int32_t *d_status, void *d_ws, size_t ws_bytes,
                             tt_stream_t stream);

/* Data-parallel training fused into the training kernel (SURVEY §8e,
 * option A: the reference's rank loss within each rank's microbatch, the
 * step's gradient = the mean of the world's microbatch gradients, replicated
 * Adam).  One launch per epoch per rank, each on its own data shard (equal
 * shard sizes).  Every gradient job stores its reduced slice into the
 * peers' exchange buffers (NVLink peer memory, opened with tt_ipc_open) as
 * 8-byte {value, step flag} words, spins on its own slots until the peers'
 * words carry the step's flag and sums them in rank order -- no fences, no
 * separate all-reduce or Adam launch.
 *   tt_tuner_dp_buffer_bytes: size of one rank's exchange buffer.
 *   d_xb: device array [world] of the exchange buffer base pointers (own
 *     included, index = rank); buffers zeroed once (tt_ipc_alloc does).
 *   gbase: global index of this launch's first step, monotone across
 *     launches (flags carry gbase + step + 1).
 * A non-finite loss sets d_status[0] on the rank where it happened, but every
 * rank runs the epoch to its end (the host combines the statuses).  For
 * world > 1, d_status points at TWO int32 {first non-finite step or -1,
 * abort word = 0}: a wait for a peer's slice longer than the timeout
 * (tt_tuner_dp_set_timeout_ms, default 30 s) sets the abort word to 1, after
 * which no exchange of the launch waits any more -- the epoch ends quickly
 * with invalid parameters and the host raises, instead of hanging all ranks.
 * tt_ipc_alloc/open/close, tt_dev_free: the cudaIpc* plumbing (64-B handles).
 * tt_tuner_train_set_grid: CTAs of the latency-path launch (0 = every SM);
 * tests run several ranks concurrently on one GPU by splitting its SMs. */
size_t tt_tuner_dp_buffer_bytes(int32_t layers, int32_t hidden, int32_t step_width, int32_t ctx_len,
                                int32_t world);
int tt_tuner_train_dp_f32(float *d_params, float *d_m, float *d_v, const float *d_steps,
                          const int64_t *d_row_offsets, const float *d_ctx, const float *d_y,
                          const int32_t *d_order, int64_t n_order, int32_t batch_size,
                          int32_t loss_kind, double lr, double b1, double b2, double eps,
                          const double *d_corr, const uint8_t *d_trainable, int32_t layers,
                          int32_t hidden, int32_t heads, int32_t unroll, int32_t step_width,
                          int32_t ctx_len, int32_t max_steps, int32_t world, int32_t rank,
                          int64_t gbase, void *const *d_xb, float *d_step_loss, int32_t *d_status,
                          void *d_ws, size_t ws_bytes, tt_stream_t stream);
int tt_ipc_alloc(size_t bytes, void **d_ptr, uint8_t *h_handle);
int tt_ipc_open(const uint8_t *h_handle, void **d_ptr);
int tt_ipc_close(void *d_ptr);
int tt_dev_free(void *d_ptr);
int tt_tuner_train_set_grid(int32_t grid);
int tt_tuner_dp_set_timeout_ms(int64_t ms);
/* 1 if tt_tuner_train_f32 / _dp_f32 would run these dimensions on the
 * latency-path kernel (the data-parallel launch requires it), else 0. */
int32_t tt_tuner_train_fast_eligible(int32_t layers, int32_t hidden, int32_t heads, int32_t unroll,
                                     int32_t step_width, int32_t ctx_len, int32_t max_steps,
                                     int32_t batch_size);

/* Kernel selection for tt_tuner_train_f32: 0 = automatic (the latency-path
 * kernel when hidden = 32, batch <= #SMs and the per-sample caches fit in
 * shared memory, else the generic kernel), 1 = generic only, 2 = latency path
 * only (TT_EINVAL when not eligible).  Process-wide; for tests and benches. */
int tt_tuner_train_set_path(int32_t path);

/* Debug aid: record clock64() phase marks of CTA 0 for minibatch `step` of the
 * next tuner training launches (-1 = off) and read them back (host memory). */
int tt_debug_profile_step(int32_t step);
int tt_debug_phase_times(int64_t *h_out, int32_t n);
/* Debug aid: clock64 marks of the tensor-core scoring kernel's first tile. */
int tt_debug_tc_phase_times(int64_t *h_out, int32_t n);
/* Same for the fp32 tensor-core LSTM kernel (tt_tuner_x3.cu: layer 1,
 * forward direction, steps 2 and 3 of CTA 0's first tile). */
int tt_debug_x3_phase_times(int64_t *h_out, int32_t n);
/* Same for the shared-memory CostMLP training kernel (clock64 of CTA 0,
 * thread 0, at its phase boundaries of minibatch 64 of the last launch). */
int tt_debug_mlp_phase_times(int64_t *h_out, int32_t n);

/* ------------------------------------------------------------ cost MLP --
 * replaces estimators/mlp.py CostMLP._forward/_backward/fit/predict
 * (mlp.py:72-155).  Params flat in dict order W1[F][64], b1[64], W2[64][64],
 * b2[64], W3[64][1], b3[1]; X is n x F row-major. */
int64_t tt_mlp_param_count(int32_t n_features);
int tt_mlp_predict_f32(const float *d_params, const float *d_X, int64_t n, int32_t n_features,
                       float *d_out, tt_stream_t stream);
int tt_mlp_predict_f64(const double *d_params, const double *d_X, int64_t n,
                       int32_t n_features, double *d_out, tt_stream_t stream);
/* tcgen05 tensor-core scoring (kind::tf32 operands, fp32 accumulation and
 * activations): TMA-fed, warp-specialised, persistent.  Requires
 * n_features*4 % 16 == 0 (TMA row stride), X 16-B aligned.  Tolerance vs the
 * float64 reference: max |d| <= 1e-2, mean |d| <= 1e-3 (tests). */
int tt_mlp_predict_tf32(const float *d_params, const float *d_X, int64_t n, int32_t n_features,
                        float *d_out, tt_stream_t stream);
/* The default fp32 scorer on the tensor cores: split-precision tf32 (each
 * operand = tf32 hi + tf32 lo, three products per layer accumulated in fp32,
 * ~2^-21 relative layer error; accurate exp-based tanh), same tcgen05/TMA
 * pipeline as tt_mlp_predict_tf32.  Eligible (tt_mlp_f32tc_eligible) when
 * F*4 is a multiple of 16, d_X is 16-B aligned and the split weights fit in
 * shared memory (F <= ~190); replaces mlp.py:146-155 predict at fp32. */
int tt_mlp_predict_f32tc(const float *d_params, const float *d_X, int64_t n, int32_t n_features,
                         float *d_out, tt_stream_t stream);
int32_t tt_mlp_f32tc_eligible(int32_t n_features, const float *d_X);
size_t tt_mlp_train_workspace_bytes(int32_t f64, int32_t n_features, int32_t batch_size);
int tt_mlp_train_f32(float *d_params, float *d_m, float *d_v, const float *d_X, const float *d_y,
                     int32_t n_features, const int32_t *d_order, int64_t n_order,
                     int32_t batch_size, int32_t loss_kind, int32_t mode, double lr, double b1,
                     double b2, double eps, const double *d_corr, float *d_step_loss,
                     float *d_grad_out, int32_t *d_status, void *d_ws, size_t ws_bytes,
                     tt_stream_t stream);
int tt_mlp_train_f64(double *d_params, double *d_m, double *d_v, const double *d_X,
                     const double *d_y, int32_t n_features, const int32_t *d_order,
                     int64_t n_order, int32_t batch_size, int32_t loss_kind, int32_t mode,
                     double lr, double b1, double b2, double eps, const double *d_corr,
                     double *d_step_loss, double *d_grad_out, int32_t *d_status, void *d_ws,
                     size_t ws_bytes, tt_stream_t stream);

/* ------------------------------------------------- pruning statistics --
 * replaces sampling.py:37-59 filter_invalid's arithmetic (+ data.py:440-446
 * throughput and numpy's linear quantile).  Records are CSR by task
 * (d_task_offsets, n_tasks+1); d_valid marks non-error records (cost must be
 * > 0 for them).  Outputs: d_thr[t] (NaN for tasks without valid records),
 * d_survivors[t], d_task_keep[t], d_keep[r] (record kept by filter_invalid).
 * Bit-exact with numpy float64. */
size_t tt_prune_workspace_bytes(int64_t n_records);
int tt_prune_stats(const int64_t *d_flops, const double *d_cost, const uint8_t *d_valid,
                   const int64_t *d_task_offsets, int32_t n_tasks, double q,
                   int32_t min_records, double *d_thr, uint8_t *d_keep, int32_t *d_survivors,
                   uint8_t *d_task_keep, void *d_ws, size_t ws_bytes, tt_stream_t stream);

/* ---------------------------------------------------------------- GBDT --
 * replaces estimators/gbdt.py:51-265 GradientBoostedTrees._grow / fit's
 * update / predict, bit-exact in float64.
 * tt_gbdt_grow: one tree on residuals d_g.  d_Xc is the n x F training matrix
 *   in COLUMN-major order (F rows of n), d_root_order the F x n stable
 *   argsort of its columns (gbdt.py:109).  Outputs the tree in LEVEL order
 *   (root 0; the host renumbers into the reference's stack order): node
 *   arrays of capacity 2n+1, *d_node_count, and d_incr[r] = the leaf value of
 *   row r's leaf.  Workspace: tt_gbdt_workspace_bytes(n, F, max_depth).
 * tt_gbdt_update: pred += lr * incr; g = y - pred (incr = NULL: g = y - pred).
 * tt_gbdt_predict: out[r] = (accumulate ? out[r] : base) + sum over trees in
 *   order of lr * leaf (one round-to-nearest add per tree, gbdt.py:242-244);
 *   trees concatenated with d_tree_offsets[t] = first node of tree t
 *   (child indices are tree-local); X row-major (col_major = 0) or
 *   column-major. */
size_t tt_gbdt_workspace_bytes(int64_t n, int32_t n_features, int32_t max_depth);
int tt_gbdt_grow(const double *d_Xc, const double *d_g, const int32_t *d_root_order, int64_t n,
                 int32_t n_features, int32_t max_depth, int32_t min_samples_leaf, int32_t *d_feature,
                 double *d_threshold, int32_t *d_left, int32_t *d_right, double *d_value,
                 int32_t *d_node_count, double *d_incr, void *d_ws, size_t ws_bytes,
                 tt_stream_t stream);
int tt_gbdt_update(double *d_pred, const double *d_incr, const double *d_y, double *d_g, double lr,
                   int64_t n, tt_stream_t stream);
int tt_gbdt_predict(const int32_t *d_feature, const double *d_threshold, const int32_t *d_left,
                    const int32_t *d_right, const double *d_value, const int64_t *d_tree_offsets,
                    int32_t n_trees, double base, double lr, const double *d_X, int64_t n,
                    int32_t n_features, int32_t col_major, double *d_out, int32_t accumulate,
                    tt_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TT_B200_H */
