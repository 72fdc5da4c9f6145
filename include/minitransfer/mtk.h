/*
 * mtk.h -- C ABI of the B200 (sm_100a) shadow-training / MMD / membership-
 * attack path.  Plain pointers and sizes only; no torch or C++ types.
 *
 * The reference (/root/reference/proj/include/minitransfer) exposes this path
 * only as a C++ header API in namespace mt (Tape ops + optimizer_step); it has
 * no FFI.  Each entry point below names the reference composition it replaces
 * (file:line).  The C++ wrapper include/minitransfer/gpu.hpp maps the status
 * codes back onto the reference exception classes (error.hpp:10-51).
 *
 * Conventions
 *   - status codes (error.hpp:10-51):
 *       0 OK, 1 ShapeError, 2 ValueError, 3 ConfigError, 4 DataError,
 *       5 Error (internal / CUDA / non-finite).
 *     mtk_last_error() returns the calling thread's message for the last
 *     failing call.
 *   - Arrays named X / y / w / logits / feats / scores / g* are DEVICE
 *     pointers owned by the caller, unless the name ends in _host.
 *     Host-side double arrays (parameters, metrics) are marked "host".
 *   - Calls are stream-ordered on the context's stream and asynchronous,
 *     except those that return host scalars (they synchronize).  Deferred
 *     device-side errors (out-of-range label, non-finite value) are reported
 *     by the next synchronizing call on the same context.
 *   - Row-major fp32 on the device; f64 on the host at the parity API.
 */
#ifndef MINITRANSFER_MTK_H
#define MINITRANSFER_MTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTK_OK 0
#define MTK_SHAPE_ERROR 1
#define MTK_VALUE_ERROR 2
#define MTK_CONFIG_ERROR 3
#define MTK_DATA_ERROR 4
#define MTK_ERROR 5
/* checkpoint load failures (error.hpp:34-46: CheckpointError and its
 * VersionError / DigestError / TruncatedError subclasses of DataError)      */
#define MTK_CHECKPOINT_ERROR 6
#define MTK_VERSION_ERROR 7
#define MTK_DIGEST_ERROR 8
#define MTK_TRUNCATED_ERROR 9

typedef struct mtk_ctx mtk_ctx;
typedef struct mtk_bank mtk_bank;
typedef struct mtk_rng mtk_rng;

int mtk_version(void);
const char* mtk_last_error(void);

/* ---- context: one per (host thread, device); mirrors "one Tape per thread"
 * (tape.hpp:84-85).  All work is ordered on `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream).                                       */
int mtk_ctx_create(int device, void* cuda_stream, mtk_ctx** out);
int mtk_ctx_destroy(mtk_ctx* ctx);
int mtk_ctx_synchronize(mtk_ctx* ctx);
/* number of kernels this library has launched in this process (all of the
 * path's kernels are the library's own; no library sort / scan is used)    */
int mtk_ctx_launch_count(mtk_ctx* ctx, uint64_t* out);
/* Optional CUDA-event timing of the bank step's phases, on the ctx stream.
 * mtk_ctx_phase_times synchronizes and returns (then resets) the summed
 * milliseconds and launch counts per phase, MTK_NUM_PHASES entries, in the
 * order: fwd_gemm, ce, mmd_beta, mmd_pairs, dx_gemm, dw_gemm, bias_sgd, other,
 * side_stream.  side_stream is the wall time of the launch groups on the ctx's
 * side stream (MMD prep pass, bias updates, skinny head dW), which overlap
 * the main-stream phases, waiting included. */
#define MTK_NUM_PHASES 9
int mtk_ctx_set_timing(mtk_ctx* ctx, int on);
int mtk_ctx_phase_times(mtk_ctx* ctx, double* ms_host, uint64_t* launches_host);

/* ---- host RNG: bit-exact restatement of mt::Rng (rng.hpp:13-75) --------- */
int mtk_rng_create(uint64_t seed, mtk_rng** out);
int mtk_rng_destroy(mtk_rng* r);
int mtk_rng_split(mtk_rng* parent, uint64_t stream, mtk_rng** out); /* rng.hpp:65-69 */
uint64_t mtk_rng_next_u64(mtk_rng* r);                             /* rng.hpp:17 */
double mtk_rng_uniform(mtk_rng* r, double lo, double hi);           /* rng.hpp:22 */
double mtk_rng_normal(mtk_rng* r);                                  /* rng.hpp:24-37 */
uint64_t mtk_rng_below(mtk_rng* r, uint64_t n);                     /* rng.hpp:39-46 */
int mtk_rng_permutation(mtk_rng* r, uint64_t n, uint64_t* out_host); /* rng.hpp:58-63 */
int mtk_rng_fill_normal(mtk_rng* r, double* out_host, uint64_t n);
/* class-conditional Gaussians: y = below(C); x = mu[y] + N(0,I) (+ shift).
 * X64_host (f64) and/or X32_host (fp32 copy) may be NULL.                  */
int mtk_synth(mtk_rng* r, int C, int d, uint64_t n, const double* mu_host,
              const double* shift_host, double* X64_host, float* X32_host, int32_t* y_host);

/* ---- counter-based synthetic data on the DEVICE.  Not
 * mt::Rng: a stateless Philox4x64-10 stream keyed by {seed, stream}, so a
 * pool of any size is generated in parallel straight into HBM.  Contract
 * (restated by oracle/oracle.c orc_synth_counter):
 *   normals: element e of a row-major [n, d] matrix <- counter {e/4,0,0,0};
 *     words (w0,w1) -> elements 4i, 4i+1, (w2,w3) -> 4i+2, 4i+3, Box-Muller
 *     with u1 = ((wa >> 40) + 1) 2^-24, u2 = (wb >> 40) 2^-24 (fp32 math);
 *   labels: row i <- word i%4 of counter {i/4,1,0,0}, y = (w * C) >> 64;
 *   X[i,k] = (mu[y_i,k] + z[i*d+k]) (+ shift[k]).
 * Raw words and labels are bit-exact against the oracle; normals agree to a
 * few fp32 ulps (libm vs device transcendental rounding).                  */
int mtk_philox4x64_fill(mtk_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t ctr0, uint64_t ctr1,
                        int64_t nblocks, uint64_t* out); /* out[4i..4i+3] = philox({ctr0+i,ctr1,0,0}) */
int mtk_counter_normals(mtk_ctx* ctx, uint64_t seed, uint64_t stream, int64_t first, int64_t count,
                        float* out);                      /* elements [first, first+count) */
/* mu [C, d] and shift [d] (or NULL) fp32 device; X [n, d] fp32, y [n] int32 device */
int mtk_synth_counter(mtk_ctx* ctx, uint64_t seed, uint64_t stream, int C, int d, int64_t n,
                      const float* mu, const float* shift, float* X, int32_t* y);

/* ---- model bank: G independent MLPs dims[0] -> ... -> dims[n_layers], ReLU
 * hidden layers, trained as ONE grouped step.  Replaces, per model, the Tape
 * composition matmul (tape.hpp:225-290) -> add_bias (:204-221) -> relu
 * (:342-352) -> ... -> cross_entropy_weighted (:475-520) -> backward
 * (:870-886) -> optimizer_step SGD (optim.hpp:30-68).
 * n_heads == 2 (parameter-based paradigm): a second head of the same shape
 * as the last layer is stored as parameter matrix index n_layers; rows
 * [0, src_rows) use head 0, rows [src_rows, B) head 1.                      */
int mtk_bank_create(mtk_ctx* ctx, int G, int n_layers, const int* dims_host, int n_heads,
                    mtk_bank** out);
int mtk_bank_destroy(mtk_bank* bank);
/* W_host[i] is [fan_in, fan_out] row-major f64, b_host[i] is [fan_out], for
 * i in [0, n_layers + n_heads - 1).  Synchronizing.                         */
int mtk_bank_set_params(mtk_bank* bank, int model, const double* const* W_host,
                        const double* const* b_host);
int mtk_bank_get_params(mtk_bank* bank, int model, double* const* W_host, double* const* b_host);
/* SPEC.md:182 init drawn from r: W uniform(-1/sqrt(fan_in), 1/sqrt(fan_in))
 * row-major, matrices in index order; b = 0.                                */
int mtk_bank_init_params(mtk_bank* bank, int model, mtk_rng* r);
/* device views of parameter matrix i: W [G, fan_in, fan_out], b [G, fan_out] */
int mtk_bank_param_device(mtk_bank* bank, int mat, float** W, float** b);

/* forward only (posterior query): X [G,B,dims[0]] ->
 * logits [G,B,C] using head `head`; hidden_last [G,B,dims[n_layers-1]] or NULL */
int mtk_bank_forward(mtk_bank* bank, const float* X, int B, int head, float* logits,
                     float* hidden_last);

typedef struct {
    const float* X;     /* [G,B,dims[0]] device */
    const int32_t* y;   /* [G,B] device, labels in [0, C) */
    const float* w;     /* [G,B] device per-row CE weights, NULL = all 1 */
    int B;              /* rows per model */
    int src_rows;       /* rows [0,src_rows) = source; used by 2 heads and MMD */
    double denom[2];    /* CE denominators head 0 / head 1; 0 selects the row count,
                           negative is a ValueError (tape.hpp:485) */
    double lr;          /* SGD learning rate (optim.hpp:46-48) */
    int frozen_layers;  /* layers [0, frozen) keep bit-identical params */
    double mmd_lambda;  /* > 0: + lambda * MMD^2(h_src, h_tgt) on the last hidden layer */
    int mmd_nb;         /* bandwidth count (<= 8); 0 selects the 5-bandwidth default */
    double mmd_mult[8]; /* s_b = beta * mmd_mult[b], beta detached (closed form) */
    int optimizer;      /* 0 SGD (optim.hpp:46-48), 1 Adam (optim.hpp:49-63); the bank
                           keeps the Adam moments and step count (mtk_bank_reset_optimizer) */
    double adam_beta1;  /* 0 selects the reference default 0.9 (optim.hpp:19) */
    double adam_beta2;  /* 0 selects 0.999 */
    double adam_eps;    /* 0 selects 1e-8 */
} mtk_step;

/* One SGD step for all G models.  loss_host [G] (CE part) and mmd_host [G]
 * (MMD^2 value) are optional; passing either synchronizes.                  */
int mtk_bank_train_step(mtk_bank* bank, const mtk_step* step, double* loss_host,
                        double* mmd_host);
/* Same step from HOST buffers (X_host [G,B,d0] fp32, y_host [G,B], w_host or
 * NULL): the library stages them to the device on its stream.  Used for the
 * end-to-end measurement; step->X/y/w are ignored.                          */
int mtk_bank_train_step_host(mtk_bank* bank, const mtk_step* step, const float* X_host,
                             const int32_t* y_host, const float* w_host, double* loss_host,
                             double* mmd_host);
/* Pipelined variant: enqueue the step (H2D copy on a library copy stream into
 * one of two staging slots, overlapping the previous step's compute) and
 * return without waiting.  X_host / y_host / w_host should be pinned.
 * mtk_bank_step_result(which = 0) waits for the most recent enqueued step and
 * returns its per-model loss / MMD (which = 1: the one before it).          */
int mtk_bank_train_step_host_async(mtk_bank* bank, const mtk_step* step, const float* X_host,
                                   const int32_t* y_host, const float* w_host);
int mtk_bank_step_result(mtk_bank* bank, int which, double* loss_host, double* mmd_host);
/* which layers run their GEMMs on the tcgen05 3xTF32 path (1) vs the SIMT
 * path (0); out_host [n_layers].  Layers with both widths >= 32 and
 * multiples of 4 qualify (env MTK_DISABLE_TC=1 at bank creation forces SIMT). */
int mtk_bank_tc_layers(mtk_bank* bank, int* out_host);
/* zero the Adam moments and step count (a fresh mt::OptimizerState).       */
int mtk_bank_reset_optimizer(mtk_bank* bank);

/* ---- bank checkpoint / resume ------
 * Text header (magic, format_version, config, payload size, SHA-256 of the
 * payload) followed by length-prefixed named little-endian fp32 tensors:
 * W<i>, b<i> per matrix and, once Adam has run, its moments m/v and step.
 * load(save(bank)) is bit-exact, so training resumes identically.  Load
 * errors: VersionError (names both versions), DigestError, TruncatedError,
 * CheckpointError (malformed).                                             */
int mtk_bank_save(mtk_bank* bank, const char* path);
/* configuration of a bank (e.g. one made by mtk_bank_load); dims_out may be
 * NULL (else n_layers + 1 entries), any other pointer may be NULL.          */
int mtk_bank_info(mtk_bank* bank, int* G, int* n_layers, int* dims_out, int* n_heads);
int mtk_bank_load(mtk_ctx* ctx, const char* path, mtk_bank** out);
/* FIPS 180-4 SHA-256 of `len` bytes (host), 32 bytes out.                  */
int mtk_sha256(const void* data, size_t len, uint8_t* out32);
/* nsteps training steps without host round trips: step s gathers its batch
 * X[g, r] = X_pool[idx[s, g, r]] (and labels) on the device, then runs
 * mtk_bank_train_step with `tmpl` (B, lr, options), w = w + s*G*B (or NULL)
 * and denom[0] = denom0_host[s] (or tmpl's).  X_pool [pool_rows, dims[0]],
 * y_pool [pool_rows], idx (int64) [nsteps, G, B], w [nsteps, G, B] on the
 * device.  Synchronizing (reports bad labels / indices / non-finite).       */
int mtk_bank_train_epoch(mtk_bank* bank, const mtk_step* tmpl, const float* X_pool,
                         const int32_t* y_pool, int64_t pool_rows, const int64_t* idx,
                         const float* w, const double* denom0_host, int nsteps);

/* Batch assembly on the device (the sweep driver's batch_iter gather,
 * SPEC.md:605-613): out[g, row0 + r, :] = src[idx[g * nb + r], :] for
 * g < G, r < nb; src [src_rows, d] and idx (int64) [G, nb] on the device,
 * out has out_rows rows per model.  4-byte elements are copied bitwise, so
 * int32 labels use the same call with d = 1.  Bad indices -> ValueError at
 * the next synchronizing call.                                              */
int mtk_gather_rows(mtk_ctx* ctx, const void* src, int64_t src_rows, int d, const int64_t* idx,
                    int G, int nb, void* out, int out_rows, int row0);
/* debug/parity: keep the last step's parameter gradients (dW, db).          */
int mtk_bank_set_keep_grads(mtk_bank* bank, int on);
int mtk_bank_get_grads(mtk_bank* bank, int model, double* const* dW_host, double* const* db_host);

/* ---- data-parallel training of a replicated bank (dp_step).
 * The gradient ARENA is one flat fp32 array: for each parameter matrix i in
 * index order, dW_i [G, fan_in, fan_out] then db_i [G, fan_out], each
 * segment starting at a multiple of 32 floats (the size is one too, so
 * arenas stacked back to back stay 128-byte aligned).                      */
int mtk_bank_grad_size(mtk_bank* bank, int64_t* n_floats);
/* Forward + backward of `step` on this worker's shard (CE weights / denom as
 * in step: a shard of a global batch uses denom = its global_rows / n so the
 * mean-reduction algebra stays exact, tape.hpp:466-468) writing the gradients
 * to `grads` (device arena, 128-byte aligned).  Parameters and optimizer state are unchanged;
 * frozen matrices report zeros.  step->lr / optimizer are ignored here.     */
int mtk_bank_compute_grads(mtk_bank* bank, const mtk_step* step, float* grads, double* loss_host,
                           double* mmd_host);
/* The aggregation + one optimizer step: per element
 * g = ((parts[0] + parts[1]) + ... + parts[n-1]) / n in ascending worker
 * order (fixed, so every replica computes the same bits), then
 * SGD / Adam per step->optimizer on every non-frozen parameter.  parts:
 * device, n_parts arenas part_stride floats apart (an all-gather output).  */
int mtk_bank_dp_apply(mtk_bank* bank, const mtk_step* step, const float* parts, int n_parts,
                      int64_t part_stride);
/* Order-independent 64-bit hash of every parameter's bits (all models):
 * equal on bit-identical replicas; compared across workers before a step
 * ("replica divergence detected before step").  Synchronizing. */
int mtk_bank_fingerprint(mtk_bank* bank, uint64_t* out_host);

/* ---- multi-bandwidth Gaussian MMD^2 (no reference
 * code).  k(x,y) = sum_b exp(-|x-y|^2/(beta*mult[b])); beta <= 0 selects the
 * detached closed form over [Xs;Xt].  Biased V-statistic.  gXs/gXt (device,
 * optional) receive d MMD^2 / dX.  Synchronizing (returns host scalars).    */
int mtk_mmd_gaussian(mtk_ctx* ctx, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                     const double* mult_host, int nb, double beta, double* value_host,
                     double* beta_host, float* gXs, float* gXt);
/* Row-sharded form for multi-GPU: only pair rows i in [row_begin, row_end)
 * of the concatenated index space [Xs;Xt] are processed.  partial_host[3] =
 * raw kernel sums (ss, tt, st) over those rows; gradients are written only
 * for those rows.  beta must be given (> 0) so all shards agree.            */
int mtk_mmd_gaussian_rows(mtk_ctx* ctx, const float* Xs, int64_t m, const float* Xt, int64_t n,
                          int d, const double* mult_host, int nb, double beta, int64_t row_begin,
                          int64_t row_end, double* partial_host, float* gXs, float* gXt);
int mtk_mmd_beta(mtk_ctx* ctx, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                 double* beta_host);
/* Multi-GPU form on the materialised kernel matrix: the
 * rank owning the 128-row tiles [tile_begin, tile_end) of [Xs; Xt] (Xs, Xt
 * views of one [m + n, d] block, the gradients likewise) evaluates every
 * tile pair touching its tiles -- pairs of two of its tiles once, pairs with
 * another rank's tile by both ranks, each keeping only its own rows of W --
 * and writes the gradients of its rows.  tile_partials_host [T][3] (T =
 * ceil((m + n) / 128)) receives the kernel sums (ss, tt, st) of its tile
 * rows (zeros elsewhere).  Per element the arithmetic is the one-rank
 * call's, so gradients are bit-identical to mtk_mmd_gaussian, and so is the
 * value from mtk_mmd_value_from_tile_partials over the ranks' partials
 * (ascending tile rows, the one-rank finish's order).  Equal tile ranges
 * balance the ranks (each does s T - s^2 / 2 tile pairs for s tiles).     */
int mtk_mmd_gaussian_tiles(mtk_ctx* ctx, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                           const double* mult_host, int nb, double beta, int64_t tile_begin,
                           int64_t tile_end, double* tile_partials_host, float* gXs, float* gXt);
int mtk_mmd_value_from_tile_partials(const double* tile_partials_host, int64_t T, int64_t m, int64_t n,
                                     double* value_host);

/* ---- attack stage -------------------------------------------------------- */
/* Tape::softmax semantics (tape.hpp:433-464), fp32 out */
int mtk_softmax(mtk_ctx* ctx, const float* logits, int64_t rows, int C, float* probs);
/* top-k descending posteriors; with labels, one extra column = CE loss of
 * the true label.  feats [rows, k (+1)]                                     */
int mtk_posterior_features(mtk_ctx* ctx, const float* logits, int64_t rows, int C, int k,
                           const int32_t* labels, float* feats);
/* softmax probability of class `col` per row (attack score) */
int mtk_posterior_column(mtk_ctx* ctx, const float* logits, int64_t rows, int C, int col,
                         float* out);
/* Mann-Whitney AUC with mid-ranks for ties + accuracy at 0.5 (either output
 * may be NULL).  labels: 1 = member.  Synchronizing.                        */
int mtk_auc(mtk_ctx* ctx, const float* scores, const uint8_t* labels, int64_t n,
            double* auc_host, double* acc_host);
/* The whole attack evaluation of `rows` queried posteriors in one call:
 * softmax -> top-k sorted features (k = the attack bank's input width) ->
 * attack model (model 0 of `attack`, linear head) -> member probability
 * (softmax column 1) -> mid-rank AUC + accuracy at 0.5.  Same results as
 * mtk_posterior_features + mtk_bank_forward + mtk_posterior_column + mtk_auc
 * (bit-identical scores); the [3, 64, 2] attack model over <= 16 classes runs
 * as one streaming kernel, each CTA staging the weights from the bank in
 * shared memory, then one scan kernel for the AUC.  scores_out
 * (device, [rows]) may be NULL.  Synchronizing.  Stands in for the absent
 * reference attack stage.                   */
int mtk_attack_auc(mtk_bank* attack, const float* logits, int64_t rows, int C, const uint8_t* labels,
                   double* auc_host, double* acc_host, float* scores_out);

/* ---- the path's one collective: shadow models shard
 * across the GPUs of a box with no gradient exchange; after querying, the
 * ranks' posterior features are all-gathered so every rank trains the attack
 * model on all shadows.  NCCL (NVLink / NVSwitch) is loaded at run time
 * (libnccl.so.2; an already-loaded copy, e.g. torch's, is reused).
 * No reference counterpart: the reference is single-process. */
typedef struct mtk_comm mtk_comm;
/* a fresh NCCL unique id (128 bytes) on one rank; ship it to the others */
int mtk_comm_unique_id(void* out128);
/* collective over nranks processes (ncclCommInitRank), bound to the calling
 * thread's current CUDA device; every rank calls it with the same id.       */
int mtk_comm_init(int nranks, int rank, const void* nccl_id, mtk_comm** out);
int mtk_comm_destroy(mtk_comm* comm);
/* any pointer may be NULL; nccl_version as ncclGetVersion reports it        */
int mtk_comm_info(mtk_comm* comm, int* nranks, int* rank, int* device, int* nccl_version);
/* recv[r * bytes_per_rank ...] = rank r's `send` (device buffers), in rank
 * order; stream-ordered on ctx's stream (asynchronous).  ctx and comm must
 * be on the same device.                                                    */
int mtk_allgather(mtk_comm* comm, mtk_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank);

/* ---- the shadow-training sweep + membership attack in one native call
 * (the reference has no code
 * for it).  One paradigm: target (model 0) + n_shadows shadow models trained
 * as one bank per rank (contiguous model blocks; stream k+1 of Rng(seed) for
 * model k on every rank), top-k posterior features of each model on its
 * members / non-members, the ranks' features all-gathered (comm, or NULL for
 * one rank), an attack MLP k -> attack_hidden -> 2 trained on the shadows'
 * features, AUC (mid-rank Mann-Whitney) and accuracy at 0.5 on the target's.
 * Same definitions, call for call, as paper_2011_09463_b200/sweep.py (its
 * docstring pins them); results are identical on one device.              */
#define MTK_PARADIGM_MODEL 0     /* fine-tuning: pretrain on source, then members */
#define MTK_PARADIGM_MAPPING 1   /* CE on [source; members] + lambda MMD^2 on the hidden layer */
#define MTK_PARADIGM_PARAMETER 2 /* shared trunk + source head + target head */
#define MTK_SWEEP_MAX_LAYERS 8
typedef struct {
    int paradigm;
    int n_layers;                      /* dims[0..n_layers] */
    int dims[MTK_SWEEP_MAX_LAYERS + 1];
    int n_shadows, pool, members, source_pool, source_per_model;
    int batch, epochs, pretrain_epochs, frozen_layers;
    double lr;
    int optimizer;                     /* 0 SGD, 1 Adam */
    double mmd_lambda, mu_scale, shift_scale;
    int k, attack_hidden, attack_epochs, attack_batch;
    double attack_lr;
    int attack_optimizer;
    int data_rng;                      /* 0 host mt::Rng (bit-exact), 1 device Philox counter */
    uint64_t seed;
} mtk_sweep_config;
typedef struct {
    double auc, accuracy;
    int models, rank_model_begin, rank_model_end;
    int64_t n_queries;
    double seconds;
} mtk_sweep_result;
/* BASELINE.md C1 (the parity config): 784-256-10, 1 target + 4 shadows,
 * 2048 members of an 8192 pool, B = 128, E = 10, SGD lr 0.05, attack 3-64-2 */
void mtk_sweep_config_default(mtk_sweep_config* cfg);
int mtk_sweep_run(mtk_ctx* ctx, const mtk_sweep_config* cfg, mtk_comm* comm, mtk_sweep_result* out);

/* ---- diagnostics (tests / profiling): C[g] = A[g] * B[g] through the
 * tcgen05 3xTF32 tensor-core GEMM used by the bank.  a_mn: A stored
 * [G][K][M] (1) or [G][M][K] (0); b_mn: B stored [G][K][N] (1) or [G][N][K]
 * (0); C [G][M][N] fp32.  Synchronizing.                                    */
int mtk_diag_gemm_tf32x3(mtk_ctx* ctx, int a_mn, int b_mn, int G, int M, int N, int K,
                         const float* A, const float* B, float* C);

#ifdef __cplusplus
}
#endif
#endif
