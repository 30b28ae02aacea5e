/*
 * autobyte.h — C ABI of the B200-native AutoByte meta-network candidate scorer.
 *
 * The library implements ONE hot path of "AutoByte: Automatic Configuration for Optimal
 * Communication Scheduling in DNN Training" (arXiv 2112.13509): the Meta Network Optimizer.
 * Citations: P:n = line n of the paper's LaTeX source; R#n = reading n of
 * DESIGN.md §3 (where the paper is silent, garbled or ambiguous).
 *
 *   f : (T, B, S_c, S_p) -> V                        (Eq. 1)
 *   "select the optimal pair with the maximum training speedup at the cost of one
 *    inference"
 *   L(V, V_bar) = || V - V_bar ||_2, online adaptation by transfer learning
 *                                                     (Eq. 2)
 *
 * Conventions that hold for every entry point unless stated otherwise:
 *  - Status: every call returns an autobyte_status; AB_OK == 0, errors are negative.
 *    Host-side checks (sizes, ranges of descriptors, NULL pointers) fail synchronously
 *    with NO kernel launched and no state changed. autobyte_last_error(ctx) returns a
 *    human-readable reason for the last failure on that ctx.
 *  - Pointers: "DEVICE" pointers must be device memory on the ctx's device (e.g. torch
 *    CUDA tensors); "HOST" pointers are ordinary host memory. All arrays are dense,
 *    row-major, naturally aligned, and owned by the caller for the duration of the call.
 *  - Asynchrony: device-pointer calls enqueue work on the ctx stream and return without
 *    synchronising; results are valid once that stream reaches them. *_host calls and
 *    autobyte_get_weights synchronise the ctx stream before returning.
 *  - Data-dependent ranges (n_workers in 1..n_max, n_layers in 1..l_max, type ids in
 *    range, partition sizes >= 4096, credit >= 1, bandwidth > 0) are the caller's
 *    contract; they are checked on the device only when the environment variable
 *    AUTOBYTE_CHECK=1 is set at autobyte_create time (then violations return
 *    AB_E_INVALID from the next call). Otherwise out-of-range data is undefined behaviour.
 *  - Threading: a ctx serves one stream and is not thread-safe. Score/argmax only read
 *    the weights; adapt mutates them in stream order.
 *  - No CPU fallback: without a usable sm_100a device, autobyte_create fails with
 *    AB_E_CUDA / AB_E_UNSUPPORTED.
 *  - Watchdogs: no kernel traps. An internal wait that exceeds its limit records a code in a
 *    device-wide status word and the kernel runs to its end with invalid results; the next call on
 *    any ctx of that device (or autobyte_synchronize / a *_host call, after its own kernels) returns
 *    AB_E_CUDA (pipeline watchdog) or AB_E_NCCL (peer timeout) once, with the reason in
 *    autobyte_last_error, and the CUDA context stays usable.
 */
#ifndef AUTOBYTE_H_
#define AUTOBYTE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AUTOBYTE_ABI_VERSION 1
#define AUTOBYTE_BLOB_MAGIC "ABYT"
#define AUTOBYTE_BLOB_VERSION 1u
#define AUTOBYTE_X_DIM 82      /* job feature vector x_j (R#4-R#8): 32 + 16 + 16 + 2 + 8 + 8 */
#define AUTOBYTE_U_DIM 2       /* candidate encoding u_c (R#8) */

typedef struct autobyte_ctx autobyte_ctx;   /* opaque; owned by the library */

typedef enum {
  AB_OK = 0,
  AB_E_INVALID = -1,       /* bad argument value / NULL pointer / bad blob / device data check */
  AB_E_SHAPE = -2,         /* inconsistent sizes (J, P, Q, shard, blob length) */
  AB_E_CUDA = -3,          /* CUDA runtime error (message in autobyte_last_error) */
  AB_E_NCCL = -4,          /* NCCL error */
  AB_E_NONFINITE = -5,     /* non-finite weights in a blob */
  AB_E_UNSUPPORTED = -6,   /* valid request this build does not implement (e.g. precision) */
  AB_E_NOMEM = -7          /* allocation failure */
} autobyte_status;

typedef enum {
  AB_PREC_BF16 = 0,   /* bf16 tensor-core operands, fp32 accumulate (parity 2e-2, R#16) */
  AB_PREC_FP32 = 1    /* split-operand bf16x3 emulation of fp32 products (parity 1e-4); every H */
} autobyte_precision;

/* Shape of the meta-network (R#1-R#6). Supported: hidden_layers (L) in 1..8,
 * hidden_width (H) in {64, 128, 256, 512}, n_max == 16, embed_dim == 16, lstm_hidden == 32,
 * n_model_types in 1..64, n_arch_types in 1..16, type_embed_dim == 8. */
typedef struct {
  int32_t hidden_layers;    /* L: hidden ReLU layers of width H after the concatenation */
  int32_t hidden_width;     /* H */
  int32_t n_max;            /* worker slots of Table 2's n x 1 vectors (R#7) */
  int32_t embed_dim;        /* d_e of the per-layer embedding of T (R#4) */
  int32_t lstm_hidden;      /* h of both LSTM layers (R#5) */
  int32_t n_model_types;    /* rows of the model-type embedding E_m (R#6) */
  int32_t n_arch_types;     /* rows of the architecture embedding E_arc (R#6) */
  int32_t type_embed_dim;   /* columns of E_m / E_arc (R#6) */
} autobyte_net_desc;

/* Table 2 runtime statistics of J jobs. */
typedef struct {
  int32_t J;                 /* number of jobs, >= 1 */
  int32_t l_max;             /* layer stride of T, >= 1 */
  const float*   T;          /* [J][l_max][n_max] layer-wise BP time in ms; entries of
                                layers >= n_layers[j] or workers >= n_workers[j] are ignored;
                                16-byte aligned (else AB_E_INVALID, no launch) */
  const float*   B_down;     /* [J][n_max] download Gbps (> 0 for valid workers) */
  const float*   B_up;       /* [J][n_max] upload Gbps (> 0 for valid workers) */
  const int32_t* n_workers;  /* [J] in 1..n_max */
  const int32_t* n_layers;   /* [J] in 1..l_max */
  const int32_t* model_type; /* [J] in 0..n_model_types-1 */
  const int32_t* arch_type;  /* [J] in 0..n_arch_types-1 (0 = PS, 1 = all-reduce) */
} autobyte_job_stats;

/* Candidate grid <S_p, S_c>: C = P*Q candidates, global index
 * c = p*Q + q, so ascending c = smaller partition first, then smaller credit (R#11).
 * This rank scores c in [shard_begin, shard_end); returned indices are global. */
typedef struct {
  int32_t P, Q;                    /* >= 1 each, P*Q <= 2^31 - 129 (AB_E_SHAPE); per call also
                                      J * ceil((shard_end - shard_begin) / 128) < 2^31 */
  const int64_t* partition_bytes;  /* [P] strictly ascending, >= 4096 */
  const float*   credit_mult;      /* [Q] strictly ascending, >= 1 (R#9) */
  int64_t shard_begin, shard_end;  /* 0 <= begin < end <= P*Q */
} autobyte_grid;

/* Per-kernel timing collected while profiling is enabled (CUDA events on the ctx stream). */
typedef struct {
  double  encode_ms;   int64_t encode_launches;    /* K1 job encoder */
  double  score_ms;    int64_t score_launches;     /* K2 fused tcgen05 MLP + arg-max */
  double  finalize_ms; int64_t finalize_launches;  /* K5 key decode */
  double  exchange_ms; int64_t exchange_calls;     /* K3 NCCL all-reduce(max) of keys */
  double  adapt_ms;    int64_t adapt_launches;     /* K4 fused forward/backward/SGD */
  double  pack_ms;     int64_t pack_launches;      /* bf16 weight re-pack after adapt */
  int64_t other_launches;                          /* every other kernel of this library */
  double  score_pairs;                             /* (job, candidate) pairs scored by K2 */
} autobyte_profile;

/* ---- library / host-only helpers (no device needed) ------------------------------- */
int32_t     autobyte_abi_version(void);
const char* autobyte_status_string(autobyte_status s);
/* Validate a net descriptor against the supported set above. */
autobyte_status autobyte_validate_desc(const autobyte_net_desc* desc);
/* Size in bytes of the weight blob for desc: 48-byte header + fp32 arrays. */
autobyte_status autobyte_blob_bytes(const autobyte_net_desc* desc, size_t* out_bytes);
/* Validate a HOST weight blob: magic "ABYT", version, descriptor equal to desc, length,
 * finite values (AB_E_NONFINITE otherwise).
 * Blob layout (little endian): char magic[4]; uint32 version; autobyte_net_desc desc;
 * uint32 n_arrays; uint32 reserved; then fp32 arrays back to back in the order
 * E_m[n_model_types][te], E_arc[n_arch_types][te], W_e[de][n_max], b_e[de],
 * lstm1_Wx[4h][de], lstm1_Wh[4h][h], lstm1_b[4h], lstm2_Wx[4h][h], lstm2_Wh[4h][h],
 * lstm2_b[4h], W1[H][84], b1[H], {W_k[H][H], b_k[H]} for k = 2..L, W_o[n_max][H], b_o[n_max].
 * LSTM gate order i, f, g, o (R#5); W1's last two columns multiply u_c (R#8). */
autobyte_status autobyte_validate_blob(const autobyte_net_desc* desc, const void* blob, size_t blob_bytes);

/* ---- context ---------------------------------------------------------------------- */
/* Create a ctx on `device` using `cuda_stream` (a cudaStream_t; NULL = legacy default
 * stream). Copies the HOST blob to device fp32 master weights and builds the bf16
 * tensor-core shadows. Fails with AB_E_UNSUPPORTED if the device is not sm_100 or the
 * (desc, precision) pair is not implemented. */
autobyte_status autobyte_create(const autobyte_net_desc* desc, const void* weight_blob,
                                size_t blob_bytes, int device, void* cuda_stream,
                                autobyte_precision precision, autobyte_ctx** out_ctx);
void            autobyte_destroy(autobyte_ctx* ctx);
const char*     autobyte_last_error(const autobyte_ctx* ctx);
autobyte_status autobyte_synchronize(autobyte_ctx* ctx);

/* ---- multi-GPU (candidate-axis sharding) ----------------------------- */
/* Fill 128 bytes with a fresh NCCL unique id (rank 0 calls it and broadcasts the bytes). */
autobyte_status autobyte_get_unique_id(void* out_128_bytes);
/* Join a world of `world` ranks (one per GPU; collective: every rank calls it). Shards of a
 * multi-rank partition may be empty (C < world): such a rank scores nothing but joins the
 * exchange. A peer wait that exceeds AUTOBYTE_PEER_TIMEOUT_S seconds (default 120, 0 = forever)
 * makes that call's results invalid and the next call (or autobyte_synchronize) return AB_E_NCCL;
 * nothing traps, the ctx stays usable. Calls may be captured into CUDA graphs (the exchange epoch
 * is a device counter; the opt-in AUTOBYTE_PEER_X gather falls back to NCCL while capturing);
 * capture only after one eager call of the same shapes (workspaces are allocated on first use),
 * and destroy such graphs before autobyte_destroy (captured NCCL work holds the communicator).
 * After this,
 * autobyte_argmax exchanges the per-job best keys so every rank returns the global result;
 * shards must partition [0, C) across ranks. world == 1 detaches.
 * Exchange (§8(a) a-7): by default every rank maps the other ranks' key windows through CUDA
 * IPC and ONE kernel stores its keys into all windows over NVLink, raises an epoch flag in each,
 * waits for every rank's flag and takes the per-job max (exchange.cu); jobs beyond the window
 * capacity (AUTOBYTE_PEER_JOBS, default 65536) or AUTOBYTE_EXCHANGE=nccl use ncclAllGather + a
 * max kernel, AUTOBYTE_EXCHANGE=allreduce uses ncclAllReduce(max). The ranks agree on the mode
 * (all mappings must succeed). Results are bit-identical in every mode and for any world. */
autobyte_status autobyte_attach_comm(autobyte_ctx* ctx, const void* unique_id_128, int rank, int world);
/* 1 if the NVLink peer-memory key exchange is active for this ctx, 0 otherwise (no comm, world 1,
 * NCCL mode, or a rank could not map a peer window). */
int32_t autobyte_peer_exchange(const autobyte_ctx* ctx);

/* ---- the hot path (DEVICE pointers, asynchronous) ---------------------------------- */
/* Encoder only: x[J][82] fp32 job feature vectors (P:402 components 1-3; "turn
 * those metrics to vector inputs"). */
autobyte_status autobyte_encode(autobyte_ctx* ctx, const autobyte_job_stats* jobs, float* x_out);

/* Predicted speed s[j][c] = mean_{w < n_j} V_hat_w(x_j, u_c) (Eq. 1; R#3) of every job
 * against this rank's shard: scores is [J][shard_end - shard_begin] fp32, column
 * c - shard_begin. */
autobyte_status autobyte_score(autobyte_ctx* ctx, const autobyte_job_stats* jobs,
                               const autobyte_grid* grid, float* scores);

/* Per-job best candidate: best_idx[j] = the global c maximising s[j][c], ties to the
 * smallest c (R#11); NaN scores never win; a job whose scores are all NaN gets -1 and a NaN
 * best_score. cur_idx (nullable) gives each job's current global configuration; cur_score[j]
 * receives s[j][cur_idx[j]] (NaN when cur_idx is NULL) for the 5% gain trigger.
 * best_idx, best_score, cur_score are [J] each; cur_score may be NULL. */
autobyte_status autobyte_argmax(autobyte_ctx* ctx, const autobyte_job_stats* jobs,
                                const autobyte_grid* grid, const int32_t* cur_idx,
                                int32_t* best_idx, float* best_score, float* cur_score);

/* The per-shard half of autobyte_argmax, for callers that reduce across ranks themselves (the
 * north star's "per-shard (score, index) bests ... reduced with an NCCL allgather"): runs the same
 * encoder and K2 as autobyte_argmax on this rank's shard and writes the 2J arg-max keys, DEVICE
 * keys_out[2J] u64, without any cross-rank exchange: keys_out[j] = max over this shard of
 * ord32(s[j][c]) << 32 | (2^32 - 1 - c) (0 when no score is a number), keys_out[J + j] = the same key
 * of the current configuration cur_idx[j] when this shard holds it, else 0 (cur_idx may be NULL).
 * ord32 is the order-preserving map of fp32 onto u32 (NaN -> 0), so the max of the keys is the
 * best score with ties to the smaller global c (R#11). With a communicator attached the encoder
 * is still sharded over the ranks (collective). Errors as autobyte_argmax. */
autobyte_status autobyte_argmax_keys(autobyte_ctx* ctx, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                                     const int32_t* cur_idx, uint64_t* keys_out);
/* Decode G blocks of such keys (DEVICE keys[G][2J], e.g. the result of an all-gather of every
 * rank's autobyte_argmax_keys) into best_idx / best_score / cur_score [J] (DEVICE; cur_score
 * nullable) exactly as autobyte_argmax does after its own exchange: the per-job max over the G
 * blocks, -1 / NaN for a job with no valid score. J, G >= 1 (else AB_E_SHAPE, no launch). The max
 * is order-free, so any partition of the grid gives the single-rank result bit for bit. */
autobyte_status autobyte_reduce_keys(autobyte_ctx* ctx, int32_t J, int32_t G, const uint64_t* keys,
                                     int32_t* best_idx, float* best_score, float* cur_score);

/* Per-job top-k candidates (R#19): idx[j][i] / score[j][i] (i < k, [J][k]
 * each, DEVICE) are the i-th best global candidate of job j over the grid — descending score,
 * ties to the smaller c (R#11), NaN never selected, (-1, NaN) padding when fewer than k scores
 * are valid; idx[j][0] == autobyte_argmax's best_idx. 1 <= k <= 32 (else AB_E_INVALID, no
 * launch). Scores the shard like autobyte_score (the [J][shard] matrix lives in a context
 * workspace), selects per job, and at G > 1 all-gathers the per-rank lists (J*k u64 per rank)
 * and merges them, so every rank returns the same, shard-layout-independent result. */
autobyte_status autobyte_topk(autobyte_ctx* ctx, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                              int32_t k, int32_t* idx, float* score);

/* Online adaptation (R#12, R#13): `steps` plain-SGD steps with learning
 * rate lr on the minibatch of B = samples->J observations: sample b has job statistics
 * samples[b], observed configuration (sp_bytes[b], sc_mult[b]) and observed per-worker speed
 * v_obs[b][n_max] (Eq. 2's V_bar). Objective (1/B) sum_b 1/2 ||mask_b (V_hat_b - V_bar_b)||^2,
 * head parameters only (W1, b1, W_k, b_k, W_o, b_o); encoder frozen. loss_before (nullable,
 * DEVICE [1] fp32) receives (1/B) sum_b ||mask_b (V_hat_b - V_bar_b)||_2 before the first step.
 * steps == 0 is a no-op apart from loss_before. The bf16 shadows are refreshed in stream
 * order, so the next score/argmax sees the adapted weights. Deterministic. */
autobyte_status autobyte_adapt(autobyte_ctx* ctx, const autobyte_job_stats* samples,
                               const int64_t* sp_bytes, const float* sc_mult, const float* v_obs,
                               float lr, int32_t steps, float* loss_before);

/* Offline training of the head ("offline training, online adapting"; R#18;
 * SURVEY §8(f) NEXT 2): `steps` optimiser steps on one minibatch, same inputs, objective,
 * frozen encoder and head scope as autobyte_adapt.
 *   AB_OPT_SGD:  theta <- theta - lr * g
 *   AB_OPT_ADAM: t <- t + 1; m <- beta1 m + (1 - beta1) g; v <- beta2 v + (1 - beta2) g^2;
 *                theta <- theta - (lr / (1 - beta1^t)) * m / (sqrt(v) / sqrt(1 - beta2^t) + eps)
 * The Adam moments m, v (fp32, one per head parameter) and the step count t live in the
 * context and carry across calls (autobyte_reset_optimizer zeroes them); autobyte_adapt does not
 * touch them. losses (nullable, DEVICE [steps] fp32) receives, per step, the mean Eq. 2 norm
 * (1/B) sum_b ||mask_b (V_hat_b - V_bar_b)||_2 before that step's update. Errors: NULL opt or
 * input pointer, steps < 0, non-finite lr, beta outside [0, 1) or eps <= 0 -> AB_E_INVALID with
 * no launch. Deterministic (fixed summation order); the bf16 shadows are refreshed in stream
 * order. */
typedef enum { AB_OPT_SGD = 0, AB_OPT_ADAM = 1 } autobyte_opt_kind;
typedef enum { AB_SCOPE_HEAD = 0, AB_SCOPE_ALL = 1 } autobyte_train_scope;
typedef struct {
  int32_t kind;    /* autobyte_opt_kind */
  float lr;
  float beta1;     /* Adam only; typical 0.9 */
  float beta2;     /* Adam only; typical 0.999 */
  float eps;       /* Adam only; typical 1e-8 */
  int32_t scope;   /* autobyte_train_scope: AB_SCOPE_ALL also fine-tunes the encoder (SURVEY NEXT 4,
                      R#20) by back-propagation through time of the LSTM; the samples are then
                      re-encoded every step (single-rank semantics; replicas stay identical) */
} autobyte_optimizer;
autobyte_status autobyte_train(autobyte_ctx* ctx, const autobyte_job_stats* samples,
                               const int64_t* sp_bytes, const float* sc_mult, const float* v_obs,
                               const autobyte_optimizer* opt, int32_t steps, float* losses);
/* Offline training over a dataset ("360000 iterations" of collected runtime samples;
 * P:418-423 "offline training"; R#18; SURVEY §8(f) NEXT 2 at scale): `steps` optimiser steps, step s
 * on the minibatch of the `batch` dataset rows order[s][0..batch). dataset (J = N samples),
 * sp_bytes / sc_mult [N] and v_obs [N][n_max] are the whole dataset (DEVICE); order is DEVICE int32
 * [steps][batch], every entry in [0, N) (caller's contract: the shuffle is an input, e.g. one
 * randperm per epoch; out-of-range entries are undefined behaviour). The samples are encoded once
 * (frozen encoder), then ONE kernel runs all steps: per step it gathers the minibatch rows, runs
 * forward, backward and the optimiser exactly as autobyte_train does on that minibatch (same
 * objective, head scope, Adam state carried in the context). losses (nullable, DEVICE [steps]) gets
 * each step's mean Eq. 2 norm before its update. opt->scope must be AB_SCOPE_HEAD
 * (AB_E_UNSUPPORTED otherwise); other errors as autobyte_train. Deterministic. */
autobyte_status autobyte_train_epoch(autobyte_ctx* ctx, const autobyte_job_stats* dataset, const int64_t* sp_bytes,
                                     const float* sc_mult, const float* v_obs, const int32_t* order,
                                     int32_t batch, int32_t steps, const autobyte_optimizer* opt, float* losses);
/* Zero the Adam moments and step count (asynchronous, stream-ordered). */
autobyte_status autobyte_reset_optimizer(autobyte_ctx* ctx);
/* Adam step count t so far (host value; no synchronisation). */
int64_t autobyte_optimizer_step(const autobyte_ctx* ctx);

/* Optimization Trigger, per job j, DEVICE pointers, [J] each:
 *   1. drift first: v_observed[j] > 0 and |cur_score - v_observed| / v_observed > drift
 *      -> action 2 (adapt, then decide again)
 *   2. gain: best_idx != cur_idx, best_idx >= 0 and
 *      best_score - cur_score > gain * |cur_score|                  -> action 1 (reconfigure)
 *   3. otherwise                                                      -> action 0 (keep)
 * Gain is predicted-vs-predicted (both scores from one autobyte_argmax call). v_observed (the
 * measured mean speed of the current configuration over the last 10-iteration group)
 * may be NULL (no drift check). NaN inputs never trigger an action. Paper defaults: gain = 0.05,
 * drift = 0.10. */
autobyte_status autobyte_trigger(autobyte_ctx* ctx, int32_t J, const int32_t* best_idx, const float* best_score,
                                 const int32_t* cur_idx, const float* cur_score, const float* v_observed,
                                 float gain, float drift, int32_t* action);

/* Ground-truth evaluator of the candidates (PAPER.md:213-255 mechanism,
 * PAPER.md:534 grid search): the time of ONE training iteration of every job under every <S_p, S_c>
 * of this rank's shard, simulated event by event, one GPU thread per (job, candidate):
 *   - backward from the back layer: layer i's gradient is ready at sum_{k >= i} Tb[k], Tb[i] = the
 *     slowest valid worker's T[i][w] (R#26);
 *   - partitioning: a tensor of size b bytes becomes ceil(b / S_p) chunks;
 *   - priority: the sender commits the next chunk of the front-most ready layer;
 *   - credit: committed-but-unacknowledged chunks total at most S_c * S_p bytes and 64 chunks
 *     (R#24);
 *   - one link sends committed chunks in commit order, s * factor / bw + delta ms each, acknowledged
 *     alpha ms later; factor 2 for PS (push + pull), 2 (n - 1) / n for ring all-reduce; bw = the
 *     smallest B_down / B_up of the valid workers (R#25, R#26);
 *   - the next forward runs front to back, layer i once its tensor is acknowledged.
 * layer_bytes: DEVICE [J][l_max] fp32 tensor bytes per layer (not part of Table 2; model-profile
 * input). fwd_ms: DEVICE [J][l_max] forward time per layer, or NULL for Tb / 2 (R#26). sp: HOST.
 * iter_ms: DEVICE [J][shard_end - shard_begin] float64, column c - shard_begin. The iteration time is
 * within 1e-12 relative of the float64 oracle (same operations; the forward pass as its max-plus
 * form). Errors: as autobyte_score; negative or non-finite alpha / delta -> AB_E_INVALID; l_max too
 * large for the per-thread state (> ~590 layers) -> AB_E_SHAPE. */
typedef struct {
  double alpha_ms;   /* per-chunk latency until acknowledgement (what stop-and-wait loses) */
  double delta_ms;   /* per-chunk partition / scheduling overhead on the link */
} autobyte_sim_params;
autobyte_status autobyte_simulate(autobyte_ctx* ctx, const autobyte_job_stats* jobs, const float* layer_bytes,
                                  const float* fwd_ms, const autobyte_grid* grid, const autobyte_sim_params* sp,
                                  double* iter_ms);

/* ---- end-to-end entry points (HOST pointers; copies inside; synchronising) ---------- */
/* Same contracts as above with every array pointer in HOST memory. The library stages the
 * inputs into its own device workspace with cudaMemcpyAsync, runs the device path, copies
 * the [J] results back and synchronises the ctx stream. With a communicator attached
 * (world > 1) every rank still passes the full job arrays, but only the statistics of the
 * jobs its own encoder shard reads (T, B_down, B_up, n_layers, model_type, arch_type of
 * ceil(J/world) jobs) are copied; n_workers is copied for all jobs. AUTOBYTE_CHECK=1 copies
 * everything (the range checks read every job). Arrays in page-locked (pinned /
 * registered) host memory that one kernel reads once are not staged but read in place over PCIe:
 * T, B_down, B_up, n_layers, model_type, arch_type (by the encoder kernel, so the transfer of T
 * overlaps the LSTM steps), the grid's partition_bytes / credit_mult (by the grid encoder) and
 * adapt's sp_bytes / sc_mult / v_obs (by the adaptation kernel). n_workers and cur_idx are always
 * copied. AUTOBYTE_ZERO_COPY=0 stages everything. The caller must not modify the inputs until the
 * call returns, which it does only after the results are on the host. */

/* Host-to-device bytes the staging above moves for the job statistics of J jobs with
 * l_max layers on this rank (the e2e accounting of bench.py). Returns 0 for a NULL ctx. */
size_t autobyte_staged_job_bytes(const autobyte_ctx* ctx, int32_t J, int32_t l_max);
autobyte_status autobyte_argmax_host(autobyte_ctx* ctx, const autobyte_job_stats* jobs,
                                     const autobyte_grid* grid, const int32_t* cur_idx,
                                     int32_t* best_idx, float* best_score, float* cur_score);
autobyte_status autobyte_adapt_host(autobyte_ctx* ctx, const autobyte_job_stats* samples,
                                    const int64_t* sp_bytes, const float* sc_mult,
                                    const float* v_obs, float lr, int32_t steps,
                                    float* loss_before);

/* ---- weights / checkpoint ----------------------------------------------------------- */
/* Write the current fp32 master weights as a blob (same layout as autobyte_validate_blob)
 * into HOST memory of exactly autobyte_blob_bytes() bytes. Synchronises the ctx stream.
 * create(blob) -> get_weights round-trips bit-identically. */
autobyte_status autobyte_get_weights(autobyte_ctx* ctx, void* host_blob, size_t blob_bytes);

/* ---- profiling ------------------------------------------------------------------------ */
/* enable != 0: bracket every kernel launch with CUDA events on the ctx stream and
 * accumulate per-kernel device time (adds a stream-ordered event pair per launch).
 * autobyte_get_profile synchronises the ctx stream and reads the totals; reset zeroes them. */
autobyte_status autobyte_set_profiling(autobyte_ctx* ctx, int enable);
autobyte_status autobyte_get_profile(autobyte_ctx* ctx, autobyte_profile* out);
autobyte_status autobyte_reset_profile(autobyte_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* AUTOBYTE_H_ */
