/* ktune_cuda.h — C ABI of the B200-native Chameleon hot path (libktune_cuda.so).
 *
 * Drop-in boundary. Every entry point is `extern "C"`, takes
 * plain pointers and sizes, never throws, and returns an int status:
 *   KTUNE_OK (0) or one of the KTUNE_ERR_* codes below; the message is
 *   available from ktune_last_error(ctx) (thread-local when ctx is NULL).
 * The C++/Python adapters map the codes back onto the reference's exception
 * types: CONFIG -> ktune::ConfigError (errors.hpp:9-12), BACKEND/CUDA ->
 * ktune::BackendError (errors.hpp:15-18), EXHAUSTED -> SpaceExhaustedError
 * (errors.hpp:22-25), LOGIC -> std::logic_error (sampling.cpp:142-144).
 *
 * Pointers: unless KTUNE_F_DEVICE is set in `flags`, array arguments are HOST
 * pointers and the call is synchronous (it stages through the context's
 * pinned buffers). With KTUNE_F_DEVICE they are device pointers on the
 * context's device and the call is stream-ordered on the context stream
 * (ktune_ctx_set_stream); calls that need host-side decisions (k-means
 * convergence, the k sweep) synchronise the stream internally.
 *
 * Threading: a context is single-threaded; use one context per host thread
 * (uploaded objects are immutable and may be shared between contexts on the
 * same device — predict stays concurrently callable, cost_model.hpp:77-82).
 */
#ifndef KTUNE_CUDA_H
#define KTUNE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KTUNE_ABI_VERSION 1

enum ktune_status {
  KTUNE_OK = 0,
  KTUNE_ERR_CONFIG = 1,    /* ConfigError: bad argument / dimension mismatch / unfitted model */
  KTUNE_ERR_BACKEND = 2,   /* BackendError */
  KTUNE_ERR_EXHAUSTED = 3, /* SpaceExhaustedError */
  KTUNE_ERR_LOGIC = 4,     /* std::logic_error (Lloyd loss increased) */
  KTUNE_ERR_CUDA = 5,      /* CUDA runtime / launch failure (mapped to BackendError) */
  KTUNE_ERR_NOMEM = 6      /* device allocation failed (mapped to BackendError) */
};

enum ktune_flags {
  KTUNE_F_DEVICE = 1,       /* array arguments are device pointers */
  KTUNE_F_EXACT_ROLLOUT = 2, /* ktune_rollout: exact fp64 forward for every config-step (logp/value
                               bit-exact too); default is the tcgen05 path with certified sampling */
  KTUNE_F_STEP_MAJOR = 4,    /* ktune_rollout: trajectories step-major, idx/score [T+1][E], actions/logp/value
                               [T][E] (rows of D knobs where applicable), instead of episode-major [E][T+1] /
                               [E][T]: the device writes one coalesced row block per step, and every
                               segment of a host-pointer call crosses PCIe as one contiguous copy */
  KTUNE_F_STEP_MAJOR_GROUPED = 8 /* ktune_rollout: step-major over ALL tasks' episodes at once: every output
                               is one [T+1 or T][Etot = sum E_k] array (rows of D knobs; every task has the
                               same D) and task k passes pointers at its episode offset sum_{j<k} E_j of task
                               0's arrays; a segment of every task crosses PCIe as ONE copy per output */
};

typedef struct ktune_ctx ktune_ctx;
typedef struct ktune_space ktune_space;
typedef struct ktune_gbt ktune_gbt;
typedef struct ktune_ac ktune_ac;

/* ------------------------------------------------------------------ context */
int ktune_abi_version(void);
const char* ktune_last_error(const ktune_ctx* ctx);

/* One context per (host thread, device). Owns the stream, workspaces, pinned
 * staging buffers and (optionally) an NCCL communicator. */
int ktune_ctx_create(int device, ktune_ctx** out);
/* Distributed variant: rank/world of a one-process-per-GPU job; nccl_id is
 * the 128-byte ncclUniqueId from rank 0 (NULL when world == 1). */
int ktune_ctx_create_dist(int device, int rank, int world, const void* nccl_id, ktune_ctx** out);
int ktune_nccl_get_unique_id(void* out128);
/* Host-transport variant for multi-process runs without one GPU per rank (tests): the
 * library's collectives (the sharded k-means exchanges, the distributed CandidateSet
 * merge) call these instead of NCCL, on pinned HOST buffers, after synchronising the
 * context stream. allreduce: in-place sum of `count` elements (dtype 0 = int64/uint64,
 * 1 = float64); allgather: rank-ordered concatenation of every rank's `bytes`. Return 0
 * on success. */
typedef int (*ktune_host_allreduce_fn)(void* buf, int64_t count, int dtype, void* user);
typedef int (*ktune_host_allgather_fn)(const void* send, void* recv, int64_t bytes, void* user);
int ktune_ctx_create_hostcomm(int device, int rank, int world, ktune_host_allreduce_fn allreduce,
                              ktune_host_allgather_fn allgather, void* user, ktune_ctx** out);
int ktune_ctx_destroy(ktune_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream()) — NULL restores the own stream. */
int ktune_ctx_set_stream(ktune_ctx* ctx, void* cuda_stream);
void* ktune_ctx_stream(ktune_ctx* ctx);
int ktune_ctx_synchronize(ktune_ctx* ctx);

enum ktune_option {
  KTUNE_OPT_FORCE_EXACT = 1, /* 1: k-means decisions always via the exact-order fallback chains */
  KTUNE_OPT_KMEANS_MODE = 2, /* 0 auto (= 2), 1 exact-order centroids every iteration with the plain exact
                                fp64 assignment scan (mode A), 2 certified integer-sum centroids with exact
                                fallback (mode B), 3 mode A with the tcgen05 screening assignment (kept for
                                comparison: slower than the default fp32-screened exact assignment) */
  KTUNE_OPT_PROFILE = 3,     /* 1: bracket the hot kernels with CUDA events on their stream (KTUNE_STAT_*_NS) */
  KTUNE_OPT_ROLLOUT_DELTA = 4, /* certification margin of the tcgen05 rollout, in units of 1e-12
                                  (0 = default) */
  KTUNE_OPT_ROLLOUT_CHECK = 5, /* 1: re-decide EVERY sampling decision exactly and count disagreements
                                  (calibration/verification mode, slow); 5: the same with PLANTED draws,
                                  each placed 2 delta below/above a fast CDF value (tests the margin
                                  where it is tightest; changes the trajectory, tests only) */
  KTUNE_OPT_ROLLOUT_FUSE_GBT = 6, /* 1: walk the GBT inside the tcgen05 rollout (during its MMA waits)
                                    instead of a separate K1 launch; measured slower on B200, DESIGN.md §5.6 */
  KTUNE_OPT_ROLLOUT_SEGMENTS = 7, /* host-buffer rollouts: step segments overlapped with the D2H copies
                                     (0 = auto, 1 = no segmentation) */
  KTUNE_OPT_FORCE_SHARDED = 8,    /* 1: run the multi-GPU k-means path (per-point state all-gathered over
                                     NCCL) even on one rank; needs a context created by
                                     ktune_ctx_create_dist with an ncclUniqueId (tests on one GPU) */
  KTUNE_OPT_KMEANS_BOUND_LOG2 = 9, /* tests: inflate the certified k-means centroid bounds by 2^value so that
                                     speculative iterations fail and the exact rescue path runs */
  KTUNE_OPT_ROLLOUT_STREAMED = 10  /* host-buffer rollouts on the tcgen05 path: 0 = auto (ONE rollout launch
                                     whose slots publish their per-segment progress in device memory; the
                                     copy stream waits on it with cuStreamWaitValue32 and copies each
                                     finished segment while the kernel runs on; scores follow in chunks),
                                     1 = one launch per segment (the pre-streamed path) */
};
int ktune_ctx_set_option(ktune_ctx* ctx, int option, int64_t value);

enum ktune_stat {
  KTUNE_STAT_LAUNCHES = 1,          /* kernels launched by this context */
  KTUNE_STAT_KPP_FALLBACKS = 2,     /* kmeans++ picks decided by the exact chain */
  KTUNE_STAT_DECISION_FALLBACKS = 3,/* restart / sweep decisions decided by exact loss chains */
  KTUNE_STAT_ASSIGN_FALLBACKS = 4,  /* Lloyd iterations that needed exact-order centroids (mode B) */
  KTUNE_STAT_SNAP_CHAINS = 5,       /* centroid coordinates recomputed by exact-order chains for snapping */
  KTUNE_STAT_LLOYD_ITERS = 6,
  KTUNE_STAT_KPP_PICKS = 7,
  KTUNE_STAT_ROLLOUT_NS = 8,        /* summed device time of rollout_kernel launches (KTUNE_OPT_PROFILE) */
  KTUNE_STAT_ROLLOUT_CALLS = 9,
  KTUNE_STAT_GBT_NS = 10,           /* summed device time of gbt_predict_idx launches */
  KTUNE_STAT_GBT_CALLS = 11,
  KTUNE_STAT_ASSIGN_NS = 12,        /* summed device time of k-means assign launches */
  KTUNE_STAT_ASSIGN_CALLS = 13,
  KTUNE_STAT_XS_SEQUENTIAL = 14,    /* exact-sum segments summed sequentially (binade crossings) */
  KTUNE_STAT_XS_SEGMENTS = 15,      /* exact-sum segments in total */
  KTUNE_STAT_ROLLOUT_FALLBACKS = 16, /* tcgen05 rollout: knob decisions re-decided by the exact fp64 forward */
  KTUNE_STAT_ROLLOUT_CHECKED = 17,   /* KTUNE_OPT_ROLLOUT_CHECK: knob decisions checked */
  KTUNE_STAT_ROLLOUT_MISMATCH = 18,  /* certified fast decisions that disagreed with the exact one (must be 0) */
  KTUNE_STAT_ROLLOUT_MAXERR = 19,    /* max |p_fast - p_exact| over every exactly re-decided knob (the
                                        certificate's fallbacks in normal runs, every knob in check
                                        mode), in units of 1e-12: the live margin monitor */
  KTUNE_STAT_ROLLOUT_TC = 20,        /* config-steps run on the tcgen05 path */
  KTUNE_STAT_KMEANS_ABORTS = 21      /* certified Lloyd runs that fell back to the exact-order mode */
};
int ktune_ctx_stat(ktune_ctx* ctx, int stat, int64_t* value);
int ktune_ctx_reset_stats(ktune_ctx* ctx);

/* ------------------------------------------------------------------ design space
 * design_space.hpp:18-60, validity.hpp:20-48. */
enum ktune_rule_code {
  KTUNE_RULE_PUSH_CONST = 0,
  KTUNE_RULE_PUSH_KNOB = 1,
  KTUNE_RULE_ADD = 2,
  KTUNE_RULE_MUL = 3,
  KTUNE_RULE_LE = 4,
  KTUNE_RULE_LT = 5,
  KTUNE_RULE_EQ = 6
};
typedef struct {
  int32_t code;
  int32_t pad;
  int64_t arg; /* constant or knob index */
} ktune_rule_op;

/* Compile a validity rule (validity.cpp:124-212 grammar) to its postfix
 * program. *nops: in = capacity, out = count. Host-only; no device needed. */
int ktune_rule_compile(const char* source, int num_knobs, const char* const* knob_names,
                       ktune_rule_op* ops, int* nops, char* err, int errlen);
/* Evaluate a compiled rule on host (validity.cpp:162-204); returns 1/0, <0 on error. */
int ktune_rule_eval(const ktune_rule_op* ops, int nops, const int64_t* knob_values);

/* card[D]; values_flat = concatenated knob values (sum(card) entries).
 * Requires 1 <= D <= 32, every card >= 1, size < 2^64 (design_space.cpp:13-58). */
int ktune_space_create(ktune_ctx* ctx, int D, const int32_t* card, const int64_t* values_flat,
                       const ktune_rule_op* ops, int nops, ktune_space** out);
int ktune_space_destroy(ktune_space* space);
/* Host-side helpers with the reference's semantics (no device work):
 * id_of (design_space.cpp:158-167), config_at (:141-156), validate (:169-173). */
int ktune_space_id_of(const ktune_space* s, const int32_t* idx, int64_t n, uint64_t* out);
int ktune_space_config_at(const ktune_space* s, const uint64_t* ids, int64_t n, int32_t* out);
int ktune_space_validate(const ktune_space* s, const int32_t* idx, int64_t n, uint8_t* out);

/* ------------------------------------------------------------------ cost model
 * GbtModel / TreeNode (cost_model.hpp:29-53). Nodes in the reference's flat
 * pre-order layout per tree; feature < 0 marks a leaf. */
typedef struct {
  int32_t feature;
  int32_t left;
  int32_t right;
  int32_t pad;
  double threshold;
  double value;
} ktune_tree_node;

/* Host fit with the reference's exact-greedy boosting (cost_model.cpp:19-177):
 * x is n x dim row-major, y >= 0. Output arrays are allocated by the library
 * and released with ktune_gbt_model_free. */
typedef struct {
  int32_t num_trees;
  int32_t num_features;
  double base_prediction;
  double learning_rate;
  int32_t* tree_offsets; /* num_trees + 1 */
  ktune_tree_node* nodes;
  double* training_sse;  /* num_trees */
} ktune_gbt_model;
int ktune_gbt_fit(const double* x, const double* y, int64_t n, int dim, int num_trees,
                  int max_depth, double learning_rate, int min_samples_leaf, uint64_t seed,
                  ktune_gbt_model* out);
void ktune_gbt_model_free(ktune_gbt_model* m);

/* Upload an ensemble. `space` may be NULL (then only the fp64-feature entry
 * point is usable); with a space the thresholds are also transformed to exact
 * integer index thresholds for ktune_gbt_predict_idx. */
int ktune_gbt_create(ktune_ctx* ctx, const ktune_space* space, int num_features, double base,
                     double learning_rate, int num_trees, const int32_t* tree_offsets,
                     const ktune_tree_node* nodes, ktune_gbt** out);
int ktune_gbt_destroy(ktune_gbt* gbt);
/* predict_batch over knob-index rows (B x D, uint8 when idx_bytes==1, uint16
 * when 2): base + lr * (sum of leaves in tree order), bit-exact with
 * cost_model.cpp:179-199 on the encoded features. */
int ktune_gbt_predict_idx(ktune_ctx* ctx, const ktune_gbt* gbt, const void* idx, int idx_bytes,
                          int64_t B, double* out, int flags);
/* predict_batch over fp64 feature rows (B x num_features row-major) — the
 * generic CostModel::predict(MatrixXd) seam (cost_model.cpp:231-236). */
int ktune_gbt_predict_features(ktune_ctx* ctx, const ktune_gbt* gbt, const double* x, int64_t B,
                               double* out, int flags);

/* ------------------------------------------------------------------ actor-critic
 * ActorCritic (actor_critic.hpp:18-64). flat_params in the header's layout
 * [W0 (h x n), b0, Wp1 (g x h), bp1, Wp2 (3n x g), bp2, Wv1 (g x h), bv1, wv2, bv2],
 * matrices column-major (Eigen::Map order). */
int64_t ktune_ac_num_params(int n, int h, int g);
/* Builder-pinned seeded init. Host-only. */
int ktune_ac_init_params(int n, int h, int g, uint64_t seed, double* out);
int ktune_ac_create(ktune_ctx* ctx, int n, int h, int g, const double* flat_params, ktune_ac** out);
int ktune_ac_destroy(ktune_ac* ac);
/* ActorCritic::forward (actor_critic.hpp:43): states B x n (fp64). Any output may be NULL. */
int ktune_ac_forward(ktune_ctx* ctx, const ktune_ac* ac, const double* states, int64_t B,
                     double* log_probs /* B x 3n */, double* probs /* B x 3n */,
                     double* values /* B */, int flags);

/* ActorCritic::forward with the full Forward cache (actor_critic.hpp:31-43): h0 B x h,
 * hp/hv B x g, logits/log_probs/probs B x 3n, values B (any may be NULL). Same exact fp64
 * arithmetic as ktune_ac_forward. Honours KTUNE_F_DEVICE. */
int ktune_ac_forward_cache(ktune_ctx* ctx, const ktune_ac* ac, const double* states, int64_t B, double* h0,
                           double* hp, double* hv, double* logits, double* log_probs, double* probs, double* values,
                           int flags);
/* ActorCritic::backward (actor_critic.hpp:45-49): the cache of a forward on the same
 * parameters (states B x n, h0, hp, hv) and upstream gradients w.r.t. the logits (B x 3n)
 * and values (B) -> flat parameter gradient (num_params). Batch reductions are sequential
 * in ascending sample order. Honours KTUNE_F_DEVICE. */
int ktune_ac_backward(ktune_ctx* ctx, const ktune_ac* ac, const double* states, const double* h0,
                      const double* hp, const double* hv, int64_t B, const double* d_logits,
                      const double* d_values, double* grad, int flags);
/* Current parameters of an agent (after ktune_ppo_update), flat layout, host memory. */
int ktune_ac_get_params(ktune_ctx* ctx, const ktune_ac* ac, double* out);

/* AdamOptimizer (actor_critic.hpp:66-79): moments on the device, step counter t. */
typedef struct ktune_adam ktune_adam;
int ktune_adam_create(ktune_ctx* ctx, int64_t dim, double step_size, double beta1, double beta2, double epsilon,
                      ktune_adam** out);
int ktune_adam_destroy(ktune_adam* adam);
/* AdamOptimizer::step(params, grad): in-place update of params (dim). Honours KTUNE_F_DEVICE. */
int ktune_adam_step(ktune_ctx* ctx, ktune_adam* adam, double* params, const double* grad, int flags);
/* Moments (host copies, may be NULL) and step count. */
int ktune_adam_state(ktune_ctx* ctx, const ktune_adam* adam, double* m, double* v, int64_t* t);

/* compute_gae for E episodes of T steps (row-major E x T):
 * delta_t = r_t + gamma v_{t+1} - v_t (v_T = terminal_values[e]), A_t = delta_t +
 * gamma lambda A_{t+1}, returns_t = A_t + v_t. Honours KTUNE_F_DEVICE. */
int ktune_compute_gae(ktune_ctx* ctx, int64_t E, int32_t T, const double* rewards, const double* values,
                      const double* terminal_values, double gamma, double lambda, double* advantages,
                      double* returns, int flags);

/* ppo_update (PpoParams SPEC.md:209-216): advantages normalised over the
 * N samples, num_epochs epochs of minibatches drawn from a Fisher-Yates permutation of
 * Rng(seed_combine(seed, epoch)), per minibatch the clipped surrogate + value_coef *
 * (V - R)^2 - entropy_coef * H loss, backward and one Adam step; agent parameters are
 * updated in place on the device. states N x n (encoded features), actions N x n in
 * {-1,0,+1}, old_logp/advantages/returns N. stats (may be NULL): mean over minibatch
 * steps of (policy loss, value loss, entropy). Honours KTUNE_F_DEVICE (inputs). */
typedef struct {
  double clip_epsilon;   /* 0.3 */
  double value_coef;     /* 1.0 */
  double entropy_coef;   /* 0.1 */
  int32_t num_epochs;    /* 3 */
  int32_t pad;
  int64_t minibatch_size; /* 256 */
} ktune_ppo_params;
int ktune_ppo_update(ktune_ctx* ctx, ktune_ac* ac, ktune_adam* adam, const ktune_ppo_params* params, int64_t N,
                     const double* states, const int8_t* actions, const double* old_logp, const double* advantages,
                     const double* returns, uint64_t seed, double* stats, int flags);

/* ------------------------------------------------------------------ rollout
 * run_episodes (pinned details DESIGN.md §5.2). One task =
 * one workload (space + agent + cost model); tasks are batched into one
 * grouped launch. */
typedef struct {
  const ktune_space* space;
  const ktune_ac* ac;
  const ktune_gbt* gbt;     /* may be NULL: no scores */
  int64_t num_episodes;     /* E */
  int64_t episode_offset;   /* global id of this shard's first episode (RNG key) */
  uint64_t explore_seed;    /* stream_seed(root, "explore") */
  const uint16_t* init_idx; /* E x D */
  /* outputs (any may be NULL except idx, see idx_u8); shapes are episode-major as written, step-major
   * ([T+1] x E x ..., [T] x E x ...) with KTUNE_F_STEP_MAJOR: */
  uint16_t* idx;            /* E x (T+1) x D visited configs, row t = Θ_t (NULL allowed with idx_u8, host pointers) */
  double* score;            /* E x (T+1) predicted fitness of Θ_t */
  int8_t* actions;          /* E x T x D directions in {-1,0,+1} */
  double* logp;             /* E x T joint log-probability */
  double* value;            /* E x T value estimate */
  float* logp_f32;          /* E x T, fp32 copies (may be NULL): the tcgen05 path computes both in fp32, */
  float* value_f32;         /* so these halve their device->host bytes without losing anything */
  uint8_t* idx_u8;          /* E x (T+1) x D visited configs as uint8 (may be NULL; every cardinality
                               <= 256). Host-pointer calls may then pass idx = NULL: only these bytes
                               cross PCIe */
  uint8_t* actions_u2;      /* E x T x ceil(D/4) bytes, 2 bits per knob: byte j holds knobs 4j..4j+3 as
                               (direction + 1) << 2*(d - 4j) (may be NULL; host-pointer calls may then
                               pass actions = NULL) */
  float* score_f32;         /* E x (T+1) cost-model scores rounded to fp32 (may be NULL; host-pointer
                               calls may then pass score = NULL): within the 1e-5 relative tolerance the
                               path promises for scores, half the bytes. Candidate ranking on the device
                               always uses the exact fp64 scores. */
  uint32_t* ids_u32;        /* E x (T+1) configuration ids id_of(Θ_t) (design_space.cpp:158-167: mixed
                               radix, last knob fastest; config_at inverts it) (may be NULL; needs
                               |space| <= 2^32). Host-pointer calls may then pass idx = NULL: 4 bytes per
                               visited configuration cross PCIe instead of D (idx_u8) or 2D (idx) */
} ktune_rollout_task;
int ktune_rollout(ktune_ctx* ctx, int num_tasks, const ktune_rollout_task* tasks, int32_t T,
                  int flags);

/* ------------------------------------------------------------------ simulated annealing
 * sa_search: the AutoTVM parallel-SA baseline, builder-pinned
 * (oracle/ktune_oracle.c ko_sa_search). One task = num_chains
 * chains on one space; T steps each. */
typedef struct {
  double initial_temperature; /* 1.0 (SPEC.md SaParams) */
  double cooling_rate;        /* 0.99 per step */
} ktune_sa_params;
typedef struct {
  const ktune_space* space;
  const ktune_gbt* gbt;       /* uploaded with `space` */
  int64_t num_chains;         /* E */
  int64_t chain_offset;       /* global id of the first chain (RNG key; sharding) */
  uint64_t sa_seed;           /* stream_seed(root, "sa") */
  const uint16_t* init_idx;   /* E x D seeds */
  uint16_t* idx;              /* E x (T+1) x D chain states */
  double* score;              /* E x (T+1) predicted fitness of the states */
  uint8_t* accepted;          /* E x T (may be NULL) */
} ktune_sa_task;
int ktune_sa_search(ktune_ctx* ctx, int num_tasks, const ktune_sa_task* tasks, int32_t T,
                    const ktune_sa_params* params, int flags);
/* ------------------------------------------------------------------ candidates
 * make_candidate_set (sampling.cpp:16-31): dedup by id (first occurrence
 * wins) then rank by (predicted fitness desc, id asc). Returns the kept raw
 * row numbers in rank order; *out_n = count. Host pointers. */
int ktune_make_candidate_set(ktune_ctx* ctx, const uint64_t* ids, const double* pred, int64_t n,
                             int64_t* out_rows, int64_t* out_n);
/* Device version over knob-index rows (e.g. a rollout trajectory, uint16 n x D):
 * ids computed on the device (design_space.cpp:158-167), dedup keeping the
 * first occurrence, rank by (pred desc, id asc) via stable radix sorts.
 * out_rows / out_ids (may be NULL) need capacity n; *out_n = kept count.
 * Honours KTUNE_F_DEVICE. */
int ktune_candidates_from_rows(ktune_ctx* ctx, const ktune_space* space, const uint16_t* idx,
                               const double* pred, int64_t n, int64_t* out_rows, uint64_t* out_ids,
                               int64_t* out_n, int flags);

/* Distributed make_candidate_set (the end-of-rollout exchange). Every rank
 * passes the rows of ITS episode shard (uint16 n x D + scores); the result is the global
 * CandidateSet over all ranks' rows, identical on every rank and identical to the
 * single-GPU make_candidate_set over the concatenated trajectories: per-rank dedup +
 * rank, an all-gather of the per-rank sets (NCCL, or the host transport of
 * ktune_ctx_create_hostcomm), and make_candidate_set of their union. The result stays in
 * the context: *out_n = its size; ktune_candidates_gather_copy copies it out (idx uint16
 * out_n x D, pred, ids; any may be NULL). Honours KTUNE_F_DEVICE (inputs and outputs). */
int ktune_candidates_gather(ktune_ctx* ctx, const ktune_space* space, const uint16_t* idx, const double* pred,
                            int64_t n, int64_t* out_n, int flags);
int ktune_candidates_gather_copy(ktune_ctx* ctx, const ktune_space* space, uint16_t* out_idx, double* out_pred,
                                 uint64_t* out_ids, int flags);

/* knob_options' counting pass (sampling.cpp:249-256) on the device: counts has
 * sum(card) entries, counts[sum(card[0..d-1]) + v] = #{i : idx[i][d] == v}.
 * Honours KTUNE_F_DEVICE. */
int ktune_knob_histogram(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                         int64_t N, uint64_t* counts, int flags);
/* ------------------------------------------------------------------ k-means
 * kmeans_run (sampling.hpp:37-38, sampling.cpp:157-175) over lattice points
 * given as knob indices (N x D, idx_bytes 1 or 2) of `space` (features are
 * idx/(card-1), design_space.cpp:189-200). Bit-exact assignments; centroids
 * and losses within the tolerance stated in DESIGN.md §6. */
typedef struct {
  double* centroids;        /* k x D */
  int32_t* assignments;     /* N */
  double* l2_loss;          /* 1 */
  double* iteration_losses; /* max_iters + 1 (may be NULL) */
  int32_t* num_losses;      /* 1 (may be NULL) */
} ktune_kmeans_out;
int ktune_kmeans_run(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                     int64_t N, int k, uint64_t seed, int max_iters, int restarts,
                     ktune_kmeans_out* out, int flags);

/* The adaptive_sample k-sweep (sampling.cpp:436-446) followed by snapping of
 * the breaking sweep's centroids (sampling.cpp:448-452, snap_centroid
 * :202-235). `idx`/`ids` are the candidates in CandidateSet order. */
typedef struct {
  double threshold;     /* 2.5 */
  int32_t k_min;        /* 8 */
  int32_t k_max_exclusive; /* 64 */
  int32_t max_iters;    /* 100 */
  int32_t restarts;     /* 3 */
} ktune_sampling_params;
typedef struct {
  int32_t* k;              /* chosen k */
  double* centroids;       /* k x D (capacity (k_max_exclusive-1) x D) */
  int32_t* assignments;    /* N (may be NULL) */
  double* l2_loss;         /* chosen run's loss (may be NULL) */
  double* k_losses;        /* loss per evaluated k (capacity k_max_exclusive; may be NULL) */
  int32_t* num_k;          /* number of k evaluated (may be NULL) */
  int32_t* snapped;        /* k x D snapped configurations, int32 (may be NULL) */
} ktune_sweep_out;
int ktune_adaptive_sweep(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                         const uint64_t* ids, int64_t N, const ktune_sampling_params* params,
                         uint64_t rng_seed, ktune_sweep_out* out, int flags);

/* snap_centroid for k centroids against the candidate set (int32 output). */
int ktune_snap(ktune_ctx* ctx, const ktune_space* space, const double* centroids, int k,
               const void* cand_idx, int idx_bytes, const uint64_t* cand_ids, int64_t N,
               int32_t* out_idx, int flags);

/* Full Algorithm 1 (adaptive_sample, sampling.cpp:409-461): sweep + snap on
 * the GPU, then the host sample synthesis (sampling.cpp:243-403) for results
 * already in `visited`. Host pointers; out_idx capacity (k_max_exclusive-1) x D. */
int ktune_adaptive_sample(ktune_ctx* ctx, const ktune_space* space, const int32_t* cand_idx,
                          const uint64_t* cand_ids, int64_t N, const uint64_t* visited,
                          int64_t n_visited, const ktune_sampling_params* params,
                          uint64_t rng_seed, int32_t* out_idx, int32_t* out_count);
/* synthesize_sample (sampling.cpp:379-403) alone, host-side. rng_state is the
 * Rng's splitmix state, advanced in place. */
int ktune_synthesize_sample(const ktune_space* space, const int32_t* cand_idx, int64_t N,
                            const uint64_t* visited, int64_t n_visited, uint64_t* rng_state,
                            int32_t* out);

/* ------------------------------------------------------------------ diagnostics
 * Evaluates the device portable transcendental used by the rollout
 * (op 0 exp, 1 log, 2 tanh) on n host doubles — lets tests pin
 * the device implementation bit-for-bit against the oracle's. */
int ktune_debug_math(ktune_ctx* ctx, int op, const double* x, int64_t n, double* out);
/* Copies the tcgen05 rollout's device counters and, after a run with
 * KTUNE_OPT_ROLLOUT_CHECK = 2, its per-phase clock trace (4 + 128 u64). */
int ktune_debug_trace(ktune_ctx* ctx, unsigned long long* out);

#ifdef __cplusplus
}
#endif
#endif /* KTUNE_CUDA_H */
