/* CPU restatement of the Chameleon (arXiv 2001.08743) reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY — the parity oracle. Only tests/, the
 * __graft_entry__.smoke() checker and bench.py's CPU-baseline leg may load it;
 * the product (paper_2001_08743_b200/) never links or calls it.
 *
 * Pinning: every function below that restates reference code is checked
 * against the reference itself compiled from /root/reference/proj/src
 * (oracle/_ref/libktune_ref.so, see oracle/Makefile) and against the SPEC
 * known-answer examples (tests/test_oracle_*.py, tests/golden/).
 * The rollout (actor-critic forward, sampling, run_episodes) has NO reference
 * code (actor_critic.hpp is declaration-only, exploration is SPEC-only); its
 * restatement here is pinned by the SPEC KATs and by the
 * builder decisions in DESIGN.md §5 — "parity pinned to SPEC KATs only".
 */
#ifndef KTUNE_ORACLE_H
#define KTUNE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- rng.hpp */
uint64_t ko_mix64(uint64_t z);
uint64_t ko_seed_combine(uint64_t a, uint64_t b);
uint64_t ko_stream_seed(uint64_t root, const char* name);
double ko_hash01(uint64_t seed, uint64_t counter);

/* ---------------------------------------------------------------- portable math */
double ko_exp(double x);
double ko_log(double x);
double ko_tanh(double x);

/* ---------------------------------------------------------------- design space */
/* Postfix validity program (validity.hpp:39-47). */
enum { KO_PUSH_CONST = 0, KO_PUSH_KNOB = 1, KO_ADD = 2, KO_MUL = 3, KO_LE = 4, KO_LT = 5, KO_EQ = 6 };
typedef struct {
  int32_t code;
  int32_t pad;
  int64_t arg;
} ko_rule_op;

typedef struct {
  int32_t D;
  const int32_t* card;          /* [D] */
  const int64_t* values;        /* concatenated knob values */
  const int64_t* value_offsets; /* [D+1] */
  const ko_rule_op* ops;        /* postfix program or NULL */
  int32_t nops;
} ko_space;

int ko_validate(const ko_space* s, const int32_t* idx);
uint64_t ko_id_of(const ko_space* s, const int32_t* idx);
void ko_config_at(const ko_space* s, uint64_t id, int32_t* out);
void ko_encode(const ko_space* s, const int32_t* idx, double* out);
void ko_validate_batch(const ko_space* s, const int32_t* idx, int64_t n, uint8_t* out);
void ko_encode_batch(const ko_space* s, const int32_t* idx, int64_t n, double* out);

/* ---------------------------------------------------------------- GBT predict */
typedef struct {
  int32_t num_trees;
  int32_t num_features;
  double base;
  double lr;
  const int32_t* offsets; /* [num_trees+1] into the node arrays */
  const int32_t* feature; /* -1 = leaf */
  const int32_t* left;
  const int32_t* right;
  const double* threshold;
  const double* value;
} ko_gbt;

double ko_gbt_predict_one(const ko_gbt* m, const double* x);
void ko_gbt_predict_features(const ko_gbt* m, const double* x, int64_t n, double* out);
void ko_gbt_predict_idx(const ko_gbt* m, const ko_space* s, const int32_t* idx, int64_t n,
                        double* out);

/* ---------------------------------------------------------------- actor-critic (builder-pinned) */
int64_t ko_ac_num_params(int n, int h, int g);
void ko_ac_init(int n, int h, int g, uint64_t seed, double* params);
/* Batched forward; any output pointer may be NULL. log_probs/probs are B x 3n,
 * h0 B x h, hp/hv B x g, values B. */
void ko_ac_forward(int n, int h, int g, const double* params, const double* states, int64_t B,
                   double* h0, double* hp, double* hv, double* logits, double* log_probs,
                   double* probs, double* values);

/* PPO training step (actor_critic.hpp:45-49,66-79), builder-pinned
 * arithmetic. */
void ko_ac_backward(int n, int h, int g, const double* params, const double* states, const double* h0,
                    const double* hp, const double* hv, int64_t B, const double* d_logits,
                    const double* d_values, double* grad);
void ko_adam_bias(double beta1, double beta2, int64_t t, double* bc1, double* bc2);
void ko_adam_step(int64_t dim, double* params, const double* grad, double* m, double* v, double lr,
                  double beta1, double beta2, double eps, double bc1, double bc2);
void ko_compute_gae(int64_t E, int32_t T, const double* rewards, const double* values,
                    const double* terminal_values, double gamma, double lambda, double* adv, double* ret);
void ko_normalize_advantages(int64_t N, const double* adv, double* out);
void ko_ppo_loss_grad(int n, int64_t B, const double* logp, const double* probs, const double* values,
                      const int8_t* actions, const double* old_logp, const double* adv, const double* ret,
                      double clip_eps, double c_v, double c_e, double* dl, double* dv, double* sums);
int ko_ppo_update(int n, int h, int g, double* params, double* adam_m, double* adam_v, int64_t* adam_t,
                  int64_t N, const double* states, const int8_t* actions, const double* old_logp,
                  const double* adv, const double* ret, int num_epochs, int64_t mb, double lr,
                  double clip_eps, double c_v, double c_e, uint64_t seed, double* stats);

/* run_episodes, builder-pinned details in DESIGN.md §5.
 * E episodes with global ids episode_offset..episode_offset+E-1, T steps each.
 * idx_out: E x (T+1) x D visited configs (row t = Θ_t), score_out E x (T+1),
 * actions_out E x T x D in {-1,0,+1}, logp_out/value_out E x T.
 * Any output except idx_out may be NULL. threads>1 splits episodes. */
int ko_sa_search(const ko_space* s, const ko_gbt* m, int64_t E, int32_t T, int64_t chain_offset,
                 uint64_t sa_seed, double t0, double rate, const int32_t* init_idx, int32_t* idx_out,
                 double* score_out, uint8_t* acc_out, int threads);
int ko_run_episodes(const ko_space* s, const ko_gbt* m, int h, int g, const double* params,
                    int64_t E, int32_t T, int64_t episode_offset, uint64_t explore_seed,
                    const int32_t* init_idx, int32_t* idx_out, double* score_out,
                    int8_t* actions_out, double* logp_out, double* value_out, int threads);

/* ---------------------------------------------------------------- candidates / sampling */
int64_t ko_make_candidate_set(int D, const int32_t* idx, const uint64_t* ids, const double* pred,
                              int64_t n, int64_t* out_rows);
/* kmeans_run (sampling.cpp:157-175). points N x D row-major. iteration_losses
 * needs max_iters+1 slots. Returns 0, 1 (ConfigError) or 4 (logic_error). */
int ko_kmeans_run(const double* points, int64_t N, int D, int k, uint64_t seed, int max_iters,
                  int restarts, double* centroids, int32_t* assignments, double* loss,
                  double* iteration_losses, int32_t* num_losses);
/* The adaptive_sample k-sweep (sampling.cpp:436-446): chosen k, its result and
 * the loss of every k evaluated (<= 63 entries). */
int ko_adaptive_sweep(const double* points, int64_t N, int D, double threshold, int k_min,
                      int k_max_exclusive, int max_iters, int restarts, uint64_t rng_seed,
                      int32_t* k_chosen, double* centroids, int32_t* assignments, double* loss,
                      double* k_losses, int32_t* num_k);
/* snap_centroid (sampling.cpp:202-235); candidates in CandidateSet order. */
void ko_snap_centroid(const ko_space* s, const double* centroid, const int32_t* cand_idx,
                      const uint64_t* cand_ids, int64_t n, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
