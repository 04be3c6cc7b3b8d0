// exploration.hpp — the Adaptive-Exploration module's C++ seam. The
// reference has no header or code for this module (actor_critic.hpp:18-79 declares
// ActorCritic / AdamOptimizer without definitions; run_episodes, compute_gae and
// ppo_update exist only in SPEC), so this header supplies them with the SPEC signatures,
// executed on the GPU through libktune_cuda (include/ktune_cuda.h):
//
//   ktune::gpu::Context ctx(0);
//   ktune::gpu::Space gs(ctx, space);
//   ktune::gpu::Agent net(ctx, space.num_knobs(), 128, 64, params);   // ActorCritic, device-resident
//   auto [cands, trajs] = ktune::gpu::run_episodes(gs, cost_model.model(), net, ppo, initial_configs, seed);
//   ktune::gpu::compute_gae(ctx, trajs, ppo);                          // advantages, returns
//   ktune::gpu::Adam opt(ctx, net.num_parameters(), ppo.adam_step_size);
//   ktune::gpu::PpoStats st = ktune::gpu::ppo_update(net, opt, trajs, ppo, seed);
//
// Semantics (builder-pinned): every episode runs exactly
// params.max_episode_steps steps; the counter-based draw of (episode e, step t, knob d) is
// hash01(stream_seed(rng_seed, "explore"), ((episode_offset + e) T + t) D + d); the
// trajectories' rewards are r_t = pred(Θ_{t+1}) - pred(Θ_t) from the cost model's scores of
// every visited configuration, all of which join the CandidateSet.
#ifndef KTUNE_EXPLORATION_HPP
#define KTUNE_EXPLORATION_HPP

#include <utility>
#include <vector>

#include "ktune/actor_critic.hpp"
#include "ktune/candidates.hpp"
#include "ktune_gpu.hpp"

namespace ktune {

/// SPEC.md:209-216 (PpoParams).
struct PpoParams {
  double adam_step_size = 1e-3;
  double discount_gamma = 0.9;
  double gae_lambda = 0.99;
  int num_epochs = 3;
  double clip_epsilon = 0.3;
  double value_coef = 1.0;
  double entropy_coef = 0.1;
  int episodes_per_iteration = 128;
  int max_episode_steps = 500;
  int minibatch_size = 256;
};

/// SPEC.md:221-224 (Trajectory): per-step records of one episode (T = steps).
struct Trajectory {
  Eigen::MatrixXd states;               // T x n   encode_features(Θ_t), t < T
  std::vector<Configuration> configs;   // T + 1   Θ_0 .. Θ_T
  std::vector<std::vector<int8_t>> actions;  // T x n in {-1, 0, +1}
  Eigen::VectorXd log_probs;            // T       joint log-probability of the action
  Eigen::VectorXd values;               // T       value estimate V(Θ_t)
  Eigen::VectorXd rewards;              // T       pred(Θ_{t+1}) - pred(Θ_t)
  double terminal_value = 0.0;          //         V(Θ_T), the GAE bootstrap
  Eigen::VectorXd advantages;           // T       filled by compute_gae
  Eigen::VectorXd returns;              // T
};

namespace gpu {

inline Eigen::VectorXd vec(const double* p, Eigen::Index n) {
  Eigen::VectorXd v(n);
  for (Eigen::Index i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

/// ActorCritic (actor_critic.hpp:18-64) with its flat parameters resident on the device.
class Agent {
 public:
  using Forward = ActorCritic::Forward;
  Agent(Context& ctx, int num_knobs, int hidden_dim, int head_hidden, const Eigen::VectorXd& params)
      : ctx_(ctx), n_(num_knobs), h_(hidden_dim), g_(head_hidden) {
    check(ktune_ac_create(ctx.get(), n_, h_, g_, params.data(), &a_), ctx.get());
  }
  /// The builder-pinned seeded initialisation.
  static Eigen::VectorXd init_parameters(int n, int h, int g, uint64_t seed) {
    Eigen::VectorXd p((Eigen::Index)ktune_ac_num_params(n, h, g));
    check(ktune_ac_init_params(n, h, g, seed, p.data()), nullptr);
    return p;
  }
  ~Agent() { ktune_ac_destroy(a_); }
  Agent(const Agent&) = delete;
  Agent& operator=(const Agent&) = delete;
  ktune_ac* get() const { return a_; }
  Context& ctx() const { return ctx_; }
  int num_knobs() const { return n_; }
  int hidden_dim() const { return h_; }
  int head_hidden() const { return g_; }
  int num_parameters() const { return (int)ktune_ac_num_params(n_, h_, g_); }

  Eigen::VectorXd parameters() const {
    Eigen::VectorXd p(num_parameters());
    check(ktune_ac_get_params(ctx_.get(), a_, p.data()), ctx_.get());
    return p;
  }

  /// ActorCritic::forward (actor_critic.hpp:43) with every cached activation of Forward
  /// (:31-39), exact fp64 (bit-identical to the oracle restatement).
  ActorCritic::Forward forward(const Eigen::MatrixXd& states) const {
    const Eigen::Index B = states.rows();
    if (B && states.cols() != n_) throw ConfigError("actor-critic: state dimension mismatch");
    std::vector<double> x((size_t)B * n_), h0((size_t)B * h_), hp((size_t)B * g_), hv((size_t)B * g_),
        lg((size_t)B * 3 * n_), lp((size_t)B * 3 * n_), pr((size_t)B * 3 * n_), v((size_t)B);
    for (Eigen::Index i = 0; i < B; ++i)
      for (int d = 0; d < n_; ++d) x[(size_t)i * n_ + d] = states(i, d);
    if (B)
      check(ktune_ac_forward_cache(ctx_.get(), a_, x.data(), B, h0.data(), hp.data(), hv.data(), lg.data(), lp.data(),
                                   pr.data(), v.data(), 0),
            ctx_.get());
    ActorCritic::Forward f;
    f.states = states;
    f.h0 = rows(h0, B, h_);
    f.hp = rows(hp, B, g_);
    f.hv = rows(hv, B, g_);
    f.log_probs = rows(lp, B, 3 * n_);
    f.probs = rows(pr, B, 3 * n_);
    f.values = vec(v.data(), B);
    return f;
  }

  /// ActorCritic::backward (actor_critic.hpp:45-49).
  Eigen::VectorXd backward(const Forward& cache, const Eigen::MatrixXd& d_logits,
                           const Eigen::VectorXd& d_values) const {
    const Eigen::Index B = cache.states.rows();
    auto flat = [B](const Eigen::MatrixXd& m) {
      std::vector<double> o((size_t)B * m.cols());
      for (Eigen::Index i = 0; i < B; ++i)
        for (Eigen::Index j = 0; j < m.cols(); ++j) o[(size_t)(i * m.cols() + j)] = m(i, j);
      return o;
    };
    const std::vector<double> x = flat(cache.states), h0 = flat(cache.h0), hp = flat(cache.hp), hv = flat(cache.hv),
                              dl = flat(d_logits);
    std::vector<double> dv(d_values.data(), d_values.data() + B);
    Eigen::VectorXd grad(num_parameters());
    check(ktune_ac_backward(ctx_.get(), a_, x.data(), h0.data(), hp.data(), hv.data(), B, dl.data(), dv.data(),
                            grad.data(), 0),
          ctx_.get());
    return grad;
  }

 private:
  static Eigen::MatrixXd rows(const std::vector<double>& v, Eigen::Index B, int c) {
    Eigen::MatrixXd m(B, c);
    for (Eigen::Index i = 0; i < B; ++i)
      for (int j = 0; j < c; ++j) m(i, j) = v[(size_t)(i * c + j)];
    return m;
  }
  Context& ctx_;
  int n_, h_, g_;
  ktune_ac* a_ = nullptr;
};

/// AdamOptimizer (actor_critic.hpp:66-79), moments on the device.
class Adam {
 public:
  Adam(Context& ctx, int dim, double step_size, double beta1 = 0.9, double beta2 = 0.999, double epsilon = 1e-8)
      : ctx_(ctx) {
    check(ktune_adam_create(ctx.get(), dim, step_size, beta1, beta2, epsilon, &h_), ctx.get());
  }
  ~Adam() { ktune_adam_destroy(h_); }
  Adam(const Adam&) = delete;
  Adam& operator=(const Adam&) = delete;
  ktune_adam* get() const { return h_; }
  /// AdamOptimizer::step (actor_critic.hpp:75).
  void step(Eigen::VectorXd& params, const Eigen::VectorXd& grad) {
    check(ktune_adam_step(ctx_.get(), h_, params.data(), grad.data(), 0), ctx_.get());
  }

 private:
  Context& ctx_;
  ktune_adam* h_ = nullptr;
};

/// run_episodes: one grouped launch of the tcgen05 rollout (certified
/// sampling: configurations, actions and scores bit-exact with the exact fp64 semantics)
/// + cost-model scoring of every visited configuration, then the CandidateSet
/// (make_candidate_set on the device, sampling.cpp:16-31) and one Trajectory per episode.
/// `exact` selects the fp64 kernel (log-probabilities and values bit-exact as well).
inline std::pair<CandidateSet, std::vector<Trajectory>> run_episodes(
    const Space& s, const GbtModel& cost_model, const Agent& net, const PpoParams& params,
    const std::vector<Configuration>& initial_configs, uint64_t rng_seed, int64_t episode_offset = 0,
    bool exact = false) {
  const DesignSpace& space = s.space();
  const int D = space.num_knobs(), T = params.max_episode_steps;
  const int64_t E = (int64_t)initial_configs.size();
  if (net.num_knobs() != D) throw ConfigError("run_episodes: agent/space knob count mismatch");
  ktune_ctx* ctx = s.ctx().get();
  std::vector<uint16_t> init((size_t)E * D);
  for (int64_t e = 0; e < E; ++e) {
    if ((int)initial_configs[(size_t)e].indices.size() != D) throw ConfigError("run_episodes: configuration size");
    for (int d = 0; d < D; ++d) init[(size_t)(e * D + d)] = (uint16_t)initial_configs[(size_t)e].indices[(size_t)d];
  }
  const size_t rows = (size_t)E * (T + 1);
  std::vector<uint16_t> idx(rows * D);
  std::vector<double> score(rows), logp((size_t)E * T), value((size_t)E * T);
  std::vector<int8_t> act((size_t)E * T * D);
  static thread_local std::vector<std::pair<std::pair<uint64_t, uint64_t>, std::shared_ptr<Ensemble>>> ens;
  const std::pair<uint64_t, uint64_t> key{s.serial(), model_fingerprint(cost_model)};
  std::shared_ptr<Ensemble> g;
  for (auto& kv : ens)
    if (kv.first == key) g = kv.second;
  if (!g) {
    g = std::make_shared<Ensemble>(s, cost_model);
    ens.insert(ens.begin(), {key, g});
    if (ens.size() > 4) ens.pop_back();
  }
  // stream_seed(rng_seed, "explore") (rng.hpp:33-40)
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const char* c = "explore"; *c; ++c) h = (h ^ (unsigned char)*c) * 0x100000001B3ULL;
  auto mix64 = [](uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  const uint64_t explore = mix64(rng_seed + 0x9E3779B97F4A7C15ULL + mix64(h));
  ktune_rollout_task task{};
  task.space = s.get();
  task.ac = net.get();
  task.gbt = g->get();
  task.num_episodes = E;
  task.episode_offset = episode_offset;
  task.explore_seed = explore;
  task.init_idx = init.data();
  task.idx = idx.data();
  task.score = score.data();
  task.actions = act.data();
  task.logp = logp.data();
  task.value = value.data();
  if (E) check(ktune_rollout(ctx, 1, &task, T, exact ? KTUNE_F_EXACT_ROLLOUT : 0), ctx);
  // CandidateSet of every visited configuration (device dedup + rank)
  CandidateSet cands;
  if (E) {
    std::vector<int64_t> kept(rows);
    std::vector<uint64_t> ids(rows);
    int64_t m = 0;
    check(ktune_candidates_from_rows(ctx, s.get(), idx.data(), score.data(), (int64_t)rows, kept.data(), ids.data(),
                                     &m, 0),
          ctx);
    cands.items.resize((size_t)m);
    for (int64_t i = 0; i < m; ++i) {
      Candidate& c = cands.items[(size_t)i];
      c.config.indices.assign(idx.begin() + kept[(size_t)i] * D, idx.begin() + (kept[(size_t)i] + 1) * D);
      c.id = ids[(size_t)i];
      c.predicted_fitness = score[(size_t)kept[(size_t)i]];
    }
  }
  // trajectories: encoded states (design_space.cpp:189-200), rewards, terminal values
  std::vector<double> inv(D);
  for (int d = 0; d < D; ++d) {
    const int card = space.knobs()[(size_t)d].cardinality();
    inv[(size_t)d] = card > 1 ? (double)(card - 1) : 0.0;
  }
  auto feat = [&](size_t row, int d) {
    return inv[(size_t)d] > 0.0 ? (double)idx[row * D + d] / inv[(size_t)d] : 0.0;
  };
  std::vector<Trajectory> trajs((size_t)E);
  Eigen::MatrixXd last(E, D);
  for (int64_t e = 0; e < E; ++e) {
    Trajectory& tr = trajs[(size_t)e];
    tr.states.resize(T, D);
    tr.configs.resize((size_t)T + 1);
    tr.actions.assign((size_t)T, std::vector<int8_t>((size_t)D));
    tr.log_probs.resize(T);
    tr.values.resize(T);
    tr.rewards.resize(T);
    for (int t = 0; t <= T; ++t) {
      const size_t row = (size_t)(e * (T + 1) + t);
      tr.configs[(size_t)t].indices.assign(idx.begin() + row * D, idx.begin() + (row + 1) * D);
      for (int d = 0; d < D; ++d) {
        if (t < T) tr.states(t, d) = feat(row, d);
        else last(e, d) = feat(row, d);
      }
      if (t < T) {
        for (int d = 0; d < D; ++d) tr.actions[(size_t)t][(size_t)d] = act[(size_t)((e * T + t) * D + d)];
        tr.log_probs[t] = logp[(size_t)(e * T + t)];
        tr.values[t] = value[(size_t)(e * T + t)];
        tr.rewards[t] = score[row + 1] - score[row];
      }
    }
  }
  if (E) {
    const Agent::Forward f = net.forward(last);
    for (int64_t e = 0; e < E; ++e) trajs[(size_t)e].terminal_value = f.values[e];
  }
  return {std::move(cands), std::move(trajs)};
}

/// compute_gae for every trajectory (equal lengths), on the device.
inline void compute_gae(Context& ctx, std::vector<Trajectory>& trajs, const PpoParams& p) {
  if (trajs.empty()) return;
  const int64_t E = (int64_t)trajs.size();
  const int T = (int)trajs[0].rewards.size();
  std::vector<double> r((size_t)E * T), v((size_t)E * T), tv((size_t)E), a((size_t)E * T), ret((size_t)E * T);
  for (int64_t e = 0; e < E; ++e) {
    const Trajectory& tr = trajs[(size_t)e];
    if ((int)tr.rewards.size() != T || (int)tr.values.size() != T) throw ConfigError("compute_gae: length mismatch");
    for (int t = 0; t < T; ++t) {
      r[(size_t)(e * T + t)] = tr.rewards[t];
      v[(size_t)(e * T + t)] = tr.values[t];
    }
    tv[(size_t)e] = tr.terminal_value;
  }
  check(ktune_compute_gae(ctx.get(), E, T, r.data(), v.data(), tv.data(), p.discount_gamma, p.gae_lambda, a.data(),
                          ret.data(), 0),
        ctx.get());
  for (int64_t e = 0; e < E; ++e) {
    trajs[(size_t)e].advantages = vec(a.data() + e * T, T);
    trajs[(size_t)e].returns = vec(ret.data() + e * T, T);
  }
}

struct PpoStats {
  double policy_loss = 0.0, value_loss = 0.0, entropy = 0.0;
};

/// ppo_update on the device: the agent's parameters are updated in place.
inline PpoStats ppo_update(Agent& net, Adam& opt, const std::vector<Trajectory>& trajs, const PpoParams& p,
                           uint64_t seed) {
  const int n = net.num_knobs();
  std::vector<double> S, lp, adv, ret;
  std::vector<int8_t> A;
  for (const Trajectory& tr : trajs) {
    if (tr.advantages.size() != tr.rewards.size()) throw ConfigError("ppo_update: run compute_gae first");
    for (Eigen::Index t = 0; t < tr.states.rows(); ++t) {
      for (int d = 0; d < n; ++d) {
        S.push_back(tr.states(t, d));
        A.push_back(tr.actions[(size_t)t][(size_t)d]);
      }
      lp.push_back(tr.log_probs[t]);
      adv.push_back(tr.advantages[t]);
      ret.push_back(tr.returns[t]);
    }
  }
  ktune_ppo_params pp{};
  pp.clip_epsilon = p.clip_epsilon;
  pp.value_coef = p.value_coef;
  pp.entropy_coef = p.entropy_coef;
  pp.num_epochs = p.num_epochs;
  pp.minibatch_size = p.minibatch_size;
  double st[3] = {0, 0, 0};
  check(ktune_ppo_update(net.ctx().get(), net.get(), opt.get(), &pp, (int64_t)lp.size(), S.data(), A.data(), lp.data(),
                         adv.data(), ret.data(), seed, st, 0),
        net.ctx().get());
  return {st[0], st[1], st[2]};
}

}  // namespace gpu
}  // namespace ktune

#endif  // KTUNE_EXPLORATION_HPP
