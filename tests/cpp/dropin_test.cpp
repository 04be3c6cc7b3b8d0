// Drop-in check (test infrastructure): the REFERENCE's own adaptive_sample,
// kmeans_run and predict_batch (compiled from /root/reference/proj/src into
// oracle/_ref/libktune_ref.so) against the same calls routed to the GPU through
// include/ktune_gpu.hpp; and the exploration seam (include/exploration.hpp:
// run_episodes, ActorCritic forward/backward, compute_gae, ppo_update) against the
// oracle restatement (oracle/libktune_oracle.so) plus the reference's own
// make_candidate_set / predict_batch over the oracle's visited configurations.
// Exit 0 iff everything is bit-identical.
#include <cstdio>
#include <unordered_set>

#include "ktune/candidates.hpp"
#include "ktune/cost_model.hpp"
#include "ktune/design_space.hpp"
#include "ktune/measurement.hpp"
#include "ktune/rng.hpp"
#include "ktune/sampling.hpp"
#include "exploration.hpp"
#include "ktune_gpu.hpp"
#include "ktune_oracle.h"

using namespace ktune;

static int fails = 0;
#define EXPECT(c, ...)                 \
  do {                                 \
    if (!(c)) {                        \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");               \
      ++fails;                         \
    }                                  \
  } while (0)

int main() {
  const std::string json =
      R"({"workload":"dropin","knobs":[{"name":"a","values":[1,2,3,4,5,6,7,8,9,10,11,12]},)"
      R"({"name":"b","values":[1,2,4,8,16]},{"name":"c","values":[0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,18,19,20]},)"
      R"({"name":"d","values":[3,5,7]},{"name":"e","values":[1,2,3,4,5,6,7,8]}],"validity_rule":"a * b + d <= 60"})";
  DesignSpace space = DesignSpace::from_json_text(json);
  Rng rng(7);
  std::vector<TrainingExample> train;
  SyntheticLandscapeParams lp;
  lp.seed = 3;
  SyntheticBackend backend(lp, space);
  for (int i = 0; i < 600; ++i) {
    Configuration c = random_configuration(space, rng);
    BackendResult br = backend.evaluate(space, c);
    train.push_back({encode_features(space, c), br.fitness.value_or(0.0)});
  }
  GbtModel model = fit_gbt(train, GbtParams{}, 11);
  std::vector<Candidate> raw;
  std::vector<Configuration> cfgs;
  for (int i = 0; i < 6000; ++i) cfgs.push_back(random_configuration(space, rng));
  Eigen::MatrixXd feats = encode_features_batch(space, cfgs);
  Eigen::VectorXd pred_ref = predict_batch(model, feats);

  gpu::Context ctx(0);
  gpu::Space gs(ctx, space);
  Eigen::VectorXd pred_gpu = gpu::predict(gs, model, feats);
  for (Eigen::Index i = 0; i < pred_ref.size(); ++i)
    EXPECT(pred_ref[i] == pred_gpu[i], "predict row %ld", (long)i);

  for (size_t i = 0; i < cfgs.size(); ++i) raw.push_back({cfgs[i], id_of(space, cfgs[i]), pred_ref[(Eigen::Index)i]});
  CandidateSet cands = make_candidate_set(raw);
  std::vector<Configuration> cc;
  for (auto& c : cands.items) cc.push_back(c.config);
  Eigen::MatrixXd pts = encode_features_batch(space, cc);

  for (int k : {1, 8, 9, 17}) {
    ClusterResult a = kmeans_run(pts, k, 100 + k, 100, 3);
    ClusterResult b = gpu::kmeans_run(gs, pts, k, 100 + k, 100, 3);
    EXPECT(a.assignments == b.assignments, "kmeans k=%d assignments", k);
    EXPECT(a.l2_loss == b.l2_loss, "kmeans k=%d loss %.17g vs %.17g", k, a.l2_loss, b.l2_loss);
    for (int c = 0; c < k; ++c)
      for (int d = 0; d < space.num_knobs(); ++d)
        EXPECT(a.centroids(c, d) == b.centroids(c, d), "kmeans k=%d centroid (%d,%d)", k, c, d);
  }

  SamplingParams sp;
  VisitedSet visited;
  for (size_t i = 0; i < cands.items.size(); i += 5) visited.insert(cands.items[i].id);
  for (uint64_t seed : {1ull, 2ull, 3ull}) {
    std::vector<Configuration> ref = adaptive_sample(cands, visited, sp, space, seed);
    std::vector<Configuration> gpu_out = adaptive_sample(cands, visited, sp, space, seed, gpu::make_clusterer(gs, sp));
    EXPECT(ref == gpu_out, "adaptive_sample seed %llu (%zu vs %zu configs)", (unsigned long long)seed, ref.size(),
           gpu_out.size());
  }
  // ---- exploration seam: run_episodes through exploration.hpp vs the oracle rollout
  const int D = space.num_knobs(), E = 300;
  PpoParams ppo;
  ppo.max_episode_steps = 40;
  ppo.minibatch_size = 128;
  const int T = ppo.max_episode_steps;
  Eigen::VectorXd p0 = gpu::Agent::init_parameters(D, 128, 64, 9);
  gpu::Agent net(ctx, D, 128, 64, p0);
  std::vector<Configuration> init;
  for (int e = 0; e < E; ++e) init.push_back(random_valid_configuration(space, rng));
  auto [ecands, trajs] = gpu::run_episodes(gs, model, net, ppo, init, 21);
  // oracle side: ko_run_episodes on the same space / model / parameters / seeds
  std::vector<int32_t> card, iidx((size_t)E * D), oidx((size_t)E * (T + 1) * D);
  std::vector<int64_t> vals, voff{0};
  for (const Knob& k : space.knobs()) {
    card.push_back(k.cardinality());
    vals.insert(vals.end(), k.values.begin(), k.values.end());
    voff.push_back((int64_t)vals.size());
  }
  ko_space ks{D, card.data(), vals.data(), voff.data(), nullptr, 0};
  std::vector<int32_t> toff, tf, tl, tr;
  std::vector<double> tt, tv;
  for (const RegressionTree& t : model.trees) {
    toff.push_back((int32_t)tf.size());
    for (const TreeNode& nd : t.nodes) {
      tf.push_back(nd.feature);
      tl.push_back(nd.left);
      tr.push_back(nd.right);
      tt.push_back(nd.threshold);
      tv.push_back(nd.value);
    }
  }
  toff.push_back((int32_t)tf.size());
  ko_gbt kg{(int32_t)model.trees.size(), model.num_features, model.base_prediction, model.learning_rate,
            toff.data(), tf.data(), tl.data(), tr.data(), tt.data(), tv.data()};
  for (int e = 0; e < E; ++e)
    for (int d = 0; d < D; ++d) iidx[(size_t)(e * D + d)] = init[(size_t)e].indices[(size_t)d];
  std::vector<double> oscore((size_t)E * (T + 1)), ologp((size_t)E * T), oval((size_t)E * T);
  std::vector<int8_t> oact((size_t)E * T * D);
  ko_run_episodes(&ks, &kg, 128, 64, p0.data(), E, T, 0, ko_stream_seed(21, "explore"), iidx.data(), oidx.data(),
                  oscore.data(), oact.data(), ologp.data(), oval.data(), 4);
  int traj_bad = 0;
  for (int e = 0; e < E; ++e) {
    const Trajectory& t = trajs[(size_t)e];
    for (int s_ = 0; s_ <= T; ++s_)
      for (int d = 0; d < D; ++d)
        traj_bad += t.configs[(size_t)s_].indices[(size_t)d] != oidx[(size_t)((e * (T + 1) + s_) * D + d)];
    for (int s_ = 0; s_ < T; ++s_) {
      for (int d = 0; d < D; ++d) traj_bad += t.actions[(size_t)s_][(size_t)d] != oact[(size_t)((e * T + s_) * D + d)];
      traj_bad += t.rewards[s_] != oscore[(size_t)(e * (T + 1) + s_ + 1)] - oscore[(size_t)(e * (T + 1) + s_)];
      traj_bad += std::fabs(t.log_probs[s_] - ologp[(size_t)(e * T + s_)]) > 1e-5 * std::max(1.0, std::fabs(ologp[(size_t)(e * T + s_)]));
      traj_bad += std::fabs(t.values[s_] - oval[(size_t)(e * T + s_)]) > 1e-5 * std::max(1.0, std::fabs(oval[(size_t)(e * T + s_)]));
    }
  }
  EXPECT(traj_bad == 0, "run_episodes trajectories differ from the oracle (%d fields)", traj_bad);
  // the reference's own make_candidate_set over the oracle's visited configurations, scored
  // by the reference's predict_batch
  std::vector<Configuration> visited_cfgs;
  for (size_t r = 0; r < (size_t)E * (T + 1); ++r) {
    Configuration c;
    c.indices.assign(oidx.begin() + r * D, oidx.begin() + (r + 1) * D);
    visited_cfgs.push_back(c);
  }
  Eigen::VectorXd vpred = predict_batch(model, encode_features_batch(space, visited_cfgs));
  std::vector<Candidate> vraw;
  for (size_t r = 0; r < visited_cfgs.size(); ++r) vraw.push_back({visited_cfgs[r], id_of(space, visited_cfgs[r]), vpred[(Eigen::Index)r]});
  CandidateSet rcands = make_candidate_set(vraw);
  bool cand_ok = rcands.items.size() == ecands.items.size();
  for (size_t i = 0; cand_ok && i < rcands.items.size(); ++i)
    cand_ok = rcands.items[i].config == ecands.items[i].config && rcands.items[i].id == ecands.items[i].id &&
              rcands.items[i].predicted_fitness == ecands.items[i].predicted_fitness;
  EXPECT(cand_ok, "run_episodes CandidateSet differs from the reference's make_candidate_set (%zu vs %zu)",
         ecands.items.size(), rcands.items.size());
  // ActorCritic::forward caches + backward vs the oracle
  Eigen::MatrixXd st = trajs[0].states;
  gpu::Agent::Forward f = net.forward(st);
  std::vector<double> xs((size_t)T * D), h0((size_t)T * 128), hp((size_t)T * 64), hv((size_t)T * 64), lpo((size_t)T * 3 * D),
      pr((size_t)T * 3 * D), vv((size_t)T);
  for (int i = 0; i < T; ++i)
    for (int d = 0; d < D; ++d) xs[(size_t)(i * D + d)] = st(i, d);
  ko_ac_forward(D, 128, 64, p0.data(), xs.data(), T, h0.data(), hp.data(), hv.data(), nullptr, lpo.data(), pr.data(), vv.data());
  int fwd_bad = 0;
  for (int i = 0; i < T; ++i) {
    for (int j = 0; j < 128; ++j) fwd_bad += f.h0(i, j) != h0[(size_t)(i * 128 + j)];
    for (int j = 0; j < 64; ++j) fwd_bad += f.hp(i, j) != hp[(size_t)(i * 64 + j)] || f.hv(i, j) != hv[(size_t)(i * 64 + j)];
    for (int a = 0; a < 3 * D; ++a) fwd_bad += f.log_probs(i, a) != lpo[(size_t)(i * 3 * D + a)] || f.probs(i, a) != pr[(size_t)(i * 3 * D + a)];
    fwd_bad += f.values[i] != vv[(size_t)i];
  }
  EXPECT(fwd_bad == 0, "ActorCritic::forward caches differ from the oracle (%d)", fwd_bad);
  Eigen::MatrixXd dl(T, 3 * D);
  Eigen::VectorXd dv(T);
  std::vector<double> dlf((size_t)T * 3 * D), dvf((size_t)T), gref(p0.size());
  for (int i = 0; i < T; ++i) {
    dv[i] = dvf[(size_t)i] = rng.uniform01() - 0.5;
    for (int a = 0; a < 3 * D; ++a) dl(i, a) = dlf[(size_t)(i * 3 * D + a)] = rng.uniform01() - 0.5;
  }
  Eigen::VectorXd grad = net.backward(f, dl, dv);
  ko_ac_backward(D, 128, 64, p0.data(), xs.data(), h0.data(), hp.data(), hv.data(), T, dlf.data(), dvf.data(), gref.data());
  int bwd_bad = 0;
  for (Eigen::Index i = 0; i < grad.size(); ++i) bwd_bad += grad[i] != gref[(size_t)i];
  EXPECT(bwd_bad == 0, "ActorCritic::backward differs from the oracle (%d)", bwd_bad);
  // compute_gae + ppo_update through the seam vs ko_compute_gae + ko_ppo_update
  gpu::compute_gae(ctx, trajs, ppo);
  gpu::Adam opt(ctx, net.num_parameters(), ppo.adam_step_size);
  gpu::PpoStats pst = gpu::ppo_update(net, opt, trajs, ppo, 77);
  std::vector<double> rw((size_t)E * T), va((size_t)E * T), tvv((size_t)E), av((size_t)E * T), rt((size_t)E * T), S, OL;
  std::vector<int8_t> AC;
  for (int e = 0; e < E; ++e) {
    for (int s_ = 0; s_ < T; ++s_) {
      rw[(size_t)(e * T + s_)] = trajs[(size_t)e].rewards[s_];
      va[(size_t)(e * T + s_)] = trajs[(size_t)e].values[s_];
      for (int d = 0; d < D; ++d) {
        S.push_back(trajs[(size_t)e].states(s_, d));
        AC.push_back(trajs[(size_t)e].actions[(size_t)s_][(size_t)d]);
      }
      OL.push_back(trajs[(size_t)e].log_probs[s_]);
    }
    tvv[(size_t)e] = trajs[(size_t)e].terminal_value;
  }
  ko_compute_gae(E, T, rw.data(), va.data(), tvv.data(), ppo.discount_gamma, ppo.gae_lambda, av.data(), rt.data());
  int gae_bad = 0;
  for (int e = 0; e < E; ++e)
    for (int s_ = 0; s_ < T; ++s_)
      gae_bad += trajs[(size_t)e].advantages[s_] != av[(size_t)(e * T + s_)] || trajs[(size_t)e].returns[s_] != rt[(size_t)(e * T + s_)];
  EXPECT(gae_bad == 0, "compute_gae differs from the oracle (%d)", gae_bad);
  std::vector<double> q(p0.data(), p0.data() + p0.size()), mm(q.size()), vm(q.size());
  int64_t tstep = 0;
  double ost[3];
  ko_ppo_update(D, 128, 64, q.data(), mm.data(), vm.data(), &tstep, (int64_t)OL.size(), S.data(), AC.data(), OL.data(),
                av.data(), rt.data(), ppo.num_epochs, ppo.minibatch_size, ppo.adam_step_size, ppo.clip_epsilon,
                ppo.value_coef, ppo.entropy_coef, 77, ost);
  Eigen::VectorXd upd = net.parameters();
  int ppo_bad = 0;
  for (Eigen::Index i = 0; i < upd.size(); ++i) ppo_bad += upd[i] != q[(size_t)i];
  EXPECT(ppo_bad == 0 && pst.policy_loss == ost[0] && pst.value_loss == ost[1] && pst.entropy == ost[2],
         "ppo_update differs from the oracle (%d parameters)", ppo_bad);
  std::printf("%s: drop-in predict/kmeans_run/adaptive_sample vs reference (%zu candidates); "
              "run_episodes/forward/backward/compute_gae/ppo_update seam (%d x %d, %zu candidates)\n",
              fails ? "FAILED" : "OK", cands.items.size(), E, T, ecands.items.size());
  return fails ? 1 : 0;
}
