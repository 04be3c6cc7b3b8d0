// Drop-in check (test infrastructure): the REFERENCE's own adaptive_sample,
// kmeans_run and predict_batch (compiled from /root/reference/proj/src into
// oracle/_ref/libktune_ref.so) against the same calls routed to the GPU through
// include/ktune_gpu.hpp. Exit 0 iff everything is bit-identical.
#include <cstdio>
#include <unordered_set>

#include "ktune/candidates.hpp"
#include "ktune/cost_model.hpp"
#include "ktune/design_space.hpp"
#include "ktune/measurement.hpp"
#include "ktune/rng.hpp"
#include "ktune/sampling.hpp"
#include "ktune_gpu.hpp"

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
  std::printf("%s: drop-in predict/kmeans_run/adaptive_sample vs reference (%zu candidates)\n",
              fails ? "FAILED" : "OK", cands.items.size());
  return fails ? 1 : 0;
}
