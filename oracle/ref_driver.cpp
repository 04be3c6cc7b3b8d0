// extern "C" driver over the REFERENCE's own C++ API (/root/reference/proj),
// compiled together with the reference sources (unmodified, in place) and the
// Eigen-subset shim into oracle/_ref/libktune_ref.so by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (to pin the C restatement in
// oracle/ktune_oracle.c and to generate golden fixtures) and by bench.py's
// CPU-baseline leg. Never linked into the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <unordered_set>
#include <vector>

#include "ktune/candidates.hpp"
#include "ktune/cost_model.hpp"
#include "ktune/design_space.hpp"
#include "ktune/errors.hpp"
#include "ktune/measurement.hpp"
#include "ktune/rng.hpp"
#include "ktune/sampling.hpp"

using namespace ktune;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// 1 ConfigError, 2 BackendError, 3 SpaceExhaustedError, 4 logic_error, 9 other.
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    return fail(e, 1);
  } catch (const BackendError& e) {
    return fail(e, 2);
  } catch (const SpaceExhaustedError& e) {
    return fail(e, 3);
  } catch (const std::logic_error& e) {
    return fail(e, 4);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

Eigen::MatrixXd rows_to_matrix(const double* x, int64_t n, int d) {
  Eigen::MatrixXd m(n, d);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) m(i, j) = x[i * d + j];
  return m;
}

Configuration cfg_from(const int32_t* idx, int d) {
  Configuration c;
  c.indices.assign(idx, idx + d);
  return c;
}

CandidateSet candidates_from(const DesignSpace& s, const int32_t* idx, const uint64_t* ids,
                             const double* pred, int64_t n) {
  // Already in CandidateSet order (the caller ran make_candidate_set).
  CandidateSet set;
  set.items.resize(static_cast<std::size_t>(n));
  const int d = s.num_knobs();
  for (int64_t i = 0; i < n; ++i) {
    set.items[i].config = cfg_from(idx + i * d, d);
    set.items[i].id = ids[i];
    set.items[i].predicted_fitness = pred[i];
  }
  return set;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- rng.hpp
uint64_t ref_mix64(uint64_t z) { return mix64(z); }
uint64_t ref_seed_combine(uint64_t a, uint64_t b) { return seed_combine(a, b); }
uint64_t ref_stream_seed(uint64_t root, const char* name) { return stream_seed(root, name); }
double ref_hash01(uint64_t seed, uint64_t counter) { return hash01(seed, counter); }
// Draws: kind 0 next_u64, 1 uniform01 (bits), 2 below(arg).
int ref_rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t n, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = r.next_u64();
    } else if (kind == 1) {
      double u = r.uniform01();
      std::memcpy(&out[i], &u, 8);
    } else {
      out[i] = r.below(arg);
    }
  }
  return 0;
}

// ---------------------------------------------------------------- design space
void* ref_space_new(const char* json) {
  DesignSpace* s = nullptr;
  int rc = guard([&] { s = new DesignSpace(DesignSpace::from_json_text(json)); });
  return rc == 0 ? s : nullptr;
}
void ref_space_free(void* s) { delete static_cast<DesignSpace*>(s); }
int ref_space_dims(void* h, int32_t* card, uint64_t* size) {
  auto* s = static_cast<DesignSpace*>(h);
  for (int i = 0; i < s->num_knobs(); ++i) card[i] = s->knobs()[i].cardinality();
  *size = s->size();
  return s->num_knobs();
}
int ref_config_at(void* h, uint64_t id, int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  return guard([&] {
    Configuration c = config_at(*s, id);
    std::memcpy(out, c.indices.data(), c.indices.size() * 4);
  });
}
int ref_id_of(void* h, const int32_t* idx, uint64_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  return guard([&] { *out = id_of(*s, cfg_from(idx, s->num_knobs())); });
}
int ref_validate(void* h, const int32_t* idx, int64_t n, uint8_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    for (int64_t i = 0; i < n; ++i) out[i] = validate(*s, cfg_from(idx + i * d, d)) ? 1 : 0;
  });
}
int ref_neighbor(void* h, const int32_t* idx, int knob, int dir, int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  return guard([&] {
    Configuration c = neighbor(*s, cfg_from(idx, s->num_knobs()), knob, dir);
    std::memcpy(out, c.indices.data(), c.indices.size() * 4);
  });
}
int ref_encode_batch(void* h, const int32_t* idx, int64_t n, double* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    std::vector<Configuration> cs;
    for (int64_t i = 0; i < n; ++i) cs.push_back(cfg_from(idx + i * d, d));
    Eigen::MatrixXd m = encode_features_batch(*s, cs);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) out[i * d + j] = m(i, j);
  });
}
int ref_random_valid_configs(void* h, uint64_t seed, int64_t n, int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) {
      Configuration c = random_valid_configuration(*s, r);
      std::memcpy(out + i * d, c.indices.data(), d * 4);
    }
  });
}

// ---------------------------------------------------------------- measurement
// SyntheticBackend fitness (NaN when the backend reports invalid).
int ref_synthetic_fitness(void* h, const char* invalid_rule, uint64_t seed, int num_peaks,
                          double sharpness, double noise, const int32_t* idx, int64_t n,
                          double* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    SyntheticLandscapeParams p;
    p.num_peaks = num_peaks;
    p.peak_sharpness = sharpness;
    p.noise_amplitude = noise;
    p.invalid_rule = invalid_rule ? invalid_rule : "";
    p.seed = seed;
    SyntheticBackend b(p, *s);
    for (int64_t i = 0; i < n; ++i) {
      BackendResult r = b.evaluate(*s, cfg_from(idx + i * d, d));
      out[i] = r.fitness.has_value() ? *r.fitness : std::nan("");
    }
  });
}

// ---------------------------------------------------------------- cost model
void* ref_gbt_fit(const double* x, const double* y, int64_t n, int dim, int num_trees,
                  int max_depth, double lr, int min_leaf, uint64_t seed) {
  GbtModel* m = nullptr;
  int rc = guard([&] {
    std::vector<TrainingExample> ex(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      ex[i].features = Eigen::VectorXd(dim);
      for (int j = 0; j < dim; ++j) ex[i].features[j] = x[i * dim + j];
      ex[i].fitness = y[i];
    }
    GbtParams p;
    p.num_trees = num_trees;
    p.max_depth = max_depth;
    p.learning_rate = lr;
    p.min_samples_leaf = min_leaf;
    m = new GbtModel(fit_gbt(ex, p, seed));
  });
  return rc == 0 ? m : nullptr;
}
void ref_gbt_free(void* h) { delete static_cast<GbtModel*>(h); }
// Sizes: returns total node count; fills num_trees/num_features.
int64_t ref_gbt_shape(void* h, int* num_trees, int* num_features) {
  auto* m = static_cast<GbtModel*>(h);
  *num_trees = static_cast<int>(m->trees.size());
  *num_features = m->num_features;
  int64_t total = 0;
  for (auto& t : m->trees) total += static_cast<int64_t>(t.nodes.size());
  return total;
}
// Flattened export: offsets[num_trees+1]; per node feature/left/right (int32),
// threshold/value (double); training_sse[num_trees].
void ref_gbt_export(void* h, double* base, double* lr, int32_t* offsets, int32_t* feature,
                    int32_t* left, int32_t* right, double* threshold, double* value,
                    double* training_sse) {
  auto* m = static_cast<GbtModel*>(h);
  *base = m->base_prediction;
  *lr = m->learning_rate;
  int64_t k = 0;
  for (std::size_t t = 0; t < m->trees.size(); ++t) {
    offsets[t] = static_cast<int32_t>(k);
    for (const TreeNode& nd : m->trees[t].nodes) {
      feature[k] = nd.feature;
      left[k] = nd.left;
      right[k] = nd.right;
      threshold[k] = nd.threshold;
      value[k] = nd.value;
      ++k;
    }
    training_sse[t] = m->training_sse[t];
  }
  offsets[m->trees.size()] = static_cast<int32_t>(k);
}
int ref_gbt_predict(void* h, const double* x, int64_t n, int dim, double* out) {
  auto* m = static_cast<GbtModel*>(h);
  return guard([&] {
    Eigen::VectorXd r = predict_batch(*m, rows_to_matrix(x, n, dim));
    for (int64_t i = 0; i < n; ++i) out[i] = r[i];
  });
}

// ---------------------------------------------------------------- candidates
// In: raw (idx n×d, ids, pred). Out: permutation of kept raw rows in rank order.
int64_t ref_make_candidate_set(int d, const int32_t* idx, const uint64_t* ids, const double* pred,
                               int64_t n, int64_t* out_rows) {
  std::vector<Candidate> raw(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    raw[i].config = cfg_from(idx + i * d, d);
    raw[i].config.indices.push_back(static_cast<int32_t>(i));  // smuggle the row number
    raw[i].id = ids[i];
    raw[i].predicted_fitness = pred[i];
  }
  CandidateSet set = make_candidate_set(std::move(raw));
  for (std::size_t i = 0; i < set.items.size(); ++i) out_rows[i] = set.items[i].config.indices[d];
  return static_cast<int64_t>(set.items.size());
}

// ---------------------------------------------------------------- sampling
int ref_kmeans_run(const double* points, int64_t n, int d, int k, uint64_t seed, int max_iters,
                   int restarts, double* centroids, int32_t* assignments, double* loss,
                   double* iteration_losses, int32_t* num_losses) {
  return guard([&] {
    ClusterResult r = kmeans_run(rows_to_matrix(points, n, d), k, seed, max_iters, restarts);
    for (int c = 0; c < k; ++c)
      for (int j = 0; j < d; ++j) centroids[c * d + j] = r.centroids(c, j);
    for (int64_t i = 0; i < n; ++i) assignments[i] = r.assignments[i];
    *loss = r.l2_loss;
    *num_losses = static_cast<int32_t>(r.iteration_losses.size());
    for (std::size_t i = 0; i < r.iteration_losses.size(); ++i) iteration_losses[i] = r.iteration_losses[i];
  });
}

int ref_snap_centroid(void* h, const double* centroid, const int32_t* cand_idx,
                      const uint64_t* cand_ids, const double* cand_pred, int64_t n,
                      int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    CandidateSet set = candidates_from(*s, cand_idx, cand_ids, cand_pred, n);
    Eigen::VectorXd c(d);
    for (int j = 0; j < d; ++j) c[j] = centroid[j];
    Configuration r = snap_centroid(c, *s, set);
    std::memcpy(out, r.indices.data(), d * 4);
  });
}

// adaptive_sample with the DEFAULT clusterer (kmeans_run). Also reports the
// chosen k and the per-k losses by wrapping the default clusterer.
int ref_adaptive_sample(void* h, const int32_t* cand_idx, const uint64_t* cand_ids,
                        const double* cand_pred, int64_t n, const uint64_t* visited,
                        int64_t n_visited, double threshold, int k_min, int k_max_excl,
                        int max_iters, int restarts, uint64_t rng_seed, int32_t* out_idx,
                        int32_t* out_count, double* k_losses, int32_t* k_count) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    CandidateSet set = candidates_from(*s, cand_idx, cand_ids, cand_pred, n);
    VisitedSet vis(visited, visited + n_visited);
    SamplingParams p;
    p.threshold = threshold;
    p.k_min = k_min;
    p.k_max_exclusive = k_max_excl;
    p.kmeans_max_iters = max_iters;
    p.kmeans_restarts = restarts;
    int nk = 0;
    Clusterer wrap = [&](const Eigen::MatrixXd& pts, int k, std::uint64_t seed) {
      ClusterResult r = kmeans_run(pts, k, seed, max_iters, restarts);
      if (k_losses) k_losses[nk] = r.l2_loss;
      ++nk;
      return r;
    };
    std::vector<Configuration> out = adaptive_sample(set, vis, p, *s, rng_seed, wrap);
    *out_count = static_cast<int32_t>(out.size());
    for (std::size_t i = 0; i < out.size(); ++i)
      std::memcpy(out_idx + i * d, out[i].indices.data(), d * 4);
    if (k_count) *k_count = nk;
  });
}

int ref_synthesize_sample(void* h, const int32_t* cand_idx, const uint64_t* cand_ids,
                          const double* cand_pred, int64_t n, const uint64_t* visited,
                          int64_t n_visited, uint64_t rng_seed, int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  return guard([&] {
    CandidateSet set = candidates_from(*s, cand_idx, cand_ids, cand_pred, n);
    VisitedSet vis(visited, visited + n_visited);
    Rng r(rng_seed);
    Configuration c = synthesize_sample(set, *s, vis, r);
    std::memcpy(out, c.indices.data(), d * 4);
  });
}

int ref_greedy_select(void* h, const int32_t* cand_idx, const uint64_t* cand_ids,
                      const double* cand_pred, int64_t n, int batch, int32_t* out) {
  auto* s = static_cast<DesignSpace*>(h);
  const int d = s->num_knobs();
  int cnt = 0;
  int rc = guard([&] {
    CandidateSet set = candidates_from(*s, cand_idx, cand_ids, cand_pred, n);
    std::vector<Configuration> r = greedy_select(set, batch);
    for (std::size_t i = 0; i < r.size(); ++i) std::memcpy(out + i * d, r[i].indices.data(), d * 4);
    cnt = static_cast<int>(r.size());
  });
  return rc == 0 ? cnt : -rc;
}

}  // extern "C"
