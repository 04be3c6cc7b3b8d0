// ktune_gpu.hpp — header-only C++ adapters that plug libktune_cuda into the
// reference's own interfaces (the drop-in seams of SURVEY.md §8b). Include it
// from code built against the reference headers (/root/reference/proj/include,
// Eigen3) and link libktune_cuda.so.
//
//   ktune::gpu::Context ctx(0);
//   ktune::gpu::Space gs(ctx, space);                     // DesignSpace -> device
//   ktune::Clusterer c = ktune::gpu::make_clusterer(gs, params);   // sampling.hpp:44-46
//   auto configs = ktune::adaptive_sample(cands, visited, params, space, seed, c);
//   Eigen::VectorXd y = ktune::gpu::predict(gs, model, features); // CostModel::predict seam
//
// Errors are mapped back onto the reference's exception types (errors.hpp).
#ifndef KTUNE_GPU_HPP
#define KTUNE_GPU_HPP

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ktune/cost_model.hpp"
#include "ktune/design_space.hpp"
#include "ktune/errors.hpp"
#include "ktune/sampling.hpp"
#include "ktune_cuda.h"

namespace ktune {
namespace gpu {

inline void check(int rc, const ktune_ctx* ctx) {
  if (rc == KTUNE_OK) return;
  const std::string msg = ktune_last_error(ctx);
  switch (rc) {
    case KTUNE_ERR_CONFIG: throw ConfigError(msg);
    case KTUNE_ERR_EXHAUSTED: throw SpaceExhaustedError(msg);
    case KTUNE_ERR_LOGIC: throw std::logic_error(msg);
    default: throw BackendError(msg);
  }
}

class Context {
 public:
  explicit Context(int device = 0) { check(ktune_ctx_create(device, &h_), nullptr); }
  ~Context() { ktune_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ktune_ctx* get() const { return h_; }

 private:
  ktune_ctx* h_ = nullptr;
};

// A DesignSpace uploaded to the device; the validity rule is recompiled from
// its source text (validity.hpp:35) with the library's parser.
class Space {
 public:
  Space(Context& ctx, const DesignSpace& s) : ctx_(ctx), space_(s), serial_(next_serial()) {
    std::vector<int32_t> card;
    std::vector<int64_t> values;
    std::vector<std::string> names;
    for (const Knob& k : s.knobs()) {
      card.push_back(k.cardinality());
      values.insert(values.end(), k.values.begin(), k.values.end());
      names.push_back(k.name);
      max_card_ = std::max(max_card_, k.cardinality());
    }
    std::vector<ktune_rule_op> ops(256);
    int nops = 0;
    if (s.validity_rule().has_value()) {
      std::vector<const char*> cn;
      for (auto& n : names) cn.push_back(n.c_str());
      nops = (int)ops.size();
      char err[256];
      check(ktune_rule_compile(s.validity_rule()->source().c_str(), (int)cn.size(), cn.data(), ops.data(),
                               &nops, err, sizeof(err)),
            nullptr);
    }
    check(ktune_space_create(ctx.get(), s.num_knobs(), card.data(), values.data(), ops.data(), nops, &h_),
          ctx.get());
  }
  ~Space() { ktune_space_destroy(h_); }
  Space(const Space&) = delete;
  Space& operator=(const Space&) = delete;
  ktune_space* get() const { return h_; }
  Context& ctx() const { return ctx_; }
  const DesignSpace& space() const { return space_; }
  int index_bytes() const { return max_card_ <= 256 ? 1 : 2; }
  uint64_t serial() const { return serial_; }  // unique per uploaded space (cache keys)

  // Lattice features back to knob indices: idx = round(x * (card - 1)) is exact
  // for x = idx / (card - 1) (design_space.cpp:195-197).
  std::vector<uint16_t> indices_of(const Eigen::MatrixXd& x) const {
    const int D = space_.num_knobs();
    std::vector<uint16_t> out((size_t)x.rows() * D);
    for (Eigen::Index i = 0; i < x.rows(); ++i)
      for (int d = 0; d < D; ++d) {
        const int card = space_.knobs()[(size_t)d].cardinality();
        const double v = card > 1 ? std::nearbyint(x(i, d) * (double)(card - 1)) : 0.0;
        if (v < 0 || v > card - 1 || (card > 1 && (double)v / (double)(card - 1) != x(i, d)))
          throw ConfigError("gpu clusterer: points are not lattice features of this design space");
        out[(size_t)i * D + d] = (uint16_t)v;
      }
    return out;
  }

 private:
  static uint64_t next_serial() {
    static std::atomic<uint64_t> n{0};
    return ++n;
  }
  Context& ctx_;
  const DesignSpace& space_;
  uint64_t serial_;
  ktune_space* h_ = nullptr;
  int max_card_ = 1;
};

inline std::vector<uint8_t> pack(const Space& s, const std::vector<uint16_t>& idx) {
  std::vector<uint8_t> b(idx.size() * (size_t)s.index_bytes());
  if (s.index_bytes() == 1) {
    for (size_t i = 0; i < idx.size(); ++i) b[i] = (uint8_t)idx[i];
  } else {
    std::memcpy(b.data(), idx.data(), b.size());
  }
  return b;
}

// kmeans_run (sampling.hpp:37-38) on the GPU, same signature semantics.
inline ClusterResult kmeans_run(const Space& s, const Eigen::MatrixXd& points, int k, uint64_t seed,
                                int max_iters = 100, int restarts = 3) {
  const int D = s.space().num_knobs();
  const std::vector<uint16_t> idx = s.indices_of(points);
  const std::vector<uint8_t> b = pack(s, idx);
  ClusterResult r;
  std::vector<double> cent((size_t)std::max(k, 1) * D), il((size_t)max_iters + 1);
  r.assignments.resize((size_t)points.rows());
  int32_t nl = 0;
  double loss = 0.0;
  ktune_kmeans_out out{cent.data(), r.assignments.data(), &loss, il.data(), &nl};
  check(ktune_kmeans_run(s.ctx().get(), s.get(), b.data(), s.index_bytes(), points.rows(), k, seed, max_iters,
                         restarts, &out, 0),
        s.ctx().get());
  r.centroids = Eigen::MatrixXd(k, D);
  for (int c = 0; c < k; ++c)
    for (int d = 0; d < D; ++d) r.centroids(c, d) = cent[(size_t)c * D + d];
  r.l2_loss = loss;
  r.iteration_losses.assign(il.begin(), il.begin() + nl);
  return r;
}

// The designed plug-in point: adaptive_sample(..., const Clusterer&) (sampling.hpp:54-58).
inline Clusterer make_clusterer(const Space& s, const SamplingParams& p) {
  return [&s, p](const Eigen::MatrixXd& points, int k, uint64_t seed) {
    return kmeans_run(s, points, k, seed, p.kmeans_max_iters, p.kmeans_restarts);
  };
}

// A fitted ensemble uploaded to the device ONCE per fit (the K1 layout with integer
// thresholds for this space); reuse it for every predict until the next fit.
class Ensemble {
 public:
  Ensemble(const Space& s, const GbtModel& m) : ctx_(s.ctx().get()), num_features_(m.num_features) {
    std::vector<int32_t> off;
    std::vector<ktune_tree_node> nodes;
    for (const RegressionTree& t : m.trees) {
      off.push_back((int32_t)nodes.size());
      for (const TreeNode& n : t.nodes) {
        ktune_tree_node x{};
        x.feature = n.feature;
        x.left = n.left;
        x.right = n.right;
        x.threshold = n.threshold;
        x.value = n.value;
        nodes.push_back(x);
      }
    }
    off.push_back((int32_t)nodes.size());
    check(ktune_gbt_create(ctx_, s.get(), m.num_features, m.base_prediction, m.learning_rate, (int)m.trees.size(),
                           off.data(), nodes.data(), &h_),
          ctx_);
  }
  ~Ensemble() { ktune_gbt_destroy(h_); }
  Ensemble(const Ensemble&) = delete;
  Ensemble& operator=(const Ensemble&) = delete;
  ktune_gbt* get() const { return h_; }

  // CostModel::predict (cost_model.cpp:231-236): fp64 feature rows.
  Eigen::VectorXd predict(const Eigen::MatrixXd& features) const {
    if (features.rows() && features.cols() != num_features_)
      throw ConfigError("cost model: feature dimension " + std::to_string(features.cols()) +
                        " does not match training dimension " + std::to_string(num_features_));
    std::vector<double> x((size_t)features.rows() * (size_t)features.cols());
    for (Eigen::Index i = 0; i < features.rows(); ++i)
      for (Eigen::Index j = 0; j < features.cols(); ++j) x[(size_t)(i * features.cols() + j)] = features(i, j);
    std::vector<double> y((size_t)features.rows());
    check(ktune_gbt_predict_features(ctx_, h_, x.data(), features.rows(), y.data(), 0), ctx_);
    Eigen::VectorXd out(features.rows());
    for (Eigen::Index i = 0; i < features.rows(); ++i) out[i] = y[(size_t)i];
    return out;
  }

 private:
  ktune_ctx* ctx_;
  int num_features_;
  ktune_gbt* h_ = nullptr;
};

// Fingerprint of a model's complete content (FNV-1a over every field): the ensemble
// cache below is keyed by it, so a refit (new trees) is never served a stale upload.
inline uint64_t model_fingerprint(const GbtModel& m) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ULL;
  };
  mix(&m.base_prediction, 8);
  mix(&m.learning_rate, 8);
  mix(&m.num_features, sizeof(int));
  for (const RegressionTree& t : m.trees) {
    const size_t k = t.nodes.size();
    mix(&k, sizeof(k));
    for (const TreeNode& n : t.nodes) {
      mix(&n.feature, sizeof(int));
      mix(&n.threshold, 8);
      mix(&n.left, sizeof(int));
      mix(&n.right, sizeof(int));
      mix(&n.value, 8);
    }
  }
  return h;
}

// predict_batch / CostModel::predict (cost_model.hpp:62,82) on the GPU. The uploaded
// ensemble is cached per (space, model content) — a handful of live entries per thread —
// so repeated predicts between fits upload nothing.
inline Eigen::VectorXd predict(const Space& s, const GbtModel& m, const Eigen::MatrixXd& features) {
  struct Entry {
    uint64_t space;
    uint64_t fp;
    std::shared_ptr<Ensemble> e;
  };
  static thread_local std::vector<Entry> cache;
  const uint64_t fp = model_fingerprint(m);
  std::shared_ptr<Ensemble> e;
  for (size_t i = 0; i < cache.size(); ++i)
    if (cache[i].space == s.serial() && cache[i].fp == fp) {
      e = cache[i].e;
      std::rotate(cache.begin(), cache.begin() + i, cache.begin() + i + 1);  // most recent first
      break;
    }
  if (!e) {
    e = std::make_shared<Ensemble>(s, m);
    cache.insert(cache.begin(), Entry{s.serial(), fp, e});
    if (cache.size() > 4) cache.pop_back();
  }
  return e->predict(features);
}

}  // namespace gpu
}  // namespace ktune

#endif  // KTUNE_GPU_HPP
