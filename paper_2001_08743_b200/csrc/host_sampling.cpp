// Host side of Adaptive Sampling: make_candidate_set (sampling.cpp:16-31),
// sample synthesis (sampling.cpp:243-403) and the full adaptive_sample
// (sampling.cpp:409-461) around the device sweep + snap.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <queue>
#include <set>
#include <unordered_set>
#include <vector>

#include "internal.cuh"

namespace {

inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
inline uint64_t seed_combine(uint64_t a, uint64_t b) { return mix64(a + 0x9E3779B97F4A7C15ULL + mix64(b)); }
inline uint64_t stream_seed(uint64_t root, const char* name) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* p = (const unsigned char*)name; *p; ++p) {
    h ^= *p;
    h *= 0x100000001B3ULL;
  }
  return seed_combine(root, h);
}

struct Rng {  // rng.hpp:50-69
  uint64_t s;
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ULL;
    return mix64(s);
  }
  double uniform01() { return (double)(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    const uint64_t t = (0 - n) % n;
    for (;;) {
      const uint64_t r = next();
      if (r >= t) return r % n;
    }
  }
};

uint64_t id_of(const ktune_space* s, const int32_t* idx) {
  uint64_t id = 0;
  for (int d = 0; d < s->D; ++d) id = id * (uint64_t)s->card[d] + (uint64_t)idx[d];
  return id;
}

void config_at(const ktune_space* s, uint64_t id, int32_t* out) {
  for (int d = s->D - 1; d >= 0; --d) {
    out[d] = (int32_t)(id % (uint64_t)s->card[d]);
    id /= (uint64_t)s->card[d];
  }
}

std::vector<int> referenced_knobs(const ktune_space* s) {  // validity.hpp:33, validity.cpp:159-161,210
  std::vector<int> r;
  for (const auto& op : s->ops)
    if (op.code == KTUNE_RULE_PUSH_KNOB && std::find(r.begin(), r.end(), (int)op.arg) == r.end())
      r.push_back((int)op.arg);
  std::sort(r.begin(), r.end());
  return r;
}

struct KnobOption {
  int32_t index;
  int count;
};

// knob_options (sampling.cpp:249-269): per knob, observed indices ordered by
// (count desc, index asc).
// Ordering of per-knob counts (counts[lut_off[d] + v], e.g. from the device histogram).
std::vector<std::vector<KnobOption>> options_from_counts(const ktune_space* s, const uint64_t* counts) {
  std::vector<std::vector<KnobOption>> out(s->D);
  int off = 0;
  for (int d = 0; d < s->D; ++d) {
    for (int v = 0; v < s->card[d]; ++v)
      if (counts[off + v] > 0) out[d].push_back({v, (int)counts[off + v]});
    off += s->card[d];
    std::sort(out[d].begin(), out[d].end(), [](const KnobOption& a, const KnobOption& b) {
      if (a.count != b.count) return a.count > b.count;
      return a.index < b.index;
    });
  }
  return out;
}

std::vector<std::vector<KnobOption>> knob_options(const ktune_space* s, const int32_t* cand, int64_t n) {
  std::vector<std::vector<KnobOption>> out(s->D);
  for (int d = 0; d < s->D; ++d) {
    std::vector<int> cnt(s->card[d], 0);
    for (int64_t i = 0; i < n; ++i) ++cnt[cand[i * s->D + d]];
    for (int v = 0; v < s->card[d]; ++v)
      if (cnt[v] > 0) out[d].push_back({v, cnt[v]});
    std::sort(out[d].begin(), out[d].end(), [](const KnobOption& a, const KnobOption& b) {
      if (a.count != b.count) return a.count > b.count;
      return a.index < b.index;
    });
  }
  return out;
}

// best_valid_assembly (sampling.cpp:276-343).
bool best_valid_assembly(const ktune_space* s, const std::vector<std::vector<KnobOption>>& opts,
                         std::vector<int32_t>& result) {
  const int n = s->D;
  auto materialize = [&](const std::vector<int>& ranks) {
    std::vector<int32_t> c(n);
    for (int k = 0; k < n; ++k) c[k] = opts[k][ranks[k]].index;
    return c;
  };
  auto score_of = [&](const std::vector<int>& ranks) {
    long long sc = 0;
    for (int k = 0; k < n; ++k) sc += opts[k][ranks[k]].count;
    return sc;
  };
  const std::vector<int> base(n, 0);
  if (s->ops.empty()) {
    result = materialize(base);
    return true;
  }
  struct Entry {
    long long score;
    std::vector<int32_t> indices;
    std::vector<int> ranks;
  };
  struct Worse {
    bool operator()(const Entry& a, const Entry& b) const {
      if (a.score != b.score) return a.score < b.score;
      return a.indices > b.indices;
    }
  };
  std::priority_queue<Entry, std::vector<Entry>, Worse> q;
  std::set<std::vector<int>> pushed;
  auto push = [&](const std::vector<int>& r) {
    if (!pushed.insert(r).second) return;
    q.push({score_of(r), materialize(r), r});
  };
  push(base);
  const std::vector<int> mut = referenced_knobs(s);
  int expansions = 0;
  while (!q.empty() && expansions < 200000) {
    ++expansions;
    const Entry e = q.top();
    q.pop();
    if (s->validate(e.indices.data())) {
      result = e.indices;
      return true;
    }
    for (int k : mut)
      if ((size_t)(e.ranks[k] + 1) < opts[k].size()) {
        std::vector<int> nx = e.ranks;
        ++nx[k];
        push(nx);
      }
  }
  return false;
}

using Visited = std::unordered_set<uint64_t>;

// random_valid_unvisited (sampling.cpp:347-377).
void random_valid_unvisited(const ktune_space* s, const Visited& vis, Rng& rng, int32_t* out) {
  const uint64_t size = (uint64_t)s->size;
  std::vector<int32_t> c(s->D);
  if (s->size <= 65536) {
    std::vector<uint64_t> pool;
    for (uint64_t id = 0; id < size; ++id) {
      if (vis.count(id)) continue;
      config_at(s, id, c.data());
      if (s->validate(c.data())) pool.push_back(id);
    }
    if (pool.empty()) kt::fail(KTUNE_ERR_EXHAUSTED, "every valid configuration has been measured");
    config_at(s, pool[rng.below(pool.size())], out);
    return;
  }
  for (int a = 0; a < 10000; ++a) {
    const uint64_t id = rng.below(size);
    if (vis.count(id)) continue;
    config_at(s, id, c.data());
    if (s->validate(c.data())) {
      std::memcpy(out, c.data(), sizeof(int32_t) * s->D);
      return;
    }
  }
  const uint64_t start = rng.below(size);
  for (uint64_t step = 0; step < size; ++step) {
    const uint64_t id = (start + step) % size;
    if (vis.count(id)) continue;
    config_at(s, id, c.data());
    if (s->validate(c.data())) {
      std::memcpy(out, c.data(), sizeof(int32_t) * s->D);
      return;
    }
  }
  kt::fail(KTUNE_ERR_EXHAUSTED, "every valid configuration has been measured");
}

// synthesize_sample (sampling.cpp:379-403).
void synthesize_with(const ktune_space* s, const std::vector<std::vector<KnobOption>>& opts, const Visited& vis,
                     Rng& rng, int32_t* out) {
  std::vector<int32_t> asm_cfg;
  const bool have = best_valid_assembly(s, opts, asm_cfg);
  if (have && !vis.count(id_of(s, asm_cfg.data()))) {
    std::memcpy(out, asm_cfg.data(), sizeof(int32_t) * s->D);
    return;
  }
  if (have) {
    const int attempts = 2 * s->D;
    std::vector<int32_t> p(s->D);
    for (int a = 0; a < attempts; ++a) {
      const int knob = (int)rng.below((uint64_t)s->D);
      const int dir = rng.uniform01() < 0.5 ? -1 : 1;
      p = asm_cfg;  // neighbor (design_space.cpp:175-187), saturating
      int v = p[knob] + dir;
      v = std::max(0, std::min(s->card[knob] - 1, v));
      p[knob] = v;
      if (!vis.count(id_of(s, p.data())) && s->validate(p.data())) {
        std::memcpy(out, p.data(), sizeof(int32_t) * s->D);
        return;
      }
    }
  }
  random_valid_unvisited(s, vis, rng, out);
}

void synthesize(const ktune_space* s, const int32_t* cand, int64_t n, const Visited& vis, Rng& rng,
                int32_t* out) {
  if (n == 0) kt::fail(KTUNE_ERR_CONFIG, "synthesize_sample: empty candidate set");
  synthesize_with(s, knob_options(s, cand, n), vis, rng, out);
}

}  // namespace

extern "C" {

int ktune_make_candidate_set(ktune_ctx* ctx, const uint64_t* ids, const double* pred, int64_t n,
                             int64_t* out_rows, int64_t* out_n) {
  return kt_guard(ctx, [&] {
    std::vector<int64_t> rows(n);
    std::iota(rows.begin(), rows.end(), 0);
    // first occurrence by id wins (sampling.cpp:19-25)
    std::stable_sort(rows.begin(), rows.end(), [&](int64_t a, int64_t b) { return ids[a] < ids[b]; });
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
      if (i == 0 || ids[rows[i]] != ids[rows[i - 1]]) rows[m++] = rows[i];
    rows.resize(m);
    std::sort(rows.begin(), rows.end(), [&](int64_t a, int64_t b) {  // sampling.cpp:26-29
      if (pred[a] != pred[b]) return pred[a] > pred[b];
      return ids[a] < ids[b];
    });
    std::memcpy(out_rows, rows.data(), sizeof(int64_t) * m);
    *out_n = m;
  });
}

int ktune_synthesize_sample(const ktune_space* space, const int32_t* cand_idx, int64_t N,
                            const uint64_t* visited, int64_t n_visited, uint64_t* rng_state,
                            int32_t* out) {
  return kt_guard(space ? space->ctx : nullptr, [&] {
    Visited vis(visited, visited + n_visited);
    Rng rng{*rng_state};
    synthesize(space, cand_idx, N, vis, rng, out);
    *rng_state = rng.s;
  });
}

int ktune_adaptive_sample(ktune_ctx* ctx, const ktune_space* space, const int32_t* cand_idx,
                          const uint64_t* cand_ids, int64_t N, const uint64_t* visited,
                          int64_t n_visited, const ktune_sampling_params* params, uint64_t rng_seed,
                          int32_t* out_idx, int32_t* out_count) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_adaptive_sample");
    if (N == 0) kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: empty candidate set");
    const int D = space->D;
    const int ib = *std::max_element(space->card.begin(), space->card.end()) <= 256 ? 1 : 2;
    std::vector<uint8_t> packed((size_t)N * D * ib);
    for (int64_t i = 0; i < N * D; ++i) {
      if (ib == 1) packed[i] = (uint8_t)cand_idx[i];
      else reinterpret_cast<uint16_t*>(packed.data())[i] = (uint16_t)cand_idx[i];
    }
    int32_t k = 0;
    std::vector<int32_t> snapped((size_t)kt::kMaxK * D);
    std::vector<double> cent((size_t)kt::kMaxK * D);
    ktune_sweep_out so{};
    so.k = &k;
    so.centroids = cent.data();
    so.snapped = snapped.data();
    const int rc = ktune_adaptive_sweep(ctx, space, packed.data(), ib, cand_ids, N, params, rng_seed, &so, 0);
    if (rc != KTUNE_OK) throw kt::Error(rc, ctx->last_error);
    Visited vis(visited, visited + n_visited);
    Rng rng{stream_seed(rng_seed, "synthesis")};  // sampling.cpp:454
    // knob_options is a function of the candidate set alone (sampling.cpp:384): its
    // counting pass runs once, on the device, the first time a snapped config is visited
    std::vector<std::vector<KnobOption>> opts;
    for (int c = 0; c < k; ++c) {
      int32_t* cfg = snapped.data() + (size_t)c * D;
      if (!vis.count(id_of(space, cfg))) continue;
      if (opts.empty()) {
        std::vector<uint64_t> counts(std::max(1, space->lut_total));
        const int rh = ktune_knob_histogram(ctx, space, packed.data(), ib, N, counts.data(), 0);
        if (rh != KTUNE_OK) throw kt::Error(rh, ctx->last_error);
        opts = options_from_counts(space, counts.data());
      }
      synthesize_with(space, opts, vis, rng, cfg);
    }
    std::memcpy(out_idx, snapped.data(), sizeof(int32_t) * k * D);
    *out_count = k;
  });
}

}  // extern "C"
