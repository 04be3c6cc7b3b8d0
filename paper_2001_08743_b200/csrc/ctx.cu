// Context, design-space upload, validity-rule compiler and staging helpers.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <string>

#include "device.cuh"
#include "internal.cuh"

thread_local std::string kt_tls_error;

namespace kt {

int sm_count(ktune_ctx* ctx) {
  int n = 0;
  KT_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ctx->device));
  return n;
}

const void* stage_in(ktune_ctx* ctx, int slot, const void* src, size_t bytes, bool device) {
  if (device || bytes == 0) return src;
  void* d = ctx->dev(slot, bytes);
  KT_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return d;
}

void* out_buf(ktune_ctx* ctx, int slot, void* dst, size_t bytes, bool device) {
  if (device) return dst;
  return ctx->dev(slot, bytes);
}

void stage_out(ktune_ctx* ctx, void* dst, const void* dev, size_t bytes, bool device) {
  if (device || bytes == 0 || dst == nullptr) return;
  KT_CUDA(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}

void check_launch(ktune_ctx* ctx, const char* what, int n) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(KTUNE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  ctx->count_launch(n);
}

void resolve_timings(ktune_ctx* ctx) {
  for (auto& t : ctx->pending) {
    cudaEventSynchronize(t.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    ctx->stats[t.stat_ns] += (int64_t)((double)ms * 1e6);
    ctx->stats[t.stat_ns + 1] += 1;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  ctx->pending.clear();
}

}  // namespace kt

// ============================================================ rule compiler
// Tokenizer + recursive-descent parser with the grammar of validity.hpp:10-19,
// producing the postfix program of validity.cpp:124-212 (same op order, same
// error conditions).
namespace {

struct Tok {
  enum K { Num, Name, Plus, Star, LP, RP, Le, Lt, Eq, End } k;
  int64_t num = 0;
  std::string name;
};

std::vector<Tok> tokenize(const std::string& s) {
  std::vector<Tok> out;
  size_t i = 0;
  while (i < s.size()) {
    const char c = s[i];
    if (std::isspace((unsigned char)c)) {
      ++i;
    } else if (std::isdigit((unsigned char)c)) {
      size_t j = i;
      while (j < s.size() && std::isdigit((unsigned char)s[j])) ++j;
      Tok t{Tok::Num};
      t.num = std::stoll(s.substr(i, j - i));
      out.push_back(t);
      i = j;
    } else if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < s.size() && (std::isalnum((unsigned char)s[j]) || s[j] == '_')) ++j;
      Tok t{Tok::Name};
      t.name = s.substr(i, j - i);
      out.push_back(t);
      i = j;
    } else if (c == '+') {
      out.push_back({Tok::Plus});
      ++i;
    } else if (c == '*') {
      out.push_back({Tok::Star});
      ++i;
    } else if (c == '(') {
      out.push_back({Tok::LP});
      ++i;
    } else if (c == ')') {
      out.push_back({Tok::RP});
      ++i;
    } else if (c == '<') {
      if (i + 1 < s.size() && s[i + 1] == '=') {
        out.push_back({Tok::Le});
        i += 2;
      } else {
        out.push_back({Tok::Lt});
        ++i;
      }
    } else if (c == '=' && i + 1 < s.size() && s[i + 1] == '=') {
      out.push_back({Tok::Eq});
      i += 2;
    } else {
      kt::fail(KTUNE_ERR_CONFIG, "validity rule: unexpected character '" + std::string(1, c) +
                                     "' in \"" + s + "\"");
    }
  }
  out.push_back({Tok::End});
  return out;
}

struct Parser {
  const std::vector<Tok>& t;
  size_t pos = 0;
  const std::vector<std::string>& names;
  const std::string& src;
  std::vector<ktune_rule_op> ops;

  void emit(int code, int64_t arg = 0) {
    ktune_rule_op op{};
    op.code = code;
    op.arg = arg;
    ops.push_back(op);
  }
  void atom() {
    const Tok& x = t[pos++];
    if (x.k == Tok::Num) {
      emit(KTUNE_RULE_PUSH_CONST, x.num);
    } else if (x.k == Tok::Name) {
      auto it = std::find(names.begin(), names.end(), x.name);
      if (it == names.end())
        kt::fail(KTUNE_ERR_CONFIG, "validity rule: unknown knob '" + x.name + "' in \"" + src + "\"");
      emit(KTUNE_RULE_PUSH_KNOB, it - names.begin());
    } else if (x.k == Tok::LP) {
      sum();
      if (t[pos++].k != Tok::RP) kt::fail(KTUNE_ERR_CONFIG, "validity rule: missing ')' in \"" + src + "\"");
    } else {
      kt::fail(KTUNE_ERR_CONFIG, "validity rule: expected value in \"" + src + "\"");
    }
  }
  void prod() {
    atom();
    while (t[pos].k == Tok::Star) {
      ++pos;
      atom();
      emit(KTUNE_RULE_MUL);
    }
  }
  void sum() {
    prod();
    while (t[pos].k == Tok::Plus) {
      ++pos;
      prod();
      emit(KTUNE_RULE_ADD);
    }
  }
};

int stack_depth(const ktune_rule_op* ops, int nops) {
  int d = 0, mx = 0;
  for (int i = 0; i < nops; ++i) {
    if (ops[i].code <= KTUNE_RULE_PUSH_KNOB) ++d;
    else --d;
    mx = std::max(mx, d);
  }
  return mx;
}

bool host_rule_eval(const ktune_rule_op* ops, int nops, const int64_t* v) {
  std::vector<__int128> st;
  for (int i = 0; i < nops; ++i) {
    const ktune_rule_op& op = ops[i];
    switch (op.code) {
      case KTUNE_RULE_PUSH_CONST: st.push_back(op.arg); break;
      case KTUNE_RULE_PUSH_KNOB: st.push_back(v[op.arg]); break;
      case KTUNE_RULE_ADD: { __int128 b = st.back(); st.pop_back(); st.back() += b; break; }
      case KTUNE_RULE_MUL: { __int128 b = st.back(); st.pop_back(); st.back() *= b; break; }
      case KTUNE_RULE_LE: { __int128 b = st.back(); st.pop_back(); return st.back() <= b; }
      case KTUNE_RULE_LT: { __int128 b = st.back(); st.pop_back(); return st.back() < b; }
      default: { __int128 b = st.back(); st.pop_back(); return st.back() == b; }
    }
  }
  return true;
}

}  // namespace

bool ktune_space::validate(const int32_t* idx) const {
  if (ops.empty()) return true;
  int64_t v[kt::kMaxKnobs];
  for (int d = 0; d < D; ++d) v[d] = values[val_off[d] + idx[d]];
  return host_rule_eval(ops.data(), (int)ops.size(), v);
}

extern "C" {

int ktune_abi_version(void) { return KTUNE_ABI_VERSION; }

const char* ktune_last_error(const ktune_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : kt_tls_error.c_str();
}

int ktune_rule_compile(const char* source, int num_knobs, const char* const* knob_names,
                       ktune_rule_op* ops, int* nops, char* err, int errlen) {
  const int rc = kt_guard(nullptr, [&] {
    const std::string src = source ? source : "";
    std::vector<std::string> names;
    for (int i = 0; i < num_knobs; ++i) names.emplace_back(knob_names[i]);
    std::vector<Tok> toks = tokenize(src);
    Parser p{toks, 0, names, src, {}};
    p.sum();
    const Tok& cmp = toks[p.pos++];
    int code;
    if (cmp.k == Tok::Le) code = KTUNE_RULE_LE;
    else if (cmp.k == Tok::Lt) code = KTUNE_RULE_LT;
    else if (cmp.k == Tok::Eq) code = KTUNE_RULE_EQ;
    else kt::fail(KTUNE_ERR_CONFIG, "validity rule: expected comparison operator in \"" + src + "\"");
    p.sum();
    p.emit(code);
    if (toks[p.pos].k != Tok::End) kt::fail(KTUNE_ERR_CONFIG, "validity rule: trailing input in \"" + src + "\"");
    if ((int)p.ops.size() > *nops) kt::fail(KTUNE_ERR_CONFIG, "validity rule: program longer than capacity");
    std::copy(p.ops.begin(), p.ops.end(), ops);
    *nops = (int)p.ops.size();
  });
  if (rc && err && errlen > 0) {
    std::snprintf(err, (size_t)errlen, "%s", kt_tls_error.c_str());
  }
  return rc;
}

int ktune_rule_eval(const ktune_rule_op* ops, int nops, const int64_t* knob_values) {
  return host_rule_eval(ops, nops, knob_values) ? 1 : 0;
}

int ktune_ctx_create(int device, ktune_ctx** out) {
  return ktune_ctx_create_dist(device, 0, 1, nullptr, out);
}

int ktune_ctx_destroy(ktune_ctx* ctx) {
  if (!ctx) return KTUNE_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->ws) b.release();
  for (auto& b : ctx->pinned) b.release();
  if (ctx->d_counters) cudaFree(ctx->d_counters);
  if (ctx->d_progress) cudaFree(ctx->d_progress);
  kt_nccl_destroy(ctx);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return KTUNE_OK;
}

int ktune_ctx_set_stream(ktune_ctx* ctx, void* s) {
  return kt_guard(ctx, [&] { ctx->stream = s ? (cudaStream_t)s : ctx->own_stream; });
}

void* ktune_ctx_stream(ktune_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int ktune_ctx_synchronize(ktune_ctx* ctx) {
  return kt_guard(ctx, [&] { KT_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int ktune_ctx_set_option(ktune_ctx* ctx, int option, int64_t value) {
  return kt_guard(ctx, [&] {
    if (option == KTUNE_OPT_FORCE_EXACT) ctx->opt_force_exact = value;
    else if (option == KTUNE_OPT_KMEANS_MODE) ctx->opt_kmeans_mode = value;
    else if (option == KTUNE_OPT_PROFILE) ctx->opt_profile = value;
    else if (option == KTUNE_OPT_ROLLOUT_DELTA) ctx->opt_rollout_delta = value;
    else if (option == KTUNE_OPT_ROLLOUT_CHECK) ctx->opt_rollout_check = value;
    else if (option == KTUNE_OPT_ROLLOUT_FUSE_GBT) ctx->opt_rollout_fuse_gbt = value;
    else if (option == KTUNE_OPT_ROLLOUT_SEGMENTS) ctx->opt_rollout_segments = value;
    else if (option == KTUNE_OPT_FORCE_SHARDED) ctx->opt_force_sharded = value;
    else if (option == KTUNE_OPT_KMEANS_BOUND_LOG2) ctx->opt_kmeans_bound_log2 = value;
    else if (option == KTUNE_OPT_ROLLOUT_STREAMED) ctx->opt_rollout_streamed = value;
    else kt::fail(KTUNE_ERR_CONFIG, "unknown option");
  });
}

int ktune_ctx_stat(ktune_ctx* ctx, int stat, int64_t* value) {
  return kt_guard(ctx, [&] {
    if (stat < 0 || stat >= ktune_ctx::kNumStats) kt::fail(KTUNE_ERR_CONFIG, "unknown stat");
    kt::resolve_timings(ctx);
    kt::resolve_counters(ctx);
    *value = ctx->stats[stat];
  });
}

int ktune_ctx_reset_stats(ktune_ctx* ctx) {
  return kt_guard(ctx, [&] {
    kt::resolve_timings(ctx);
    kt::resolve_counters(ctx);
    std::fill(std::begin(ctx->stats), std::end(ctx->stats), 0);
  });
}

// ------------------------------------------------------------ design space
int ktune_space_create(ktune_ctx* ctx, int D, const int32_t* card, const int64_t* values_flat,
                       const ktune_rule_op* ops, int nops, ktune_space** out) {
  return kt_guard(ctx, [&] {
    if (D < 1) kt::fail(KTUNE_ERR_CONFIG, "design space: needs at least one knob");
    if (D > kt::kMaxKnobs) kt::fail(KTUNE_ERR_CONFIG, "design space: at most 32 knobs on the device path");
    auto* s = new ktune_space();
    s->ctx = ctx;
    s->D = D;
    s->card.assign(card, card + D);
    s->val_off.assign(D + 1, 0);
    unsigned __int128 size = 1;
    for (int d = 0; d < D; ++d) {
      if (card[d] < 1) { delete s; kt::fail(KTUNE_ERR_CONFIG, "knob values must be non-empty"); }
      if (card[d] > 65536) { delete s; kt::fail(KTUNE_ERR_CONFIG, "knob cardinality > 65536 unsupported on the device path"); }
      s->val_off[d + 1] = s->val_off[d] + card[d];
      size *= (unsigned __int128)card[d];
      if (size >> 64) { delete s; kt::fail(KTUNE_ERR_CONFIG, "design space: size overflows 64 bits"); }
    }
    s->size = size;
    s->values.assign(values_flat, values_flat + s->val_off[D]);
    for (int d = 0; d < D; ++d)
      for (int i = s->val_off[d] + 1; i < s->val_off[d + 1]; ++i)
        if (s->values[i] <= s->values[i - 1]) {
          delete s;
          kt::fail(KTUNE_ERR_CONFIG, "knob values not strictly increasing");
        }
    if (nops > kt::kMaxRuleOps || (nops > 0 && stack_depth(ops, nops) > 16)) {
      delete s;
      kt::fail(KTUNE_ERR_CONFIG, "validity rule too long for the device evaluator");
    }
    s->ops.assign(ops, ops + nops);
    // Feature LUT: x = (double)i / (double)(card - 1), 0 for card 1 (design_space.cpp:195-197).
    s->lut.clear();
    for (int d = 0; d < D; ++d)
      for (int i = 0; i < card[d]; ++i)
        s->lut.push_back(card[d] > 1 ? (double)i / (double)(card[d] - 1) : 0.0);
    s->lut_total = (int)s->lut.size();
    cudaSetDevice(ctx->device);
    KT_CUDA(cudaMalloc(&s->d_lut, sizeof(double) * s->lut.size()));
    KT_CUDA(cudaMemcpy(s->d_lut, s->lut.data(), sizeof(double) * s->lut.size(), cudaMemcpyHostToDevice));
    KT_CUDA(cudaMalloc(&s->d_values, sizeof(int64_t) * s->values.size()));
    KT_CUDA(cudaMemcpy(s->d_values, s->values.data(), sizeof(int64_t) * s->values.size(), cudaMemcpyHostToDevice));
    KtSpaceParams& p = s->params;
    std::memset(&p, 0, sizeof(p));
    p.D = D;
    p.nops = nops;
    for (int d = 0; d < D; ++d) p.card[d] = card[d];
    for (int d = 0; d <= D; ++d) {
      p.lut_off[d] = (int32_t)s->val_off[d];
      p.val_off[d] = (int32_t)s->val_off[d];
    }
    p.lut = s->d_lut;
    p.values = s->d_values;
    for (int i = 0; i < nops; ++i) {
      p.op_code[i] = ops[i].code;
      p.op_arg[i] = ops[i].arg;
    }
    *out = s;
  });
}

int ktune_space_destroy(ktune_space* s) {
  if (!s) return KTUNE_OK;
  if (s->d_lut) cudaFree(s->d_lut);
  if (s->d_values) cudaFree(s->d_values);
  delete s;
  return KTUNE_OK;
}

int ktune_space_id_of(const ktune_space* s, const int32_t* idx, int64_t n, uint64_t* out) {
  return kt_guard(s->ctx, [&] {
    for (int64_t i = 0; i < n; ++i) {
      uint64_t id = 0;
      for (int d = 0; d < s->D; ++d) {
        const int32_t v = idx[i * s->D + d];
        if (v < 0 || v >= s->card[d]) kt::fail(KTUNE_ERR_CONFIG, "index out of range");
        id = id * (uint64_t)s->card[d] + (uint64_t)v;
      }
      out[i] = id;
    }
  });
}

int ktune_space_config_at(const ktune_space* s, const uint64_t* ids, int64_t n, int32_t* out) {
  return kt_guard(s->ctx, [&] {
    for (int64_t i = 0; i < n; ++i) {
      uint64_t id = ids[i];
      if ((unsigned __int128)id >= s->size) kt::fail(KTUNE_ERR_CONFIG, "ordinal out of range");
      for (int d = s->D - 1; d >= 0; --d) {
        out[i * s->D + d] = (int32_t)(id % (uint64_t)s->card[d]);
        id /= (uint64_t)s->card[d];
      }
    }
  });
}

int ktune_space_validate(const ktune_space* s, const int32_t* idx, int64_t n, uint8_t* out) {
  return kt_guard(s->ctx, [&] {
    for (int64_t i = 0; i < n; ++i) {
      for (int d = 0; d < s->D; ++d) {
        const int32_t v = idx[i * s->D + d];
        if (v < 0 || v >= s->card[d]) kt::fail(KTUNE_ERR_CONFIG, "index out of range");
      }
      out[i] = s->validate(idx + i * s->D) ? 1 : 0;
    }
  });
}

}  // extern "C"
