// Internal definitions shared by the libktune_cuda translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ktune_cuda.h"

namespace kt {

constexpr int kMaxKnobs = 32;   // device kernels keep one config in registers/smem
constexpr int kMaxRuleOps = 64; // postfix program length passed by value
constexpr int kMaxK = 64;       // k-means clusters (sweep is [8, 64))

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define KT_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      ::kt::fail(e_ == cudaErrorMemoryAllocation ? KTUNE_ERR_NOMEM : KTUNE_ERR_CUDA,      \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

// Device buffer owned by a context workspace slot (grow-only).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      KT_CUDA(cudaMalloc(&p, need < 256 ? 256 : need));
      bytes = need < 256 ? 256 : need;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      KT_CUDA(cudaMallocHost(&p, need < 4096 ? 4096 : need));
      bytes = need < 4096 ? 4096 : need;
    }
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

enum WsSlot {
  WS_IN0, WS_IN1, WS_IN2, WS_OUT0, WS_OUT1, WS_OUT2, WS_OUT3, WS_OUT4,
  WS_D2, WS_D2B, WS_ASSIGN, WS_ASSIGN2, WS_MEMBERS, WS_BLOCK, WS_BLOCK2, WS_CENT, WS_CENT2,
  WS_SCRATCH, WS_SCRATCH2, WS_KPP, WS_SNAP, WS_VALID, WS_TASKS, WS_BEST_ASSIGN, WS_BEST_D2,
  WS_PREV_ASSIGN, WS_PREV_D2, WS_SORTED, WS_XS_APPROX, WS_XS_MAPS, WS_TILESUM, WS_ROLLOUT, WS_XS_RB, WS_KM_CERT, WS_KPP_X, WS_CERT_SNAP, WS_CAND_LOCAL, WS_CAND_SEND, WS_CAND_RECV, WS_CAND_OUT, WS_NUM_SLOTS
};

}  // namespace kt

struct ktune_ctx {
  int device = 0;
  int rank = 0;
  int world = 1;
  void* nccl = nullptr;  // ncclComm_t
  // Host-memory collectives supplied by the caller (ktune_ctx_create_hostcomm): the same
  // sharded code paths as NCCL, with every exchange staged through pinned host memory
  // (multi-process tests on one GPU; gloo or any host transport underneath).
  ktune_host_allreduce_fn hc_allreduce = nullptr;
  ktune_host_allgather_fn hc_allgather = nullptr;
  void* hc_user = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H of segmented rollouts, overlapping the compute
  unsigned int* d_progress = nullptr;  // streamed rollouts: per segment, the slots that finished it
  void* fn_wait_value = nullptr;       // cuStreamWaitValue32 (driver entry point), resolved once
  int wait_value_state = 0;            // 0 unresolved, 1 available, -1 unavailable
  int64_t opt_rollout_streamed = 0;    // 0 auto (streamed when available), 1 off
  std::string last_error;
  int64_t opt_force_exact = 0;
  int64_t opt_force_sharded = 0;
  int64_t opt_kmeans_bound_log2 = 0;  // tests: inflate the certified k-means bounds by 2^v (forces rescues)  // k-means: the NCCL-sharded path on one rank (tests)
  int64_t opt_kmeans_mode = 0;
  int64_t opt_profile = 0;
  int64_t opt_rollout_delta = 0;  // 1e-12 units, 0 = default
  int64_t opt_rollout_check = 0;
  int64_t opt_rollout_fuse_gbt = 0;
  int64_t opt_rollout_segments = 0;  // 0 auto  // 1: GBT walk inside the rollout kernel instead of a separate K1
  static constexpr int kNumStats = 32;
  int64_t stats[kNumStats] = {0};
  unsigned long long* d_counters = nullptr;  // device counters of the tcgen05 rollout (4 x u64)
  struct PendingTiming {
    cudaEvent_t a, b;
    int stat_ns;
  };
  std::vector<PendingTiming> pending;  // resolved lazily by ktune_ctx_stat
  int64_t cand_count = -1;  // rows of the last ktune_candidates_gather result (WS_CAND_OUT)
  kt::DevBuf ws[kt::WS_NUM_SLOTS];
  kt::HostBuf pinned[4];
  void* dev(int slot, size_t bytes) { return ws[slot].get(bytes); }
  void* host(int slot, size_t bytes) { return pinned[slot].get(bytes); }
  void count_launch(int n = 1) { stats[KTUNE_STAT_LAUNCHES] += n; }
};

// Device-side view of a design space, passed to kernels by value.
struct KtSpaceParams {
  int32_t D;
  int32_t nops;
  int32_t card[kt::kMaxKnobs];
  int32_t lut_off[kt::kMaxKnobs + 1];  // offsets into the feature LUT (sum of cards)
  int32_t val_off[kt::kMaxKnobs + 1];  // offsets into the knob values
  const double* lut;                   // feature LUT: idx / (card - 1) (0 for card 1)
  const int64_t* values;               // knob values (validity rule operands)
  int32_t op_code[kt::kMaxRuleOps];
  int64_t op_arg[kt::kMaxRuleOps];
};

struct ktune_space {
  ktune_ctx* ctx = nullptr;
  int D = 0;
  std::vector<int32_t> card;
  std::vector<int64_t> values;
  std::vector<int64_t> val_off;
  std::vector<ktune_rule_op> ops;
  std::vector<double> lut;  // host copy of the feature LUT
  unsigned __int128 size = 0;
  double* d_lut = nullptr;
  int64_t* d_values = nullptr;
  KtSpaceParams params{};
  int lut_total = 0;
  bool validate(const int32_t* idx) const;
};

// Complete-tree layout of a GBT ensemble.
struct ktune_gbt {
  ktune_ctx* ctx = nullptr;
  int num_trees = 0;
  int num_features = 0;
  int depth = 0;          // padded depth of every tree (complete binary trees)
  double base = 0.0;
  double lr = 0.0;
  bool has_space = false;
  int D = 0;
  int idx_card_max = 0;
  // device arrays
  uint32_t* d_inode_idx = nullptr;  // [T][2^depth - 1] (feature << 24) | idx threshold t1
  uint32_t* d_inode_pk = nullptr;   // [T][2^depth - 1] (column byte offset << 16) | t1 (fast path)
  double* d_inode_thr = nullptr;    // [T][2^depth - 1] fp64 thresholds (feature path)
  int32_t* d_inode_feat = nullptr;  // [T][2^depth - 1]
  double* d_leaf = nullptr;         // [T][2^depth]
  // generic pointer-walk layout when depth > kMaxCompleteDepth
  int32_t* d_offsets = nullptr;
  ktune_tree_node* d_nodes = nullptr;
  bool complete = true;
};

struct ktune_ac {
  ktune_ctx* ctx = nullptr;
  int n = 0, h = 0, g = 0;
  int64_t num_params = 0;
  double* d_params = nullptr;
  std::vector<double> host_params;
  uint64_t version = 1;  // bumped whenever host_params change (ppo_update)
  // tcgen05 rollout: power-of-two weight scales for (version, space), computed once
  mutable uint64_t scale_version = 0;
  mutable const ktune_space* scale_space = nullptr;
  mutable int scale_e[3] = {0, 0, 0};
};

namespace kt {

// ---------------------------------------------------------------- helpers
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count(ktune_ctx* ctx);

// Copy host->device (when !device) through pinned staging, returns device ptr.
const void* stage_in(ktune_ctx* ctx, int slot, const void* src, size_t bytes, bool device);
void* out_buf(ktune_ctx* ctx, int slot, void* dst, size_t bytes, bool device);
void stage_out(ktune_ctx* ctx, void* dst, const void* dev, size_t bytes, bool device);

void check_launch(ktune_ctx* ctx, const char* what, int n = 1);
void allreduce_sum(ktune_ctx* ctx, void* buf, size_t count, bool is_double);
void allgather(ktune_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank);

}  // namespace kt

void kt_nccl_destroy(ktune_ctx* ctx);

namespace kt {
// Row map of a strided scoring pass: the j-th scored row is
// (j / len) * stride + off + j % len (identity when len == 0).
struct RowMap {
  int64_t len = 0, stride = 0, off = 0;
  __host__ __device__ bool identity() const { return len == 0; }
  __host__ __device__ int64_t operator()(int64_t j) const {
    if (len == 0) return j;
    const uint32_t q = (uint32_t)((uint64_t)j / (uint64_t)len), r = (uint32_t)((uint64_t)j % (uint64_t)len);
    return (int64_t)q * stride + off + r;
  }
};
void gbt_predict_idx_device(ktune_ctx* ctx, const ktune_gbt* g, const void* d_idx, int idx_bytes, int64_t B,
                            double* d_out, RowMap map = RowMap());
struct GbtJob {
  const ktune_gbt* g;
  const void* idx;
  int64_t B;
  double* out;
  RowMap map;
};
// the jobs in one K1 launch (same depth and knob count; else one launch per job)
void gbt_predict_idx_device_multi(ktune_ctx* ctx, const std::vector<GbtJob>& jobs, int idx_bytes);
// One rollout workload with device pointers (shared by the exact and the
// tcgen05 rollout kernels).
struct RolloutWork {
  const ktune_space* space;
  const ktune_ac* ac;
  int64_t E;
  int64_t episode_offset;
  uint64_t seed;
  const uint16_t* init_idx;
  uint16_t* idx;
  int8_t* actions;
  double* logp;
  double* value;
  const ktune_gbt* gbt;  // may be NULL
  double* score;         // E x (T+1), may be NULL
  float* logp32 = nullptr;   // fp32 copies (may be NULL)
  float* value32 = nullptr;
  uint8_t* idx8 = nullptr;   // compact outputs written by the tcgen05 rollout (may be NULL):
  uint32_t* ids = nullptr;   //   uint8 rows (idx layout), configuration ids (score layout),
  uint8_t* act2 = nullptr;   //   2-bit direction codes (actions layout, ceil(n/4) bytes per step)
  bool scored = false;   // set by rollout_tc when the scores were fused into the rollout
  // trajectory layout in rows: (e, t) of idx/score at e*sE + t*sT, of actions/logp/value at
  // e*aE + t*aT (episode-major: T+1, 1, T, 1; step-major, KTUNE_F_STEP_MAJOR: 1, E, 1, E)
  int64_t sE = 0, sT = 1, aE = 0, aT = 1;
};
// tcgen05 rollout (rollout_tc.cu): eligibility (h = 128, g = 64, n <= 21,
// cardinalities <= 2049, representable weight scales) and the launch.
bool rollout_tc_eligible(const ktune_ac* ac, const ktune_space* sp);
// progress/nseg (streamed host-buffer calls): every slot adds 1 to progress[s] when it has
// finished segment s (segment of step x = floor(x nseg / T)); segment s of the whole call is
// complete once progress[s] reaches the returned slot count (summed over the launches).
int64_t rollout_tc(ktune_ctx* ctx, std::vector<RolloutWork>& work, int T, int t_begin, int t_end,
                   unsigned int* progress = nullptr, int nseg = 0);
// Folds the device counters of the tcgen05 rollout into ctx->stats.
void resolve_counters(ktune_ctx* ctx);
}  // namespace kt

namespace kt {
// Brackets one launch with CUDA events on ctx->stream when KTUNE_OPT_PROFILE is set.
struct ProfScope {
  ktune_ctx* ctx;
  int stat_ns;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(ktune_ctx* c, int s) : ctx(c), stat_ns(s) {
    if (!ctx->opt_profile) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, ctx->stream);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, ctx->stream);
    ctx->pending.push_back({a, b, stat_ns});
  }
};
void resolve_timings(ktune_ctx* ctx);
}  // namespace kt

namespace kt {

}  // namespace kt

// Run `body` converting exceptions to status codes.
// NVTX range over a C-ABI call (header-only NVTX v3: a no-op unless a tool such as
// Nsight Systems / ncu --nvtx injects itself).
struct KtRange {
  explicit KtRange(const char* name) { nvtxRangePushA(name); }
  ~KtRange() { nvtxRangePop(); }
};
#define KT_RANGE(name) KtRange kt_range_(name)

template <class F>
int kt_guard(ktune_ctx* ctx, F&& body) {
  try {
    body();
    return KTUNE_OK;
  } catch (const kt::Error& e) {
    if (ctx) ctx->last_error = e.what();
    extern thread_local std::string kt_tls_error;
    kt_tls_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return KTUNE_ERR_NOMEM;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    extern thread_local std::string kt_tls_error;
    kt_tls_error = e.what();
    return KTUNE_ERR_BACKEND;
  }
}
