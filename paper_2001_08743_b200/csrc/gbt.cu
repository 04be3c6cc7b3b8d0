// Gradient-boosted-tree cost model: host fit (cost_model.cpp:19-177), device
// upload in a complete-tree layout, and the K1 scoring kernels
// (cost_model.cpp:117-124, 179-199).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "device.cuh"
#include "internal.cuh"

namespace {

constexpr int kMaxCompleteDepth = 8;
constexpr uint32_t kAlwaysLeft = 0xFFFFFFu;

// ---------------------------------------------------------------- host fit
// Restatement of the reference TreeBuilder (cost_model.cpp:19-113).
constexpr double kPureLeafSse = 1e-12;

struct Builder {
  const std::vector<double>& x;  // n x dim row-major
  int dim;
  const std::vector<double>& r;
  int max_depth, min_leaf;
  std::vector<int> order;
  std::vector<ktune_tree_node> nodes;
  std::vector<double> leaf_pred;

  static double node_sse(double sum, double sum_sq, double count) {
    const double sse = sum_sq - sum * sum / count;
    return std::max(0.0, sse);
  }

  int build(std::vector<int>& idx, int depth) {
    const double count = (double)idx.size();
    double sum = 0.0, sum_sq = 0.0;
    for (int i : idx) {
      sum += r[i];
      sum_sq += r[i] * r[i];
    }
    const double mean = sum / count;
    const double parent = node_sse(sum, sum_sq, count);
    auto leaf = [&]() {
      ktune_tree_node n{};
      n.feature = -1;
      n.left = n.right = -1;
      n.value = mean;
      for (int i : idx) leaf_pred[i] = mean;
      nodes.push_back(n);
      return (int)nodes.size() - 1;
    };
    if (depth >= max_depth || (int)idx.size() < 2 * min_leaf || parent <= kPureLeafSse) return leaf();
    int best_f = -1;
    double best_thr = 0.0;
    double best_children = parent - kPureLeafSse;
    std::vector<std::pair<double, double>> col(idx.size());
    for (int f : order) {
      for (size_t j = 0; j < idx.size(); ++j) col[j] = {x[(size_t)idx[j] * dim + f], r[idx[j]]};
      std::sort(col.begin(), col.end());
      double ls = 0.0, lq = 0.0;
      for (size_t j = 1; j < col.size(); ++j) {
        ls += col[j - 1].second;
        lq += col[j - 1].second * col[j - 1].second;
        if (col[j - 1].first == col[j].first) continue;
        const double ln = (double)j;
        const double rn = count - ln;
        if (ln < min_leaf || rn < min_leaf) continue;
        const double ch = node_sse(ls, lq, ln) + node_sse(sum - ls, sum_sq - lq, rn);
        if (ch < best_children) {
          best_children = ch;
          best_f = f;
          best_thr = 0.5 * (col[j - 1].first + col[j].first);
        }
      }
    }
    if (best_f < 0) return leaf();
    std::vector<int> li, ri;
    li.reserve(idx.size());
    ri.reserve(idx.size());
    for (int i : idx) (x[(size_t)i * dim + best_f] <= best_thr ? li : ri).push_back(i);
    nodes.emplace_back();
    const int id = (int)nodes.size() - 1;
    nodes[id].feature = best_f;
    nodes[id].threshold = best_thr;
    const int l = build(li, depth + 1);
    const int rr = build(ri, depth + 1);
    nodes[id].left = l;
    nodes[id].right = rr;
    return id;
  }
};

// Eigen's contiguous VectorXd::sum() order (SSE2 two-packet).
double vec_sum(const std::vector<double>& v, bool squares) {
  const int64_t n = (int64_t)v.size();
  auto f = [&](int64_t i) { return squares ? v[i] * v[i] : v[i]; };
  if (n == 0) return 0.0;
  const int64_t a2 = (n / 4) * 4, a = (n / 2) * 2;
  if (a == 0) {
    double s = f(0);
    for (int64_t i = 1; i < n; ++i) s = s + f(i);
    return s;
  }
  double p0 = f(0), p1 = f(1);
  if (a > 2) {
    double q0 = f(2), q1 = f(3);
    for (int64_t i = 4; i < a2; i += 4) {
      p0 = p0 + f(i);
      p1 = p1 + f(i + 1);
      q0 = q0 + f(i + 2);
      q1 = q1 + f(i + 3);
    }
    p0 = p0 + q0;
    p1 = p1 + q1;
    if (a > a2) {
      p0 = p0 + f(a2);
      p1 = p1 + f(a2 + 1);
    }
  }
  double s = p0 + p1;
  for (int64_t i = a; i < n; ++i) s = s + f(i);
  return s;
}

int tree_depth(const ktune_tree_node* nodes, int n, int node, int guard) {
  if (node < 0 || node >= n || guard > 64) kt::fail(KTUNE_ERR_CONFIG, "cost model: malformed tree");
  if (nodes[node].feature < 0) return 0;
  return 1 + std::max(tree_depth(nodes, n, nodes[node].left, guard + 1),
                      tree_depth(nodes, n, nodes[node].right, guard + 1));
}

// ---------------------------------------------------------------- kernels
// One thread per configuration; the block's knob indices are held in a
// transposed shared-memory tile (conflict-free dynamic indexing), the trees
// in shared memory in complete-binary layout: descend `depth` levels with
// node = 2*node + 1 + (idx[f] >= t1), then add the leaf in tree order.
template <class IdxT>
__global__ void __launch_bounds__(256) gbt_predict_idx_kernel(
    const IdxT* __restrict__ idx, int64_t B, int D, int T, int depth,
    const uint32_t* __restrict__ g_inode, const double* __restrict__ g_leaf, double base,
    double lr, double* __restrict__ out, int use_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int ni = (1 << depth) - 1, nl = 1 << depth;
  double* s_leaf = reinterpret_cast<double*>(smem);
  uint32_t* s_inode = reinterpret_cast<uint32_t*>(s_leaf + (use_smem ? (size_t)T * nl : 0));
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_inode + (use_smem ? (size_t)T * ni : 0));
  const double* leaf = g_leaf;
  const uint32_t* inode = g_inode;
  if (use_smem) {
    for (int i = threadIdx.x; i < T * nl; i += blockDim.x) s_leaf[i] = g_leaf[i];
    for (int i = threadIdx.x; i < T * ni; i += blockDim.x) s_inode[i] = g_inode[i];
    __syncthreads();
    leaf = s_leaf;
    inode = s_inode;
  }
  int32_t* my = s_idx + threadIdx.x;  // column: my[d * blockDim.x]
  const int stride = blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x) {
    const IdxT* row = idx + i * D;
    const int row_bytes = D * (int)sizeof(IdxT);
    if (row_bytes == 16 && (((uintptr_t)row) & 15) == 0) {
      const uint4 v = *reinterpret_cast<const uint4*>(row);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      if (sizeof(IdxT) == 1) {
#pragma unroll
        for (int d = 0; d < 16; ++d) my[d * stride] = (w[d >> 2] >> ((d & 3) * 8)) & 0xFF;
      } else {
#pragma unroll
        for (int d = 0; d < 8; ++d) my[d * stride] = (w[d >> 1] >> ((d & 1) * 16)) & 0xFFFF;
      }
    } else if (row_bytes == 8 && (((uintptr_t)row) & 7) == 0) {
      const uint2 v = *reinterpret_cast<const uint2*>(row);
      const uint32_t w[2] = {v.x, v.y};
      if (sizeof(IdxT) == 1) {
#pragma unroll
        for (int d = 0; d < 8; ++d) my[d * stride] = (w[d >> 2] >> ((d & 3) * 8)) & 0xFF;
      } else {
#pragma unroll
        for (int d = 0; d < 4; ++d) my[d * stride] = (w[d >> 1] >> ((d & 1) * 16)) & 0xFFFF;
      }
    } else {
      for (int d = 0; d < D; ++d) my[d * stride] = (int32_t)row[d];
    }
    double s = 0.0;
    for (int t = 0; t < T; ++t) {
      const uint32_t* tn = inode + (size_t)t * ni;
      int node = 0;
      for (int l = 0; l < depth; ++l) {
        const uint32_t w = tn[node];
        const int f = (int)(w >> 24);
        const int t1 = (int)(w & 0xFFFFFFu);
        node = 2 * node + 1 + (my[f * stride] >= t1 ? 1 : 0);
      }
      s = kt::dadd(s, leaf[(size_t)t * nl + (node - ni)]);
    }
    out[i] = kt::dadd(base, kt::dmul(lr, s));
  }
}

// K1 fast path. Complete trees of compile-time depth; node word = (feature
// column byte offset << 16) | t1, so a level is: LDS node, LDS idx at
// column+offset, compare, 2n+1+right. kScoreCfg configurations per thread (ILP), a
// persistent grid over kScoreCfg*256-config chunks, trees + knob-index columns in smem.
constexpr int kScoreThreads = 256;
constexpr int kScoreCfg = 3;  // configurations per thread (independent walks in flight)
// One launch scores up to kScoreJobs (model, rows) jobs: CTAs [cta_base, cta_base + ctas) serve job j
// (every task of a grouped rollout at once: one tail instead of one per task).
constexpr int kScoreJobs = 16;
struct ScoreJob {
  const void* idx;
  int64_t B;
  int32_t D, T;
  const uint32_t* node;
  const double* leaf;
  double base, lr;
  double* out;
  kt::RowMap map;
  int32_t cta_base, ctas;
};
struct ScoreLaunch {
  int32_t njobs;
  ScoreJob job[kScoreJobs];
};
template <class IdxT, int DEPTH>
__global__ void __launch_bounds__(kScoreThreads) gbt_score_kernel(const __grid_constant__ ScoreLaunch SL) {
  int ji = 0;
  while (ji + 1 < SL.njobs && SL.job[ji + 1].cta_base <= (int)blockIdx.x) ++ji;
  const ScoreJob& J = SL.job[ji];
  const IdxT* __restrict__ idx = reinterpret_cast<const IdxT*>(J.idx);
  const int64_t B = J.B;
  const int D = J.D, T = J.T;
  const uint32_t* __restrict__ g_node = J.node;
  const double* __restrict__ g_leaf = J.leaf;
  const double base = J.base, lr = J.lr;
  double* __restrict__ out = J.out;
  const kt::RowMap map = J.map;
  const int64_t cta = (int)blockIdx.x - J.cta_base, nctas = J.ctas;
  constexpr int NI = (1 << DEPTH) - 1, NL = 1 << DEPTH;
  constexpr int NIP = (NI + 3) & ~3;  // node words per tree, padded: every tree starts 16-byte aligned
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_leaf = reinterpret_cast<double*>(smem);
  uint32_t* s_node = reinterpret_cast<uint32_t*>(s_leaf + (size_t)T * NL);
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_node + (size_t)T * NIP);
  for (int i = threadIdx.x; i < T * NL; i += kScoreThreads) s_leaf[i] = g_leaf[i];
  if constexpr (NIP > 0) {  // depth 0 (single-leaf trees) has no internal nodes
    for (int i = threadIdx.x; i < T * NIP; i += kScoreThreads) {
      const int tr = i / NIP, k = i % NIP;
      s_node[i] = k < NI ? g_node[tr * NI + k] : 0u;
    }
  }
  __syncthreads();
  // Byte offsets inside the dynamic smem window. A column entry carries its own
  // byte offset in the high half, (coff << 16) | idx, so the node test
  // idx >= t1 is ONE unsigned compare against the node word (coff << 16) | t1
  // (the high halves are equal by construction). Node addresses are walked as
  // byte offsets inside the tree (r = 4n).
  const unsigned char* sb = smem;
  const uint32_t nodes = (uint32_t)(reinterpret_cast<const unsigned char*>(s_node) - sb);
  const uint32_t col0 = (uint32_t)(reinterpret_cast<const unsigned char*>(s_idx + threadIdx.x) - sb);
  auto ld32 = [&](uint32_t a) { return *reinterpret_cast<const uint32_t*>(sb + a); };
  constexpr int NC = kScoreCfg;
  for (int64_t c0 = cta * NC * kScoreThreads; c0 < B; c0 += nctas * NC * kScoreThreads) {
    int64_t row[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t j = c0 + q * kScoreThreads + threadIdx.x;
      row[q] = j < B ? map(j) : -1;  // row of the j-th scored configuration
    }
    for (int d = 0; d < D; ++d) {  // transposed columns: thread-private, conflict-free
      const uint32_t tag = (uint32_t)(d * kScoreThreads * 4) << 16;
#pragma unroll
      for (int q = 0; q < NC; ++q)
        s_idx[(q * D + d) * kScoreThreads + threadIdx.x] =
            (int32_t)(tag | (row[q] >= 0 ? (uint32_t)idx[row[q] * D + d] : 0u));
    }
    double s[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) s[q] = 0.0;
#pragma unroll 2
    for (int t = 0; t < T; ++t) {
      const uint32_t tb = nodes + (uint32_t)(t * NIP * 4);
      uint32_t r[NC];  // byte offset of the current node inside the tree: 4n
      if constexpr (DEPTH >= 2) {
        // levels 0 and 1 from ONE broadcast 16-byte load of nodes 0..3 (shared by all configs)
        const uint4 q01 = *reinterpret_cast<const uint4*>(sb + tb);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const uint32_t v = ld32(col0 + (uint32_t)(q * D * kScoreThreads * 4) + (q01.x >> 16));
          const bool right = v >= q01.x;
          const uint32_t w = right ? q01.z : q01.y;
          const uint32_t v1 = ld32(col0 + (uint32_t)(q * D * kScoreThreads * 4) + (w >> 16));
          r[q] = (right ? 16u : 8u) + (v1 >= w ? 8u : 4u);  // 2 * (4n1) + 4|8 with n1 = 1|2
        }
      } else {
#pragma unroll
        for (int q = 0; q < NC; ++q) r[q] = 0;
      }
#pragma unroll
      for (int l = DEPTH >= 2 ? 2 : 0; l < DEPTH; ++l) {
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const uint32_t w = ld32(tb + r[q]);
          const uint32_t v = ld32(col0 + (uint32_t)(q * D * kScoreThreads * 4) + (w >> 16));
          r[q] = 2 * r[q] + (v >= w ? 8u : 4u);  // children of n: 2n+1, 2n+2
        }
      }
      // leaf of node n = r/4 is n - NI; s_leaf sits at smem offset 0
      const uint32_t lb = (uint32_t)(t * NL * 8) - (uint32_t)(NI * 8);
#pragma unroll
      for (int q = 0; q < NC; ++q) s[q] = kt::dadd(s[q], *reinterpret_cast<const double*>(sb + lb + 2 * r[q]));
    }
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (row[q] >= 0) out[row[q]] = kt::dadd(base, kt::dmul(lr, s[q]));
  }
}

// fp64 feature rows (generic CostModel::predict(MatrixXd) seam).
__global__ void __launch_bounds__(256) gbt_predict_feat_kernel(
    const double* __restrict__ x, int64_t B, int F, int T, int depth,
    const int32_t* __restrict__ feat, const double* __restrict__ thr,
    const double* __restrict__ g_leaf, double base, double lr, double* __restrict__ out) {
  const int ni = (1 << depth) - 1, nl = 1 << depth;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* row = x + i * F;
    double s = 0.0;
    for (int t = 0; t < T; ++t) {
      int node = 0;
      for (int l = 0; l < depth; ++l) {
        const size_t k = (size_t)t * ni + node;
        node = 2 * node + 1 + (row[feat[k]] <= thr[k] ? 0 : 1);
      }
      s = kt::dadd(s, g_leaf[(size_t)t * nl + (node - ni)]);
    }
    out[i] = kt::dadd(base, kt::dmul(lr, s));
  }
}

// Generic pointer walk over the reference layout (trees deeper than 8).
template <class IdxT>
__global__ void gbt_predict_walk_kernel(const IdxT* __restrict__ idx, const double* __restrict__ x,
                                        int64_t B, int F, int T, const int32_t* __restrict__ off,
                                        const ktune_tree_node* __restrict__ nodes,
                                        const double* __restrict__ lut,
                                        const int32_t* __restrict__ lut_off, double base, double lr,
                                        double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) {
      const ktune_tree_node* tn = nodes + off[t];
      int node = 0;
      while (tn[node].feature >= 0) {
        const int f = tn[node].feature;
        const double v = idx ? lut[lut_off[f] + (int)idx[i * F + f]] : x[i * F + f];
        node = v <= tn[node].threshold ? tn[node].left : tn[node].right;
      }
      s = kt::dadd(s, tn[node].value);
    }
    out[i] = kt::dadd(base, kt::dmul(lr, s));
  }
}

}  // namespace

namespace kt {

// Launch K1 over device arrays on ctx->stream (also used by the rollout).
void gbt_predict_idx_device(ktune_ctx* ctx, const ktune_gbt* g, const void* d_idx, int idx_bytes,
                            int64_t B, double* d_out, RowMap map) {
  if (B <= 0) return;
  if (!map.identity() && !g->d_inode_pk) fail(KTUNE_ERR_CONFIG, "cost model: strided scoring needs the K1 layout");
  if (!g->has_space) fail(KTUNE_ERR_CONFIG, "cost model: uploaded without a design space; use predict_features");
  const int threads = 256;
  if (!g->complete) fail(KTUNE_ERR_CONFIG, "cost model: trees deeper than 8 levels are not supported on the index path");
  const int ni = (1 << g->depth) - 1, nl = 1 << g->depth;
  const size_t tree_bytes = (size_t)g->num_trees * (ni * 4 + nl * 8);
  if (g->d_inode_pk) {  // K1 fast path (node words padded to a multiple of 4 per tree)
    const size_t smem = (size_t)g->num_trees * (((ni + 3) & ~3) * 4 + nl * 8) + 16 +
                        (size_t)kScoreCfg * g->D * kScoreThreads * 4;
    if (smem <= 200 * 1024) {
      const int per_sm = std::max(1, std::min(8, (int)((220 * 1024) / smem)));
      const int grid = (int)std::min<int64_t>(ceil_div(B, kScoreCfg * kScoreThreads), (int64_t)sm_count(ctx) * per_sm);
      ScoreLaunch SL{};
      SL.njobs = 1;
      SL.job[0] = ScoreJob{d_idx, B, g->D, g->num_trees, g->d_inode_pk, g->d_leaf, g->base, g->lr, d_out, map, 0, grid};
      kt::ProfScope prof(ctx, KTUNE_STAT_GBT_NS);
#define KT_SCORE(T_, DEP)                                                                                    \
  {                                                                                                          \
    auto kern = gbt_score_kernel<T_, DEP>;                                                                   \
    KT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
    kern<<<grid, kScoreThreads, smem, ctx->stream>>>(SL);                                                    \
  }
#define KT_SCORE_D(T_)                         \
  switch (g->depth) {                          \
    case 0: KT_SCORE(T_, 0) break;             \
    case 1: KT_SCORE(T_, 1) break;             \
    case 2: KT_SCORE(T_, 2) break;             \
    case 3: KT_SCORE(T_, 3) break;             \
    case 4: KT_SCORE(T_, 4) break;             \
    case 5: KT_SCORE(T_, 5) break;             \
    case 6: KT_SCORE(T_, 6) break;             \
    case 7: KT_SCORE(T_, 7) break;             \
    default: KT_SCORE(T_, 8) break;            \
  }
      if (idx_bytes == 1) KT_SCORE_D(uint8_t) else KT_SCORE_D(uint16_t)
#undef KT_SCORE_D
#undef KT_SCORE
      check_launch(ctx, "gbt_score");
      return;
    }
  }
  const size_t idx_bytes_smem = (size_t)threads * g->D * 4;
  const bool use_smem = tree_bytes + idx_bytes_smem <= 200 * 1024;
  const size_t smem = (use_smem ? tree_bytes : 0) + idx_bytes_smem;
  const int per_sm = use_smem ? std::max(1, (int)((220 * 1024) / smem)) : 4;
  const int64_t want = ceil_div(B, threads);
  const int grid = (int)std::min<int64_t>(want, (int64_t)sm_count(ctx) * std::min(per_sm, 8));
  kt::ProfScope prof(ctx, KTUNE_STAT_GBT_NS);
  if (idx_bytes == 1) {
    auto k = gbt_predict_idx_kernel<uint8_t>;
    KT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, threads, smem, ctx->stream>>>((const uint8_t*)d_idx, B, g->D, g->num_trees, g->depth,
                                            g->d_inode_idx, g->d_leaf, g->base, g->lr, d_out, use_smem);
  } else {
    auto k = gbt_predict_idx_kernel<uint16_t>;
    KT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, threads, smem, ctx->stream>>>((const uint16_t*)d_idx, B, g->D, g->num_trees, g->depth,
                                            g->d_inode_idx, g->d_leaf, g->base, g->lr, d_out, use_smem);
  }
  check_launch(ctx, "gbt_predict_idx");
}

// Several (model, rows) jobs in ONE K1 launch when they share the tree depth and index width
// (the rollout's tasks): CTAs split in proportion to the rows, so the launch has one tail
// instead of one per task (each per-task launch ran ceil(rounds) of ~3 rounds of chunks).
void gbt_predict_idx_device_multi(ktune_ctx* ctx, const std::vector<GbtJob>& jobs, int idx_bytes) {
  std::vector<GbtJob> live;
  for (const GbtJob& j : jobs)
    if (j.B > 0) live.push_back(j);
  if (live.empty()) return;
  bool same = live.size() <= (size_t)kScoreJobs;
  size_t smem = 0;
  for (const GbtJob& j : live) {
    const ktune_gbt* g = j.g;
    same = same && g->d_inode_pk && g->has_space && g->complete && g->depth == live[0].g->depth &&
           g->D == live[0].g->D;
    const int ni = (1 << g->depth) - 1, nl = 1 << g->depth;
    smem = std::max(smem, (size_t)g->num_trees * (((ni + 3) & ~3) * 4 + nl * 8) + 16 +
                              (size_t)kScoreCfg * g->D * kScoreThreads * 4);
  }
  if (!same || smem > 200 * 1024) {
    for (const GbtJob& j : live) gbt_predict_idx_device(ctx, j.g, j.idx, idx_bytes, j.B, j.out, j.map);
    return;
  }
  const int per_sm = std::max(1, std::min(8, (int)((220 * 1024) / smem)));
  const int64_t slots = (int64_t)sm_count(ctx) * per_sm;
  int64_t rows = 0;
  for (const GbtJob& j : live) rows += j.B;
  ScoreLaunch SL{};
  SL.njobs = (int)live.size();
  int ctas = 0;
  for (size_t q = 0; q < live.size(); ++q) {
    const GbtJob& j = live[q];
    const ktune_gbt* g = j.g;
    const int64_t chunks = ceil_div(j.B, kScoreCfg * kScoreThreads);
    const int c = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (slots * j.B + rows - 1) / rows));
    SL.job[q] = ScoreJob{j.idx, j.B, g->D, g->num_trees, g->d_inode_pk, g->d_leaf, g->base, g->lr, j.out, j.map, ctas, c};
    ctas += c;
  }
  kt::ProfScope prof(ctx, KTUNE_STAT_GBT_NS);
#define KT_SCORE(T_, DEP)                                                                         \
  {                                                                                               \
    auto kern = gbt_score_kernel<T_, DEP>;                                                        \
    KT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<ctas, kScoreThreads, smem, ctx->stream>>>(SL);                                         \
  }
#define KT_SCORE_D(T_)                         \
  switch (live[0].g->depth) {                  \
    case 0: KT_SCORE(T_, 0) break;             \
    case 1: KT_SCORE(T_, 1) break;             \
    case 2: KT_SCORE(T_, 2) break;             \
    case 3: KT_SCORE(T_, 3) break;             \
    case 4: KT_SCORE(T_, 4) break;             \
    case 5: KT_SCORE(T_, 5) break;             \
    case 6: KT_SCORE(T_, 6) break;             \
    case 7: KT_SCORE(T_, 7) break;             \
    default: KT_SCORE(T_, 8) break;            \
  }
  if (idx_bytes == 1) KT_SCORE_D(uint8_t) else KT_SCORE_D(uint16_t)
#undef KT_SCORE_D
#undef KT_SCORE
  check_launch(ctx, "gbt_score");
}

}  // namespace kt

extern "C" {

int ktune_gbt_fit(const double* x, const double* y, int64_t n, int dim, int num_trees,
                  int max_depth, double learning_rate, int min_samples_leaf, uint64_t seed,
                  ktune_gbt_model* out) {
  return kt_guard(nullptr, [&] {
    if (n <= 0) kt::fail(KTUNE_ERR_CONFIG, "cost model: cannot fit on an empty training set");
    if (num_trees <= 0 || max_depth <= 0 || min_samples_leaf <= 0 || learning_rate <= 0.0 ||
        learning_rate > 1.0)
      kt::fail(KTUNE_ERR_CONFIG, "cost model: invalid boosting parameters");
    for (int64_t i = 0; i < n; ++i)
      if (!(y[i] >= 0.0) || !std::isfinite(y[i]))
        kt::fail(KTUNE_ERR_CONFIG, "cost model: fitness must be finite and non-negative");
    std::vector<double> X(x, x + n * dim);
    std::vector<double> Y(y, y + n);
    const double base = vec_sum(Y, false) / (double)n;  // y.mean() (cost_model.cpp:155)
    std::vector<double> r(n);
    for (int64_t i = 0; i < n; ++i) r[i] = Y[i] - base;
    std::vector<int> order(dim);
    std::iota(order.begin(), order.end(), 0);
    uint64_t st = kt::seed_combine(seed, 0x6B74756E65ULL);
    std::vector<std::vector<ktune_tree_node>> trees;
    std::vector<double> sse;
    for (int t = 0; t < num_trees; ++t) {
      std::vector<int> sh = order;
      for (size_t i = sh.size(); i > 1; --i) std::swap(sh[i - 1], sh[kt::rng_below(st, i)]);  // rng.hpp:86-91
      Builder b{X, dim, r, max_depth, min_samples_leaf, sh, {}, std::vector<double>(n, 0.0)};
      std::vector<int> all(n);
      std::iota(all.begin(), all.end(), 0);
      b.build(all, 0);
      for (int64_t i = 0; i < n; ++i) r[i] -= learning_rate * b.leaf_pred[i];
      trees.push_back(std::move(b.nodes));
      sse.push_back(vec_sum(r, true));
    }
    out->num_trees = num_trees;
    out->num_features = dim;
    out->base_prediction = base;
    out->learning_rate = learning_rate;
    size_t total = 0;
    for (auto& t : trees) total += t.size();
    out->tree_offsets = (int32_t*)std::malloc(sizeof(int32_t) * (num_trees + 1));
    out->nodes = (ktune_tree_node*)std::malloc(sizeof(ktune_tree_node) * std::max<size_t>(1, total));
    out->training_sse = (double*)std::malloc(sizeof(double) * num_trees);
    size_t k = 0;
    for (int t = 0; t < num_trees; ++t) {
      out->tree_offsets[t] = (int32_t)k;
      for (auto& nd : trees[t]) out->nodes[k++] = nd;
      out->training_sse[t] = sse[t];
    }
    out->tree_offsets[num_trees] = (int32_t)k;
  });
}

void ktune_gbt_model_free(ktune_gbt_model* m) {
  if (!m) return;
  std::free(m->tree_offsets);
  std::free(m->nodes);
  std::free(m->training_sse);
  m->tree_offsets = nullptr;
  m->nodes = nullptr;
  m->training_sse = nullptr;
}

int ktune_gbt_create(ktune_ctx* ctx, const ktune_space* space, int num_features, double base,
                     double learning_rate, int num_trees, const int32_t* off,
                     const ktune_tree_node* nodes, ktune_gbt** out) {
  return kt_guard(ctx, [&] {
    if (num_trees < 0) kt::fail(KTUNE_ERR_CONFIG, "cost model: negative tree count");
    if (space && space->D != num_features)
      kt::fail(KTUNE_ERR_CONFIG, "cost model: feature dimension " + std::to_string(num_features) +
                                     " does not match the design space's " + std::to_string(space->D));
    int depth = 0;
    for (int t = 0; t < num_trees; ++t) {
      const int n = off[t + 1] - off[t];
      if (n < 1) kt::fail(KTUNE_ERR_CONFIG, "cost model: empty tree");
      for (int k = off[t]; k < off[t + 1]; ++k)
        if (nodes[k].feature >= num_features) kt::fail(KTUNE_ERR_CONFIG, "cost model: feature index out of range");
      depth = std::max(depth, tree_depth(nodes + off[t], n, 0, 0));
    }
    auto* g = new ktune_gbt();
    g->ctx = ctx;
    g->num_trees = num_trees;
    g->num_features = num_features;
    g->base = base;
    g->lr = learning_rate;
    g->has_space = space != nullptr;
    g->D = num_features;
    g->depth = depth;
    g->complete = depth <= kMaxCompleteDepth;
    cudaSetDevice(ctx->device);
    if (g->complete) {
      const int ni = (1 << depth) - 1, nl = 1 << depth;
      std::vector<uint32_t> inode_idx((size_t)num_trees * ni + 1, kAlwaysLeft);
      std::vector<uint32_t> inode_pk((size_t)num_trees * ni + 1, 0xFFFFu);  // always left (idx < 65535)
      std::vector<int32_t> inode_feat((size_t)num_trees * ni + 1, 0);
      std::vector<double> inode_thr((size_t)num_trees * ni + 1, INFINITY);
      std::vector<double> leaf((size_t)num_trees * nl);
      for (int t = 0; t < num_trees; ++t) {
        const ktune_tree_node* tn = nodes + off[t];
        // pos = complete-tree position, nd = reference node id
        std::vector<std::pair<int, int>> stack{{0, 0}};
        std::vector<int> level_of(ni + nl, 0);
        while (!stack.empty()) {
          auto [pos, nd] = stack.back();
          stack.pop_back();
          int level = 0;
          for (int p = pos; p > 0; p = (p - 1) / 2) ++level;
          if (level == depth) {
            leaf[(size_t)t * nl + (pos - ni)] = tn[nd].value;
            continue;
          }
          const size_t k = (size_t)t * ni + pos;
          if (tn[nd].feature < 0) {  // pad a shallow leaf: both children keep its value
            inode_idx[k] = kAlwaysLeft;
            inode_pk[k] = 0xFFFFu;
            inode_feat[k] = 0;
            inode_thr[k] = INFINITY;
            stack.push_back({2 * pos + 1, nd});
            stack.push_back({2 * pos + 2, nd});
          } else {
            const int f = tn[nd].feature;
            const double thr = tn[nd].threshold;
            inode_feat[k] = f;
            inode_thr[k] = thr;
            if (space) {
              // t1 = 1 + max{i : lut(i) <= thr}: idx <= thr_idx  <=>  idx < t1
              const int card = space->card[f];
              int t1 = 0;
              for (int i = 0; i < card; ++i)
                if (space->lut[space->val_off[f] + i] <= thr) t1 = i + 1;
              inode_idx[k] = ((uint32_t)f << 24) | (uint32_t)t1;
              inode_pk[k] = ((uint32_t)(f * kScoreThreads * 4) << 16) | (uint32_t)std::min(t1, 65535);
            }
            stack.push_back({2 * pos + 1, tn[nd].left});
            stack.push_back({2 * pos + 2, tn[nd].right});
          }
        }
      }
      KT_CUDA(cudaMalloc(&g->d_inode_idx, sizeof(uint32_t) * inode_idx.size()));
      bool pk_ok = space != nullptr;
      if (space)
        for (int d = 0; d < space->D; ++d) pk_ok = pk_ok && space->card[d] < 65535;
      if (pk_ok) {
        KT_CUDA(cudaMalloc(&g->d_inode_pk, sizeof(uint32_t) * inode_pk.size()));
        KT_CUDA(cudaMemcpy(g->d_inode_pk, inode_pk.data(), sizeof(uint32_t) * inode_pk.size(), cudaMemcpyHostToDevice));
      }
      KT_CUDA(cudaMalloc(&g->d_inode_feat, sizeof(int32_t) * inode_feat.size()));
      KT_CUDA(cudaMalloc(&g->d_inode_thr, sizeof(double) * inode_thr.size()));
      KT_CUDA(cudaMalloc(&g->d_leaf, sizeof(double) * std::max<size_t>(1, leaf.size())));
      KT_CUDA(cudaMemcpy(g->d_inode_idx, inode_idx.data(), sizeof(uint32_t) * inode_idx.size(), cudaMemcpyHostToDevice));
      KT_CUDA(cudaMemcpy(g->d_inode_feat, inode_feat.data(), sizeof(int32_t) * inode_feat.size(), cudaMemcpyHostToDevice));
      KT_CUDA(cudaMemcpy(g->d_inode_thr, inode_thr.data(), sizeof(double) * inode_thr.size(), cudaMemcpyHostToDevice));
      if (!leaf.empty())
        KT_CUDA(cudaMemcpy(g->d_leaf, leaf.data(), sizeof(double) * leaf.size(), cudaMemcpyHostToDevice));
    } else {
      const int total = off[num_trees];
      KT_CUDA(cudaMalloc(&g->d_offsets, sizeof(int32_t) * (num_trees + 1)));
      KT_CUDA(cudaMalloc(&g->d_nodes, sizeof(ktune_tree_node) * total));
      KT_CUDA(cudaMemcpy(g->d_offsets, off, sizeof(int32_t) * (num_trees + 1), cudaMemcpyHostToDevice));
      KT_CUDA(cudaMemcpy(g->d_nodes, nodes, sizeof(ktune_tree_node) * total, cudaMemcpyHostToDevice));
    }
    *out = g;
  });
}

int ktune_gbt_destroy(ktune_gbt* g) {
  if (!g) return KTUNE_OK;
  cudaFree(g->d_inode_idx);
  cudaFree(g->d_inode_pk);
  cudaFree(g->d_inode_feat);
  cudaFree(g->d_inode_thr);
  cudaFree(g->d_leaf);
  cudaFree(g->d_offsets);
  cudaFree(g->d_nodes);
  delete g;
  return KTUNE_OK;
}

int ktune_gbt_predict_idx(ktune_ctx* ctx, const ktune_gbt* g, const void* idx, int idx_bytes,
                          int64_t B, double* out, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_gbt_predict_idx");
    if (idx_bytes != 1 && idx_bytes != 2) kt::fail(KTUNE_ERR_CONFIG, "idx_bytes must be 1 or 2");
    if (B < 0) kt::fail(KTUNE_ERR_CONFIG, "negative batch");
    if (B == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const void* d_idx = kt::stage_in(ctx, kt::WS_IN0, idx, (size_t)B * g->D * idx_bytes, dev);
    double* d_out = (double*)kt::out_buf(ctx, kt::WS_OUT0, out, sizeof(double) * B, dev);
    kt::gbt_predict_idx_device(ctx, g, d_idx, idx_bytes, B, d_out);
    kt::stage_out(ctx, out, d_out, sizeof(double) * B, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_gbt_predict_features(ktune_ctx* ctx, const ktune_gbt* g, const double* x, int64_t B,
                               double* out, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_gbt_predict_features");
    if (B < 0) kt::fail(KTUNE_ERR_CONFIG, "negative batch");
    if (B == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const double* d_x = (const double*)kt::stage_in(ctx, kt::WS_IN0, x, sizeof(double) * B * g->num_features, dev);
    double* d_out = (double*)kt::out_buf(ctx, kt::WS_OUT0, out, sizeof(double) * B, dev);
    const int threads = 256;
    const int grid = (int)std::min<int64_t>(kt::ceil_div(B, threads), (int64_t)kt::sm_count(ctx) * 8);
    if (g->complete) {
      gbt_predict_feat_kernel<<<grid, threads, 0, ctx->stream>>>(d_x, B, g->num_features, g->num_trees,
                                                                 g->depth, g->d_inode_feat, g->d_inode_thr,
                                                                 g->d_leaf, g->base, g->lr, d_out);
    } else {
      gbt_predict_walk_kernel<uint8_t><<<grid, threads, 0, ctx->stream>>>(
          nullptr, d_x, B, g->num_features, g->num_trees, g->d_offsets, g->d_nodes, nullptr, nullptr,
          g->base, g->lr, d_out);
    }
    kt::check_launch(ctx, "gbt_predict_features");
    kt::stage_out(ctx, out, d_out, sizeof(double) * B, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
