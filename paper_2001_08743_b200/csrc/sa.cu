// K7: parallel simulated annealing (sa_search, SPEC.md:229-237 — the AutoTVM
// baseline Chameleon's Adaptive Exploration replaces).
// No reference code exists: the semantics are builder-pinned in
// oracle/ktune_oracle.c ko_sa_search and reproduced here
// bit-for-bit: counter-RNG proposal (knob, direction), saturating move, exact
// fp64 cost-model score of the proposal (the K1 walk, cost_model.cpp:179-187),
// Metropolis acceptance with the portable exp, geometric cooling.
//
// Layout: one thread = one chain. The ensemble is staged in shared memory
// (complete-tree node words carrying this block's column byte offset, fp64
// leaves); the chain's configuration lives in a thread-private shared-memory
// column (conflict-free lookups whichever knob a node tests). Per step only
// the proposed knob changes: write it, walk the trees, keep or restore.
#include <algorithm>

#include "device.cuh"
#include "internal.cuh"

namespace {

constexpr int kSaThreads = 128;
constexpr int kMaxSaTasks = 12;

struct SaTask {
  int32_t card[kt::kMaxKnobs];
  int32_t D, T;
  int64_t E, chain_offset;
  uint64_t seed;
  double t0, rate;
  const uint32_t* gnode;  // (feature << 24) | t1 (ktune_gbt::d_inode_idx), complete trees
  const double* gleaf;
  int32_t ntrees, depth;
  double base, lr;
  const uint16_t* init_idx;
  uint16_t* idx;
  double* score;
  uint8_t* accepted;
  int32_t cta_base;
  int32_t row_vec;  // 8: uint4 row stores, 2: uint32, 1: uint16 (from D and the idx alignment)
};

struct SaLaunch {
  int32_t num_tasks;
  SaTask task[kMaxSaTasks];
};

__host__ __device__ inline size_t sa_smem_bytes(int D, int ntrees, int depth) {
  return (size_t)ntrees * (8u << depth) + (((size_t)ntrees * 4 * ((1u << depth) - 1) + 15) & ~(size_t)15) +
         (size_t)D * kSaThreads * 4;
}

// One ensemble evaluation of the chain's column: the trees are walked G at a
// time level by level (G independent smem chains in flight per thread), then
// their leaves are added in tree order — the reference's sequential sum
// (cost_model.cpp:179-187) — and scaled: base + lr * sum.
template <int DEPTH>
__device__ __forceinline__ double walk(const uint32_t* __restrict__ s_node, const double* __restrict__ s_leaf,
                                       const unsigned char* col, int ntrees, double base, double lr) {
  constexpr int NI = (1 << DEPTH) - 1, NL = 1 << DEPTH, G = 8;
  double s = 0.0;
  int tr = 0;
  for (; tr + G <= ntrees; tr += G) {
    int nd[G];
#pragma unroll
    for (int g = 0; g < G; ++g) nd[g] = 0;
#pragma unroll
    for (int l = 0; l < DEPTH; ++l) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t w = s_node[(tr + g) * NI + nd[g]];
        const uint32_t v = *reinterpret_cast<const uint32_t*>(col + (w >> 16));
        nd[g] = 2 * nd[g] + 1 + (v >= w ? 1 : 0);  // tagged column entry vs node word: one compare
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) s = kt::dadd(s, s_leaf[(tr + g) * NL + (nd[g] - NI)]);
  }
  for (; tr < ntrees; ++tr) {
    int nd = 0;
#pragma unroll
    for (int l = 0; l < DEPTH; ++l) {
      const uint32_t w = s_node[tr * NI + nd];
      const uint32_t v = *reinterpret_cast<const uint32_t*>(col + (w >> 16));
      nd = 2 * nd + 1 + (v >= w ? 1 : 0);
    }
    s = kt::dadd(s, s_leaf[tr * NL + (nd - NI)]);
  }
  return kt::dadd(base, kt::dmul(lr, s));
}

// The chain's configuration (thread-private smem column) -> trajectory row t.
__device__ __forceinline__ void store_row(uint16_t* row, const int32_t* col, int D, int vec) {
  if (vec == 8) {
    for (int d = 0; d < D; d += 8) {
      uint4 q;
      q.x = __byte_perm((uint32_t)col[(d + 0) * kSaThreads], (uint32_t)col[(d + 1) * kSaThreads], 0x5410);
      q.y = __byte_perm((uint32_t)col[(d + 2) * kSaThreads], (uint32_t)col[(d + 3) * kSaThreads], 0x5410);
      q.z = __byte_perm((uint32_t)col[(d + 4) * kSaThreads], (uint32_t)col[(d + 5) * kSaThreads], 0x5410);
      q.w = __byte_perm((uint32_t)col[(d + 6) * kSaThreads], (uint32_t)col[(d + 7) * kSaThreads], 0x5410);
      *reinterpret_cast<uint4*>(row + d) = q;
    }
  } else if (vec == 2) {
    for (int d = 0; d < D; d += 2)
      *reinterpret_cast<uint32_t*>(row + d) =
          __byte_perm((uint32_t)col[d * kSaThreads], (uint32_t)col[(d + 1) * kSaThreads], 0x5410);
  } else {
    for (int d = 0; d < D; ++d) row[d] = (uint16_t)col[d * kSaThreads];
  }
}

template <int DEPTH>
__global__ void __launch_bounds__(kSaThreads) sa_kernel(const __grid_constant__ SaLaunch L) {
  extern __shared__ __align__(16) unsigned char sm[];
  int ti = 0;
  while (ti + 1 < L.num_tasks && L.task[ti + 1].cta_base <= (int)blockIdx.x) ++ti;
  const SaTask& tk = L.task[ti];
  const int D = tk.D, T = tk.T;
  constexpr int NI = (1 << DEPTH) - 1, NL = 1 << DEPTH;
  double* s_leaf = reinterpret_cast<double*>(sm);
  uint32_t* s_node = reinterpret_cast<uint32_t*>(sm + (size_t)tk.ntrees * NL * 8);
  int32_t* s_col = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(s_node) +
                                              (((size_t)tk.ntrees * 4 * NI + 15) & ~(size_t)15));
  for (int i = threadIdx.x; i < tk.ntrees * NL; i += kSaThreads) s_leaf[i] = tk.gleaf[i];
  for (int i = threadIdx.x; i < tk.ntrees * NI; i += kSaThreads) {
    const uint32_t wd = tk.gnode[i];
    s_node[i] = ((uint32_t)((wd >> 24) * kSaThreads * 4) << 16) | min(wd & 0xFFFFFFu, 0xFFFFu);
  }
  __syncthreads();
  const int64_t c = (int64_t)((int)blockIdx.x - tk.cta_base) * kSaThreads + threadIdx.x;
  if (c >= tk.E) return;
  int32_t* col = s_col + threadIdx.x;  // col[d * kSaThreads]
  const unsigned char* colb = reinterpret_cast<const unsigned char*>(col);
  uint16_t* out = tk.idx + c * (int64_t)(T + 1) * D;
  // column entries carry their own byte offset in the high half, (coff << 16) | idx, like the
  // node words (coff << 16) | t1: a node test is one unsigned compare (the K1 encoding)
  for (int d = 0; d < D; ++d) col[d * kSaThreads] = (int32_t)(((uint32_t)(d * kSaThreads * 4) << 16) | tk.init_idx[c * D + d]);
  store_row(out, col, D, tk.row_vec);
  double f = walk<DEPTH>(s_node, s_leaf, colb, tk.ntrees, tk.base, tk.lr);
  double* sc = tk.score + c * (int64_t)(T + 1);
  sc[0] = f;
  double temp = tk.t0;
  const uint64_t gc = (uint64_t)(tk.chain_offset + c);
  for (int t = 0; t < T; ++t) {
    const uint64_t base = (gc * (uint64_t)T + (uint64_t)t) * 3u;
    const double u0 = kt::hash01(tk.seed, base), u1 = kt::hash01(tk.seed, base + 1),
                 u2 = kt::hash01(tk.seed, base + 2);
    const int knob = (int)kt::dmul(u0, (double)D);
    const int dir = u1 < 0.5 ? -1 : 1;
    const int old = col[knob * kSaThreads];
    const int tag = old & ~0xFFFF;
    int v = (old & 0xFFFF) + dir;
    v = v < 0 ? 0 : (v > tk.card[knob] - 1 ? tk.card[knob] - 1 : v);
    col[knob * kSaThreads] = tag | v;
    const double fp = walk<DEPTH>(s_node, s_leaf, colb, tk.ntrees, tk.base, tk.lr);
    const double delta = kt::dsub(fp, f);
    const bool accept = delta >= 0.0 || u2 < kt::kt_exp(kt::ddiv(delta, temp));
    if (accept) f = fp;
    else col[knob * kSaThreads] = old;
    store_row(out + (int64_t)(t + 1) * D, col, D, tk.row_vec);
    sc[t + 1] = f;
    if (tk.accepted) tk.accepted[c * (int64_t)T + t] = accept ? 1 : 0;
    temp = kt::dmul(temp, tk.rate);
  }
}

using SaKernel = void (*)(SaLaunch);
constexpr SaKernel kSaKernels[9] = {sa_kernel<0>, sa_kernel<1>, sa_kernel<2>, sa_kernel<3>, sa_kernel<4>,
                                    sa_kernel<5>, sa_kernel<6>, sa_kernel<7>, sa_kernel<8>};

}  // namespace

extern "C" int ktune_sa_search(ktune_ctx* ctx, int num_tasks, const ktune_sa_task* tasks, int32_t T,
                               const ktune_sa_params* params, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_sa_search");
    if (num_tasks < 0 || T < 0 || !params) kt::fail(KTUNE_ERR_CONFIG, "sa_search: bad task count, steps or params");
    if (!(params->initial_temperature > 0.0) || !(params->cooling_rate > 0.0) || !(params->cooling_rate < 1.0))
      kt::fail(KTUNE_ERR_CONFIG, "sa_search: temperature must be positive and 0 < cooling_rate < 1");
    if (num_tasks == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    std::vector<SaTask> st(num_tasks);
    std::vector<void*> temp;
    auto alloc = [&](size_t bytes) {  // host-pointer calls: stream-ordered device buffers
      void* q = nullptr;
      KT_CUDA(cudaMallocAsync(&q, std::max<size_t>(bytes, 8), ctx->stream));
      temp.push_back(q);
      return q;
    };
    size_t smem = 0;
    for (int k = 0; k < num_tasks; ++k) {
      const ktune_sa_task& t = tasks[k];
      if (!t.space || !t.gbt || !t.idx || !t.score || !t.init_idx || t.num_chains < 0)
        kt::fail(KTUNE_ERR_CONFIG, "sa_search: task needs a space, a cost model, seeds and idx/score outputs");
      const ktune_gbt* g = t.gbt;
      if (!g->has_space || g->num_features != t.space->D)
        kt::fail(KTUNE_ERR_CONFIG, "sa_search: cost model must be uploaded with this design space");
      if (!g->complete || !g->d_inode_idx || g->depth > 8)
        kt::fail(KTUNE_ERR_CONFIG, "sa_search: trees deeper than 8 levels are not supported");
      SaTask& s = st[k];
      const int D = t.space->D;
      for (int d = 0; d < kt::kMaxKnobs; ++d) s.card[d] = d < D ? t.space->card[d] : 1;
      s.D = D;
      s.T = T;
      s.E = t.num_chains;
      s.chain_offset = t.chain_offset;
      s.seed = t.sa_seed;
      s.t0 = params->initial_temperature;
      s.rate = params->cooling_rate;
      s.gnode = g->d_inode_idx;
      s.gleaf = g->d_leaf;
      s.ntrees = g->num_trees;
      s.depth = g->depth;
      s.base = g->base;
      s.lr = g->lr;
      const size_t E = (size_t)t.num_chains;
      if (dev) {
        s.init_idx = t.init_idx;
        s.idx = t.idx;
        s.score = t.score;
        s.accepted = t.accepted;
      } else {
        uint16_t* di = (uint16_t*)alloc(E * D * 2);
        if (E) KT_CUDA(cudaMemcpyAsync(di, t.init_idx, E * D * 2, cudaMemcpyHostToDevice, ctx->stream));
        s.init_idx = di;
        s.idx = (uint16_t*)alloc(E * (T + 1) * D * 2);
        s.score = (double*)alloc(E * (T + 1) * 8);
        s.accepted = t.accepted ? (uint8_t*)alloc(E * T) : nullptr;
      }
      const uintptr_t a = reinterpret_cast<uintptr_t>(s.idx);
      s.row_vec = (D % 8 == 0 && a % 16 == 0) ? 8 : (D % 2 == 0 && a % 4 == 0) ? 2 : 1;
      smem = std::max(smem, sa_smem_bytes(D, g->num_trees, g->depth));
    }
    if (smem > 227 * 1024) kt::fail(KTUNE_ERR_CONFIG, "sa_search: cost model too large for shared memory");
    // one launch per tree depth present (complete trees: the walk is compiled per depth)
    for (int dep = 0; dep <= 8; ++dep) {
      std::vector<SaTask> sel;
      for (const SaTask& s : st)
        if (s.depth == dep) sel.push_back(s);
      if (sel.empty()) continue;
      KT_CUDA(cudaFuncSetAttribute(kSaKernels[dep], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (size_t t0 = 0; t0 < sel.size(); t0 += kMaxSaTasks) {
        SaLaunch L{};
        L.num_tasks = (int)std::min<size_t>(kMaxSaTasks, sel.size() - t0);
        int ctas = 0;
        for (int q = 0; q < L.num_tasks; ++q) {
          L.task[q] = sel[t0 + q];
          L.task[q].cta_base = ctas;
          ctas += (int)kt::ceil_div(sel[t0 + q].E, kSaThreads);
        }
        if (ctas > 0) kSaKernels[dep]<<<(unsigned)ctas, kSaThreads, smem, ctx->stream>>>(L);
      }
    }
    kt::check_launch(ctx, "sa_search");
    if (!dev) {
      for (int k = 0; k < num_tasks; ++k) {
        const ktune_sa_task& t = tasks[k];
        const size_t E = (size_t)t.num_chains, D = (size_t)t.space->D;
        KT_CUDA(cudaMemcpyAsync(t.idx, st[k].idx, E * (T + 1) * D * 2, cudaMemcpyDeviceToHost, ctx->stream));
        KT_CUDA(cudaMemcpyAsync(t.score, st[k].score, E * (T + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (t.accepted) KT_CUDA(cudaMemcpyAsync(t.accepted, st[k].accepted, E * T, cudaMemcpyDeviceToHost, ctx->stream));
      }
      for (void* p : temp) KT_CUDA(cudaFreeAsync(p, ctx->stream));
      KT_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}
