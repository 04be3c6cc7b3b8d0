// make_candidate_set on the device (sampling.cpp:16-31):
//   ids = id_of(row) (design_space.cpp:158-167, mixed radix, last knob fastest)
//   dedup by id, FIRST occurrence wins  -> stable radix sort of (id, row) by id over
//                                          ceil(log2 |space|) key bits, keep the head of
//                                          every equal-id run (an order-keeping compaction)
//   rank by (predicted desc, id asc)    -> the kept rows are already in id order; a stable
//                                          radix sort on a descending 64-bit image of the
//                                          fitness keeps id order within ties
// Sorts: the hand-written LSD radix sort of radix.cuh. No host round trip inside the
// pipeline: the kept count stays in device memory and sizes the ranking sort's tiles.
#include "internal.cuh"
#include "radix.cuh"

namespace {

template <class K>
__global__ void ids_kernel(KtSpaceParams sp, const uint16_t* __restrict__ idx, int64_t n, uint64_t* __restrict__ ids,
                           K* __restrict__ keys, uint32_t* __restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t id = 0;
    for (int d = 0; d < sp.D; ++d) id = id * (uint64_t)sp.card[d] + (uint64_t)idx[i * sp.D + d];
    ids[i] = id;
    keys[i] = (K)id;
    rows[i] = (uint32_t)i;
  }
}

// Descending order on doubles as an ascending unsigned key.
__device__ __forceinline__ uint64_t desc_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 ties with +0.0 as in the reference comparator
  uint64_t b = (uint64_t)__double_as_longlong(x);
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending total order
  return ~b;                                          // descending
}

constexpr int kCT = kt::rsort::kThreads, kCPer = kt::rsort::kPer, kCTile = kt::rsort::kTile;

// Heads of equal-key runs of the id-sorted keys: per-tile head counts.
template <class K>
__global__ void __launch_bounds__(kCT) head_count_kernel(const K* __restrict__ k, int64_t n, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kCTile;
  uint32_t mine = 0;
  for (int q = 0; q < kCPer; ++q) {
    const int64_t i = base + q * kCT + threadIdx.x;
    if (i < n && (i == 0 || k[i] != k[i - 1])) ++mine;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&c, mine);
  __syncthreads();
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// Exclusive scan of the per-tile counts (one block), total -> *d_m.
__global__ void __launch_bounds__(1024) tile_scan_kernel(uint32_t* __restrict__ cnt, int tiles, int64_t* __restrict__ d_m) {
  __shared__ uint32_t part[1024];
  const int per = (tiles + 1023) / 1024, b0 = threadIdx.x * per, b1 = min(tiles, b0 + per);
  uint32_t s = 0;
  for (int b = b0; b < b1; ++b) s += cnt[b];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (int b = b0; b < b1; ++b) {
    const uint32_t c = cnt[b];
    cnt[b] = run;
    run += c;
  }
  if (threadIdx.x == 1023) *d_m = part[1023];
}

// Order-keeping compaction of the run heads (blocked: thread t owns items t*kCPer..):
// kept[j] = row, key2[j] = desc_key(pred[row]).
template <class K>
__global__ void __launch_bounds__(kCT) head_write_kernel(const K* __restrict__ k, const uint32_t* __restrict__ rows,
                                                         int64_t n, const uint32_t* __restrict__ off,
                                                         const double* __restrict__ pred, uint32_t* __restrict__ kept,
                                                         uint64_t* __restrict__ key2) {
  __shared__ uint32_t part[kCT];
  const int64_t base = (int64_t)blockIdx.x * kCTile + (int64_t)threadIdx.x * kCPer;
  uint32_t mask = 0;
  for (int q = 0; q < kCPer; ++q) {
    const int64_t i = base + q;
    if (i < n && (i == 0 || k[i] != k[i - 1])) mask |= 1u << q;
  }
  const uint32_t c = __popc(mask);
  part[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < kCT; o <<= 1) {
    const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t pos = off[blockIdx.x] + part[threadIdx.x] - c;
  for (int q = 0; q < kCPer; ++q)
    if ((mask >> q) & 1u) {
      const uint32_t r = rows[base + q];
      kept[pos] = r;
      key2[pos] = desc_key(pred[r]);
      ++pos;
    }
}

__global__ void rows_out_kernel(const uint32_t* __restrict__ kept, const int64_t* __restrict__ d_m, int64_t cap,
                                int64_t* __restrict__ out) {
  const int64_t m = *d_m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m && i < cap; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)kept[i];
}

__global__ void gather_ids_kernel(const int64_t* __restrict__ rows, const uint64_t* __restrict__ ids_by_row,
                                  int64_t m, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ids_by_row[rows[i]];
}

template <class K>
int64_t candidate_rows_impl(ktune_ctx* ctx, const ktune_space* space, const uint16_t* d_idx, const double* d_pred,
                            int64_t n, int bits, int64_t** d_rows_out, uint64_t** d_ids_by_row) {
  cudaStream_t s = ctx->stream;
  const int tiles = (int)kt::ceil_div(n, kCTile);
  // workspace: ids_row u64[n] | keys K[2n] | key2 u64[2n] | rows out i64[n] | vals u32[2n] | kept u32[2n] | counts
  const size_t words = kt::rsort::scratch_words(n);
  char* base = (char*)ctx->dev(kt::WS_SCRATCH, (size_t)n * (8 + 2 * sizeof(K) + 16 + 8 + 8 + 8) + 4 * (words + tiles) + 1024);
  uint64_t* ids_row = (uint64_t*)base;
  uint64_t* key2a = ids_row + n;
  uint64_t* key2b = key2a + n;
  int64_t* rows64 = (int64_t*)(key2b + n);
  K* ka = (K*)(rows64 + n);
  K* kb = ka + n;
  uint32_t* va = (uint32_t*)(kb + n);
  uint32_t* vb = va + n;
  uint32_t* kept_a = vb + n;
  uint32_t* kept_b = kept_a + n;
  uint32_t* scratch = kept_b + n;
  uint32_t* tcnt = scratch + words;
  int64_t* d_m = (int64_t*)ctx->dev(kt::WS_VALID, 64);
  const int th = 256;
  const int grid = (int)std::min<int64_t>(kt::ceil_div(n, th), (int64_t)kt::sm_count(ctx) * 16);
  ids_kernel<K><<<grid, th, 0, s>>>(space->params, d_idx, n, ids_row, ka, va);
  // 1) stable sort (id, row) by the id's significant bits
  const bool f1 = kt::rsort::sort_pairs<K>(s, ka, va, kb, vb, nullptr, n, bits, scratch);
  const K* ks = f1 ? kb : ka;
  const uint32_t* vs = f1 ? vb : va;
  // 2) first occurrence of every id, in id order, with its descending fitness key
  head_count_kernel<K><<<tiles, kCT, 0, s>>>(ks, n, tcnt);
  tile_scan_kernel<<<1, 1024, 0, s>>>(tcnt, tiles, d_m);
  head_write_kernel<K><<<tiles, kCT, 0, s>>>(ks, vs, n, tcnt, d_pred, kept_a, key2a);
  // 3) stable sort of the kept rows by descending fitness (count from device memory)
  const bool f2 = kt::rsort::sort_pairs<uint64_t>(s, key2a, kept_a, key2b, kept_b, d_m, n, 64, scratch);
  rows_out_kernel<<<grid, th, 0, s>>>(f2 ? kept_b : kept_a, d_m, n, rows64);
  kt::check_launch(ctx, "make_candidate_set", 5 + 3 * ((bits + 7) / 8) + 3 * 8);
  int64_t m = 0;
  KT_CUDA(cudaMemcpyAsync(&m, d_m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  KT_CUDA(cudaStreamSynchronize(s));
  *d_rows_out = rows64;
  *d_ids_by_row = ids_row;
  return m;
}

}  // namespace

namespace kt {
// make_candidate_set over n > 0 device rows: *d_rows_out (kept rows in CandidateSet order)
// and *d_ids_by_row (id of every input row) point into the WS_SCRATCH workspace, valid
// until the next call; returns the kept count.
int64_t candidate_rows_dev(ktune_ctx* ctx, const ktune_space* space, const uint16_t* d_idx, const double* d_pred,
                           int64_t n, int64_t** d_rows_out, uint64_t** d_ids_by_row) {
  if (n > (int64_t)INT32_MAX) fail(KTUNE_ERR_CONFIG, "make_candidate_set: at most 2^31-1 rows per call");
  // significant id bits: ids < |space| (design_space.cpp:13-58 checks it fits 64 bits)
  unsigned __int128 size = 1;
  for (int d = 0; d < space->D; ++d) size *= (unsigned __int128)space->card[d];
  int bits = 0;
  while (bits < 64 && (((unsigned __int128)1) << bits) < size) ++bits;
  if (bits <= 32) return candidate_rows_impl<uint32_t>(ctx, space, d_idx, d_pred, n, bits, d_rows_out, d_ids_by_row);
  return candidate_rows_impl<uint64_t>(ctx, space, d_idx, d_pred, n, bits, d_rows_out, d_ids_by_row);
}
}  // namespace kt

extern "C" int ktune_candidates_from_rows(ktune_ctx* ctx, const ktune_space* space, const uint16_t* idx,
                                          const double* pred, int64_t n, int64_t* out_rows, uint64_t* out_ids,
                                          int64_t* out_n, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_candidates_from_rows");
    if (n < 0) kt::fail(KTUNE_ERR_CONFIG, "make_candidate_set: negative count");
    const bool dev = flags & KTUNE_F_DEVICE;
    if (n == 0) {
      *out_n = 0;
      return;
    }
    const int D = space->D;
    cudaStream_t s = ctx->stream;
    const uint16_t* d_idx = (const uint16_t*)kt::stage_in(ctx, kt::WS_IN0, idx, sizeof(uint16_t) * n * D, dev);
    const double* d_pred = (const double*)kt::stage_in(ctx, kt::WS_IN1, pred, sizeof(double) * n, dev);
    int64_t* rows = nullptr;
    uint64_t* ids_row = nullptr;
    const int64_t m = kt::candidate_rows_dev(ctx, space, d_idx, d_pred, n, &rows, &ids_row);
    const int th = 256;
    const int grid = (int)std::min<int64_t>(kt::ceil_div(std::max<int64_t>(m, 1), th), (int64_t)kt::sm_count(ctx) * 16);
    int64_t* d_rows = (int64_t*)kt::out_buf(ctx, kt::WS_OUT0, out_rows, sizeof(int64_t) * m, dev);
    KT_CUDA(cudaMemcpyAsync(d_rows, rows, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, s));
    if (out_ids && m) {
      uint64_t* d_ids = (uint64_t*)kt::out_buf(ctx, kt::WS_OUT1, out_ids, sizeof(uint64_t) * m, dev);
      gather_ids_kernel<<<grid, th, 0, s>>>(d_rows, ids_row, m, d_ids);
      kt::check_launch(ctx, "gather_ids");
      kt::stage_out(ctx, out_ids, d_ids, sizeof(uint64_t) * m, dev);
    }
    kt::stage_out(ctx, out_rows, d_rows, sizeof(int64_t) * m, dev);
    KT_CUDA(cudaStreamSynchronize(s));
    *out_n = m;
  });
}

// ------------------------------------------------------------------ distributed CandidateSet
// Every rank holds the trajectory of its episode shard. The global CandidateSet (1-GPU
// semantics: dedup by id over ALL rows, rank by (pred desc, id asc)) is the
// make_candidate_set of the union of the per-rank candidate sets: dedup keeps the set of
// distinct ids, and every id carries one score (the cost model is a function of the
// configuration), so the union's ranking equals the single-GPU ranking.
namespace {
__global__ void gather_rows_kernel(const int64_t* __restrict__ rows, int64_t m, int D, const uint16_t* __restrict__ idx,
                                   const double* __restrict__ pred, uint16_t* __restrict__ oidx,
                                   double* __restrict__ opred) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[i];
    for (int d = 0; d < D; ++d) oidx[i * D + d] = idx[r * D + d];
    opred[i] = pred[r];
  }
}
}  // namespace

extern "C" int ktune_candidates_gather(ktune_ctx* ctx, const ktune_space* space, const uint16_t* idx,
                                       const double* pred, int64_t n, int64_t* out_n, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_candidates_gather");
    if (n < 0 || !space) kt::fail(KTUNE_ERR_CONFIG, "candidates_gather: bad space or count");
    const bool dev = flags & KTUNE_F_DEVICE;
    const int D = space->D, W = ctx->world;
    cudaStream_t s = ctx->stream;
    const int th = 256;
    auto grid_of = [&](int64_t m) {
      return (int)std::min<int64_t>(kt::ceil_div(std::max<int64_t>(m, 1), th), (int64_t)kt::sm_count(ctx) * 16);
    };
    const uint16_t* d_idx = (const uint16_t*)kt::stage_in(ctx, kt::WS_IN0, idx, sizeof(uint16_t) * n * D, dev);
    const double* d_pred = (const double*)kt::stage_in(ctx, kt::WS_IN1, pred, sizeof(double) * n, dev);
    // 1) this rank's candidate set, compacted (rows in CandidateSet order)
    int64_t m = 0;
    int64_t* rows = nullptr;
    uint64_t* ids_row = nullptr;
    if (n > 0) m = kt::candidate_rows_dev(ctx, space, d_idx, d_pred, n, &rows, &ids_row);
    // 2) counts of every rank
    int64_t* d_cnt = (int64_t*)ctx->dev(kt::WS_CAND_LOCAL, sizeof(int64_t) * (W + 1));
    KT_CUDA(cudaMemcpyAsync(d_cnt + W, &m, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    kt::allgather(ctx, d_cnt + W, d_cnt, sizeof(int64_t));
    std::vector<int64_t> cnt(W);
    KT_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, s));
    KT_CUDA(cudaStreamSynchronize(s));
    int64_t M = 0, total = 0;
    for (int r = 0; r < W; ++r) {
      M = std::max(M, cnt[r]);
      total += cnt[r];
    }
    // 3) padded send rows (idx then pred) -> rank-ordered all-gather
    const size_t row_bytes = sizeof(uint16_t) * D, blk = (size_t)M * (row_bytes + 8);
    char* send = (char*)ctx->dev(kt::WS_CAND_SEND, std::max<size_t>(blk, 16));
    if (m > 0) {
      gather_rows_kernel<<<grid_of(m), th, 0, s>>>(rows, m, D, d_idx, d_pred, (uint16_t*)send,
                                                   (double*)(send + (size_t)M * row_bytes));
      kt::check_launch(ctx, "gather_rows");
    }
    char* recv = (char*)ctx->dev(kt::WS_CAND_RECV, std::max<size_t>(blk * W, 16) + (size_t)total * (row_bytes + 8));
    if (M > 0) kt::allgather(ctx, send, recv, blk);
    // 4) the union, contiguous in rank order
    uint16_t* all_idx = (uint16_t*)(recv + blk * W);
    double* all_pred = (double*)(all_idx + (size_t)total * D);
    int64_t off = 0;
    for (int r = 0; r < W; ++r) {
      if (!cnt[r]) continue;
      KT_CUDA(cudaMemcpyAsync(all_idx + off * D, recv + blk * r, row_bytes * cnt[r], cudaMemcpyDeviceToDevice, s));
      KT_CUDA(cudaMemcpyAsync(all_pred + off, recv + blk * r + (size_t)M * row_bytes, 8 * cnt[r],
                              cudaMemcpyDeviceToDevice, s));
      off += cnt[r];
    }
    // 5) make_candidate_set of the union -> the global CandidateSet (kept in WS_CAND_OUT)
    int64_t g = 0;
    if (total > 0) {
      int64_t* grows = nullptr;
      uint64_t* gids_row = nullptr;
      g = kt::candidate_rows_dev(ctx, space, all_idx, all_pred, total, &grows, &gids_row);
      char* out = (char*)ctx->dev(kt::WS_CAND_OUT, (size_t)g * (row_bytes + 16) + 16);
      uint16_t* oidx = (uint16_t*)out;
      double* opred = (double*)(out + (size_t)g * row_bytes + (8 - ((size_t)g * row_bytes) % 8) % 8);
      uint64_t* oids = (uint64_t*)(opred + g);
      gather_rows_kernel<<<grid_of(g), th, 0, s>>>(grows, g, D, all_idx, all_pred, oidx, opred);
      gather_ids_kernel<<<grid_of(g), th, 0, s>>>(grows, gids_row, g, oids);
      kt::check_launch(ctx, "gather_candidates", 2);
    }
    KT_CUDA(cudaStreamSynchronize(s));
    ctx->cand_count = g;
    *out_n = g;
  });
}

extern "C" int ktune_candidates_gather_copy(ktune_ctx* ctx, const ktune_space* space, uint16_t* out_idx,
                                            double* out_pred, uint64_t* out_ids, int flags) {
  return kt_guard(ctx, [&] {
    if (ctx->cand_count < 0) kt::fail(KTUNE_ERR_CONFIG, "candidates_gather_copy: no gathered candidate set");
    const bool dev = flags & KTUNE_F_DEVICE;
    const int64_t g = ctx->cand_count;
    const size_t row_bytes = sizeof(uint16_t) * space->D;
    char* out = (char*)ctx->dev(kt::WS_CAND_OUT, (size_t)g * (row_bytes + 16) + 16);
    const double* opred = (const double*)(out + (size_t)g * row_bytes + (8 - ((size_t)g * row_bytes) % 8) % 8);
    const uint64_t* oids = (const uint64_t*)(opred + g);
    const cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (g) {
      if (out_idx) KT_CUDA(cudaMemcpyAsync(out_idx, out, row_bytes * g, k, ctx->stream));
      if (out_pred) KT_CUDA(cudaMemcpyAsync(out_pred, opred, 8 * g, k, ctx->stream));
      if (out_ids) KT_CUDA(cudaMemcpyAsync(out_ids, oids, 8 * g, k, ctx->stream));
    }
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------------------------ knob histograms
// knob_options' counting pass (sampling.cpp:249-256) over a candidate set on the
// device: counts[lut_off[d] + v] = #{i : idx[i][d] == v}. Block-private shared
// histograms when the space's total cardinality fits, global atomics otherwise.
namespace {
constexpr int kHistThreads = 256;
constexpr int kHistSmemBins = 12288;

template <class IdxT>
__global__ void __launch_bounds__(kHistThreads) knob_hist_kernel(KtSpaceParams sp, int total, const IdxT* __restrict__ idx,
                                                                 int64_t N, unsigned long long* __restrict__ counts,
                                                                 int use_smem) {
  __shared__ int32_t h[kHistSmemBins];
  const int D = sp.D;
  if (use_smem) {
    for (int i = threadIdx.x; i < total; i += blockDim.x) h[i] = 0;
    __syncthreads();
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N * D; e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const int bin = sp.lut_off[d] + (int)idx[e];
    if (use_smem) atomicAdd(&h[bin], 1);
    else atomicAdd(&counts[bin], 1ull);
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < total; i += blockDim.x)
      if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
  }
}
}  // namespace

namespace kt {
void knob_histogram_device(ktune_ctx* ctx, const ktune_space* space, const void* d_idx, int idx_bytes, int64_t N,
                           unsigned long long* d_counts) {
  const int total = space->lut_total;
  KT_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(unsigned long long) * std::max(1, total), ctx->stream));
  if (N <= 0) return;
  const int use_smem = total <= kHistSmemBins ? 1 : 0;
  const int grid = (int)std::min<int64_t>(ceil_div(N * space->D, kHistThreads), (int64_t)sm_count(ctx) * 8);
  if (idx_bytes == 1)
    knob_hist_kernel<uint8_t><<<grid, kHistThreads, 0, ctx->stream>>>(space->params, total, (const uint8_t*)d_idx,
                                                                      N, d_counts, use_smem);
  else
    knob_hist_kernel<uint16_t><<<grid, kHistThreads, 0, ctx->stream>>>(space->params, total, (const uint16_t*)d_idx,
                                                                       N, d_counts, use_smem);
  check_launch(ctx, "knob_hist");
}
}  // namespace kt

extern "C" int ktune_knob_histogram(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                                    int64_t N, uint64_t* counts, int flags) {
  return kt_guard(ctx, [&] {
    if (!space || N < 0 || (idx_bytes != 1 && idx_bytes != 2))
      kt::fail(KTUNE_ERR_CONFIG, "knob_histogram: bad space, count or index width");
    const bool dev = flags & KTUNE_F_DEVICE;
    const void* d_idx = kt::stage_in(ctx, kt::WS_IN0, idx, (size_t)N * space->D * idx_bytes, dev);
    unsigned long long* d_c = (unsigned long long*)kt::out_buf(ctx, kt::WS_OUT0, counts,
                                                               sizeof(uint64_t) * std::max(1, space->lut_total), dev);
    kt::knob_histogram_device(ctx, space, d_idx, idx_bytes, N, d_c);
    kt::stage_out(ctx, counts, d_c, sizeof(uint64_t) * space->lut_total, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}
