// make_candidate_set on the device (sampling.cpp:16-31):
//   ids = id_of(row) (design_space.cpp:158-167, mixed radix, last knob fastest)
//   dedup by id, FIRST occurrence wins  -> stable radix sort of (id, row) by id,
//                                          keep the head of every equal-id run
//   rank by (predicted desc, id asc)    -> the kept rows are already in id order;
//                                          a stable radix sort on the descending
//                                          fitness key keeps id order within ties
// Radix sorts: CUB (CUDA toolkit CCCL) DeviceRadixSort — library primitive.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "internal.cuh"

namespace {

__global__ void ids_kernel(KtSpaceParams sp, const uint16_t* __restrict__ idx, int64_t n,
                           uint64_t* __restrict__ ids, int64_t* __restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t id = 0;
    for (int d = 0; d < sp.D; ++d) id = id * (uint64_t)sp.card[d] + (uint64_t)idx[i * sp.D + d];
    ids[i] = id;
    rows[i] = i;
  }
}

__global__ void head_flags_kernel(const uint64_t* __restrict__ ids, int64_t n, uint8_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || ids[i] != ids[i - 1]) ? 1 : 0;
}

// Descending order on doubles as an ascending unsigned key.
__device__ __forceinline__ uint64_t desc_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 ties with +0.0 as in the reference comparator
  uint64_t b = (uint64_t)__double_as_longlong(x);
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending total order
  return ~b;                                          // descending
}

__global__ void rank_keys_kernel(const int64_t* __restrict__ rows, const double* __restrict__ pred, int64_t m,
                                 uint64_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = desc_key(pred[rows[i]]);
}

__global__ void gather_ids_kernel(const int64_t* __restrict__ rows, const uint64_t* __restrict__ ids_by_row,
                                  int64_t m, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ids_by_row[rows[i]];
}

}  // namespace

namespace kt {
// make_candidate_set over n > 0 device rows: *d_rows_out (kept rows in CandidateSet order)
// and *d_ids_by_row (id of every input row) point into the WS_SCRATCH workspace, valid
// until the next call; returns the kept count.
int64_t candidate_rows_dev(ktune_ctx* ctx, const ktune_space* space, const uint16_t* d_idx, const double* d_pred,
                           int64_t n, int64_t** d_rows_out, uint64_t** d_ids_by_row) {
  if (n > (int64_t)INT32_MAX) fail(KTUNE_ERR_CONFIG, "make_candidate_set: at most 2^31-1 rows per call");
  cudaStream_t s = ctx->stream;
  // scratch: ids_row[n] (id per original row), keys/vals ping-pong, flags
  char* base = (char*)ctx->dev(kt::WS_SCRATCH, (size_t)n * (8 * 5 + 8 + 1) + 256);
  uint64_t* ids_row = (uint64_t*)base;
  uint64_t* k0 = ids_row + n;
  uint64_t* k1 = k0 + n;
  int64_t* v0 = (int64_t*)(k1 + n);
  int64_t* v1 = v0 + n;
  int64_t* kept = v1 + n;
  uint8_t* flag = (uint8_t*)(kept + n);
  int64_t* d_count = (int64_t*)ctx->dev(kt::WS_VALID, 64);
  const int th = 256;
  const int grid = (int)std::min<int64_t>(kt::ceil_div(n, th), (int64_t)kt::sm_count(ctx) * 16);
  ids_kernel<<<grid, th, 0, s>>>(space->params, d_idx, n, ids_row, v0);
  KT_CUDA(cudaMemcpyAsync(k0, ids_row, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
  // 1) stable sort (id, row) by id
  cub::DoubleBuffer<uint64_t> keys(k0, k1);
  cub::DoubleBuffer<int64_t> vals(v0, v1);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, (int)n, 0, 64, s);
  void* d_tmp = ctx->dev(kt::WS_SCRATCH2, tmp + 256);
  KT_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, keys, vals, (int)n, 0, 64, s));
  // 2) first occurrence of every id
  head_flags_kernel<<<grid, th, 0, s>>>(keys.Current(), n, flag);
  size_t tmp2 = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp2, vals.Current(), flag, kept, d_count, (int)n, s);
  d_tmp = ctx->dev(kt::WS_SCRATCH2, std::max(tmp, tmp2) + 256);
  KT_CUDA(cub::DeviceSelect::Flagged(d_tmp, tmp2, vals.Current(), flag, kept, d_count, (int)n, s));
  int64_t m = 0;
  KT_CUDA(cudaMemcpyAsync(&m, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  KT_CUDA(cudaStreamSynchronize(s));
  // 3) stable sort of the id-ordered kept rows by descending predicted fitness
  rank_keys_kernel<<<grid, th, 0, s>>>(kept, d_pred, m, k0);
  cub::DoubleBuffer<uint64_t> keys2(k0, k1);
  cub::DoubleBuffer<int64_t> vals2(kept, v0);
  size_t tmp3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp3, keys2, vals2, (int)m, 0, 64, s);
  d_tmp = ctx->dev(kt::WS_SCRATCH2, std::max(std::max(tmp, tmp2), tmp3) + 256);
  KT_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp3, keys2, vals2, (int)m, 0, 64, s));
  check_launch(ctx, "make_candidate_set", 5);
  *d_rows_out = vals2.Current();
  *d_ids_by_row = ids_row;
  return m;
}
}  // namespace kt

extern "C" int ktune_candidates_from_rows(ktune_ctx* ctx, const ktune_space* space, const uint16_t* idx,
                                          const double* pred, int64_t n, int64_t* out_rows, uint64_t* out_ids,
                                          int64_t* out_n, int flags) {
  return kt_guard(ctx, [&] {
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
