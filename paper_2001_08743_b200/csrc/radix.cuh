// Hand-written stable LSD radix sort of (key, uint32 value) pairs on the device, for
// make_candidate_set (sampling.cpp:16-31): the id sort (keys = ids_of the visited
// configurations, only ceil(log2 |space|) bits) and the ranking sort (keys = an
// order-preserving 64-bit image of the predicted fitness, descending).
//
// 8-bit digits; a pass over n items = three kernels:
//   rs_hist   one 2048-item tile per block: the tile's 256-bin digit histogram,
//             written digit-major (hist[d * tiles + b]);
//   rs_scan   one block per digit: exclusive scan of that digit's per-tile counts
//             (hist becomes tile offsets within the digit) + the digit total;
//   rs_scatter one tile per block: every item's stable rank inside the tile (rounds of
//             256 items in index order; warp ranks by __match_any_sync, earlier warps'
//             counts from shared memory), the tile sorted by digit in shared memory, then
//             written out in runs: position = digit base (scan of the 256 totals) + the
//             tile's offset within the digit + rank within the tile's run — consecutive
//             threads write consecutive addresses.
// The item count may live in device memory (d_n): grids are sized for the capacity and
// tiles past the count do nothing, so a pipeline of sorts needs no host round trip.
#pragma once

#include <cstdint>

namespace kt {
namespace rsort {

constexpr int kThreads = 256, kPer = 8, kTile = kThreads * kPer, kBins = 256;

template <class K>
__device__ __forceinline__ uint32_t digit(K k, int shift) {
  return (uint32_t)(k >> shift) & 0xFFu;
}

__device__ __forceinline__ int64_t count_of(const int64_t* d_n, int64_t n) { return d_n ? *d_n : n; }

template <class K>
__global__ void __launch_bounds__(kThreads) rs_hist(const K* __restrict__ keys, const int64_t* d_n, int64_t n_cap,
                                                    int shift, int tiles_cap, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kBins];
  const int64_t n = count_of(d_n, n_cap);
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  if (base < n) {
#pragma unroll 4
    for (int k = 0; k < kPer; ++k) {
      const int64_t i = base + k * kThreads + threadIdx.x;
      if (i < n) atomicAdd(&h[digit(keys[i], shift)], 1u);
    }
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * tiles_cap + blockIdx.x] = h[threadIdx.x];
}

// Block d: exclusive scan of hist[d][0 .. tiles) in place, total -> totals[d].
__global__ void __launch_bounds__(kThreads) rs_scan(uint32_t* __restrict__ hist, const int64_t* d_n, int64_t n_cap,
                                                    int tiles_cap, uint32_t* __restrict__ totals) {
  __shared__ uint32_t part[kThreads];
  const int64_t n = count_of(d_n, n_cap);
  const int tiles = (int)((n + kTile - 1) / kTile);
  uint32_t* h = hist + (int64_t)blockIdx.x * tiles_cap;
  const int per = (tiles + kThreads - 1) / kThreads;  // contiguous chunk per thread
  const int b0 = threadIdx.x * per, b1 = min(tiles, b0 + per);
  uint32_t s = 0;
  for (int b = b0; b < b1; ++b) s += h[b];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {  // inclusive Hillis-Steele scan of the chunk sums
    const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s;
  for (int b = b0; b < b1; ++b) {
    const uint32_t c = h[b];
    h[b] = run;
    run += c;
  }
  if (threadIdx.x == kThreads - 1) totals[blockIdx.x] = part[kThreads - 1];
}

template <class K>
__global__ void __launch_bounds__(kThreads) rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                       const int64_t* d_n, int64_t n_cap, int shift, int tiles_cap,
                                                       const uint32_t* __restrict__ hist,
                                                       const uint32_t* __restrict__ totals) {
  __shared__ K sk[kTile];
  __shared__ uint32_t sv[kTile];
  __shared__ uint32_t dstart[kBins];   // tile-local start of each digit's run
  __shared__ uint32_t gbase[kBins];    // global position of the tile's run of each digit
  __shared__ uint32_t running[kBins];  // items of each digit placed so far (rounds)
  __shared__ uint32_t wcnt[kThreads / 32][kBins];
  __shared__ uint32_t scan[kBins];
  const int64_t n = count_of(d_n, n_cap);
  const int64_t base = (int64_t)blockIdx.x * kTile;
  if (base >= n) return;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int cnt = n - base < kTile ? (int)(n - base) : kTile;
  // digit base = exclusive scan of the 256 totals (every block redundantly)
  scan[t] = totals[t];
  running[t] = 0;
#pragma unroll
  for (int q = 0; q < kThreads / 32; ++q) wcnt[q][t] = 0;
  __syncthreads();
  for (int o = 1; o < kBins; o <<= 1) {
    const uint32_t v = t >= o ? scan[t - o] : 0u;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  gbase[t] = scan[t] - totals[t] + hist[(int64_t)t * tiles_cap + blockIdx.x];
  // the tile's own digit histogram -> run starts
  __syncthreads();
  scan[t] = 0;
  __syncthreads();
  for (int k = 0; k < kPer; ++k) {
    const int i = k * kThreads + t;
    if (i < cnt) atomicAdd(&scan[digit(kin[base + i], shift)], 1u);
  }
  __syncthreads();
  {
    const uint32_t c = scan[t];
    __syncthreads();
    for (int o = 1; o < kBins; o <<= 1) {
      const uint32_t v = t >= o ? scan[t - o] : 0u;
      __syncthreads();
      scan[t] += v;
      __syncthreads();
    }
    dstart[t] = scan[t] - c;
  }
  __syncthreads();
  // stable ranks: rounds of 256 consecutive items
  for (int k = 0; k < kPer; ++k) {
    const int i = k * kThreads + t;
    const bool live = i < cnt;
    K key = 0;
    uint32_t val = 0, d = 0xFFFFFFFFu;
    if (live) {
      key = kin[base + i];
      val = vin[base + i];
      d = digit(key, shift);
    }
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int lrank = __popc(mask & ((1u << lane) - 1u));
    const bool leader = lrank == 0;
    if (live && leader) wcnt[w][d] = __popc(mask);
    __syncthreads();
    if (live) {
      uint32_t before = running[d];
      for (int q = 0; q < w; ++q) before += wcnt[q][d];
      const uint32_t pos = dstart[d] + before + (uint32_t)lrank;
      sk[pos] = key;
      sv[pos] = val;
    }
    __syncthreads();
    {  // thread t owns digit t: fold this round's warp counts into running[t]
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < kThreads / 32; ++q) {
        s += wcnt[q][t];
        wcnt[q][t] = 0;
      }
      running[t] += s;
    }
    __syncthreads();
  }
  // write out the digit runs: tile position p -> gbase[d] + (p - dstart[d])
  for (int k = 0; k < kPer; ++k) {
    const int p = k * kThreads + t;
    if (p < cnt) {
      const K key = sk[p];
      const uint32_t d = digit(key, shift);
      const uint32_t g = gbase[d] + (uint32_t)(p - (int)dstart[d]);
      kout[g] = key;
      vout[g] = sv[p];
    }
  }
}

// Scratch: hist (256 x tiles) + totals (256) words.
inline size_t scratch_words(int64_t n_cap) {
  const int64_t tiles = (n_cap + kTile - 1) / kTile;
  return (size_t)kBins * (size_t)(tiles < 1 ? 1 : tiles) + kBins;
}

// Stable sort of (k0, v0) by key bits [0, bits); ping-pongs with (k1, v1). Returns true
// when the result is in (k1, v1). d_n: device item count (or nullptr: n_cap items).
template <class K>
bool sort_pairs(cudaStream_t s, K* k0, uint32_t* v0, K* k1, uint32_t* v1, const int64_t* d_n, int64_t n_cap, int bits,
                uint32_t* scratch) {
  if (n_cap <= 0 || bits <= 0) return false;
  const int tiles = (int)((n_cap + kTile - 1) / kTile);
  uint32_t* hist = scratch;
  uint32_t* totals = scratch + (size_t)kBins * tiles;
  bool flip = false;
  for (int shift = 0; shift < bits; shift += 8) {
    const K* ki = flip ? k1 : k0;
    const uint32_t* vi = flip ? v1 : v0;
    K* ko = flip ? k0 : k1;
    uint32_t* vo = flip ? v0 : v1;
    rs_hist<K><<<tiles, kThreads, 0, s>>>(ki, d_n, n_cap, shift, tiles, hist);
    rs_scan<<<kBins, kThreads, 0, s>>>(hist, d_n, n_cap, tiles, totals);
    rs_scatter<K><<<tiles, kThreads, 0, s>>>(ki, vi, ko, vo, d_n, n_cap, shift, tiles, hist, totals);
    flip = !flip;
  }
  return flip;
}

}  // namespace rsort
}  // namespace kt
