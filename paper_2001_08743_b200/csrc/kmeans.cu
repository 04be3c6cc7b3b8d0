// K3-K6: k-means for Adaptive Sampling (sampling.cpp:39-175, 202-235, 409-452).
//
// Exactness contract:
//  * per-point squared distances are computed exactly as the reference
//    (strided Eigen rows => sequential over knobs, no FMA), so every
//    assignment and every d2 value is bit-identical;
//  * centroids are the reference's exact-order sums: members of each cluster
//    are gathered in ascending point order (stable counting sort) and one
//    thread per (cluster, knob) accumulates them sequentially (mode A);
//  * order-sensitive REDUCTIONS that only feed decisions (the kmeans++ total
//    and cumulative scan, restart selection, the sweep's break test) are
//    computed in parallel with a rigorous error bound; a decision whose
//    outcome is not certified by the bound is re-decided by an exact
//    sequential chain that reproduces the reference order bit-for-bit.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "device.cuh"
#include "exactsum.cuh"
#include "tcgen05.cuh"
#include <cuda_fp16.h>
#include "internal.cuh"

namespace {

constexpr int kChunk = 1024;  // points per block-sum chunk (kmeans++ / loss)
constexpr int kBT = 256;      // threads per block for point kernels
// Runs STMT with DM_ = the compile-time knob bound (8 / 16 / 32) covering D.
#define KT_DISPATCH_DM(D, ...)             \
  do {                                     \
    if ((D) <= 8) {                        \
      constexpr int DM_ = 8;               \
      __VA_ARGS__;                         \
    } else if ((D) <= 16) {                \
      constexpr int DM_ = 16;              \
      __VA_ARGS__;                         \
    } else {                               \
      constexpr int DM_ = kt::kMaxKnobs;   \
      __VA_ARGS__;                         \
    }                                      \
  } while (0)
constexpr double kU = 1.1102230246251565e-16;  // 2^-53

template <class IdxT>
__device__ __forceinline__ double feat(const KtSpaceParams& sp, const double* lut_s, const IdxT* p, int d) {
  return lut_s[sp.lut_off[d] + (int)p[d]];
}

// The D knob indices of row p as fp64 features, one 16-byte (or 8-byte) load when the row
// is that wide and aligned (D = 8 uint16 / uint8 rows), else per element.
template <class IdxT, int DM>
__device__ __forceinline__ void load_feats(const KtSpaceParams& sp, const double* lut_s, const IdxT* p, int D,
                                           double (&x)[DM]) {
  if (DM == 8 && D == 8 && (reinterpret_cast<uintptr_t>(p) & (sizeof(IdxT) * 8 - 1)) == 0) {
    uint32_t w[4];
    if (sizeof(IdxT) == 2) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
#pragma unroll
      for (int d = 0; d < 8; ++d) x[d] = lut_s[sp.lut_off[d] + (int)((w[d >> 1] >> (16 * (d & 1))) & 0xFFFFu)];
    } else {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = v.x; w[1] = v.y;
#pragma unroll
      for (int d = 0; d < 8; ++d) x[d] = lut_s[sp.lut_off[d] + (int)((w[d >> 2] >> (8 * (d & 3))) & 0xFFu)];
    }
    return;
  }
#pragma unroll
  for (int d = 0; d < DM; ++d) x[d] = d < D ? feat(sp, lut_s, p, d) : 0.0;
}

// Raw 8-knob row (one 16- or 8-byte load) and its features: the split lets a loop issue the
// next point's loads before it works on the current one (fast path of load_feats).
template <class IdxT>
__device__ __forceinline__ uint4 load_row8(const IdxT* p) {
  if (sizeof(IdxT) == 2) return __ldg(reinterpret_cast<const uint4*>(p));
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  return make_uint4(v.x, v.y, 0u, 0u);
}
template <class IdxT, int DM>
__device__ __forceinline__ void feats_row8(const KtSpaceParams& sp, const double* lut_s, uint4 v, double (&x)[DM]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int d = 0; d < 8; ++d)
    x[d] = sizeof(IdxT) == 2 ? lut_s[sp.lut_off[d] + (int)((w[d >> 1] >> (16 * (d & 1))) & 0xFFFFu)]
                             : lut_s[sp.lut_off[d] + (int)((w[d >> 2] >> (8 * (d & 3))) & 0xFFu)];
#pragma unroll
  for (int d = 8; d < DM; ++d) x[d] = 0.0;
}

// Sequential squared distance.
template <class IdxT>
__device__ __forceinline__ double row_d2(const KtSpaceParams& sp, const double* lut, const IdxT* p,
                                         const double* c, int D) {
  double t = kt::dsub(feat(sp, lut, p, 0), c[0]);
  double s = kt::dmul(t, t);
  for (int d = 1; d < D; ++d) {
    t = kt::dsub(feat(sp, lut, p, d), c[d]);
    s = kt::dadd(s, kt::dmul(t, t));
  }
  return s;
}

// Block reduction (sum) of a double in deterministic tree order.
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = kt::dadd(v, __shfl_down_sync(0xffffffff, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (w == 0) {
    v = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = kt::dadd(v, __shfl_down_sync(0xffffffff, v, o));
  }
  __syncthreads();
  return v;  // valid in thread 0
}

// One warp: in-place exclusive prefix of a[0..n) (stride `stride`), 32 at a time.
// Only feeds approximations / certified bounds, so the tree order is fine.
__device__ double warp_exclusive_scan(double* a, int64_t n, int64_t stride) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  for (int64_t i0 = 0; i0 < n; i0 += 32) {
    const int64_t i = i0 + lane;
    const double v = i < n ? a[i * stride] : 0.0;
    double x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffff, x, o);
      if (lane >= o) x = kt::dadd(x, y);
    }
    if (i < n) a[i * stride] = kt::dadd(carry, kt::dsub(x, v));
    carry = kt::dadd(carry, __shfl_sync(0xffffffff, x, 31));
  }
  return carry;
}

// Block-wide exclusive scans (blockDim.x = 1024) of a strided column, 1024 entries per round: the
// exact-order centroid path scans ~N/1024 block counts and ~N/256 segment prefixes per (cluster,
// knob), which one warp per column walked with a long latency chain at tens of millions of points.
template <class T, class Add>
__device__ T block_exclusive_scan(T* a, int64_t n, int64_t stride, Add add) {
  __shared__ T wsum[32];
  __shared__ T carry_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_sh = T(0);
  __syncthreads();
  for (int64_t i0 = 0; i0 < n; i0 += 1024) {
    const int64_t i = i0 + threadIdx.x;
    const T v = i < n ? a[i * stride] : T(0);
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffff, x, o);
      if (lane >= o) x = add(x, y);
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      T s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffff, s, o);
        if (lane >= o) s = add(s, y);
      }
      wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const T before = add(carry_sh, w > 0 ? wsum[w - 1] : T(0));
    if (i < n) a[i * stride] = add(before, x - v);
    __syncthreads();
    if (threadIdx.x == 0) carry_sh = add(carry_sh, wsum[31]);
    __syncthreads();
  }
  return carry_sh;
}

// Load the feature LUT into shared memory.
__device__ const double* stage_lut(const KtSpaceParams& sp, double* s_lut, int lut_total) {
  for (int i = threadIdx.x; i < lut_total; i += blockDim.x) s_lut[i] = sp.lut[i];
  return s_lut;
}

// ------------------------------------------------------------------ kmeans++ (K5)
struct KppState {
  uint64_t rng;
  int64_t pick;
  int32_t fallbacks;   // picks decided by the exact parallel replay (kpp_x_* kernels)
  int32_t need_exact;  // set by kpp_select when the certified decision is undecided
  uint64_t rng_fb;     // generator state the exact replay starts from
  int32_t c;           // index of the centroid the next kpp_d2 adds (advanced by kpp_select)
  int32_t pad;
};

// d2[i] = (first ? v : min(d2[i], v)), v = |p_i - centroid c|^2, plus chunk sums.
template <class IdxT>
__global__ void __launch_bounds__(kBT) kpp_d2_kernel(KtSpaceParams sp, int lut_total,
                                                     const IdxT* __restrict__ pts, int64_t N,
                                                     const KppState* __restrict__ st,
                                                     double* __restrict__ cent, double* __restrict__ d2,
                                                     double* __restrict__ chunk_sum) {
  extern __shared__ double sdyn[];
  __shared__ double red[32];
  __shared__ double cs[kt::kMaxKnobs];
  const double* lut = stage_lut(sp, sdyn, lut_total);
  __syncthreads();  // the staged table is read below by other threads than those that wrote it
  const int D = sp.D;
  const int64_t pick = st->pick;
  const int c = st->c, first = c == 0;  // the round's centroid index lives on the device (graph replay)
  if (threadIdx.x < D) {
    const double v = lut[sp.lut_off[threadIdx.x] + (int)pts[pick * D + threadIdx.x]];
    cs[threadIdx.x] = v;
    if (blockIdx.x == 0) cent[c * D + threadIdx.x] = v;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  double part = 0.0;
  for (int j = 0; j < kChunk / kBT; ++j) {
    const int64_t i = base + j * kBT + threadIdx.x;
    if (i < N) {
      const double v = row_d2(sp, lut, pts + i * D, cs, D);
      double o = v;
      if (!first) {
        const double old = d2[i];
        o = v < old ? v : old;  // std::min(d2, v) (sampling.cpp:92)
      }
      d2[i] = o;
      part = kt::dadd(part, o);
    }
  }
  const double s = block_sum(part, red);
  if (threadIdx.x == 0) chunk_sum[blockIdx.x] = s;
}

__device__ __forceinline__ double gamma_bound(double terms) { return terms * kU * 1.0625; }


// One CTA of 1024 threads: decide the next kmeans++ pick.
// mode 0: first pick (below(N)); mode 1: D^2 sampling; force_exact: always chain.
__global__ void __launch_bounds__(1024) kpp_select_kernel(const double* __restrict__ d2,
                                                          const double* __restrict__ chunk_sum,
                                                          int64_t N, KppState* st, int mode,
                                                          int force_exact,
                                                          double* __restrict__ scratch) {
  __shared__ double red[32];
  __shared__ double sh_u, sh_tot;
  __shared__ int sh_branch;  // 0 below, 1 sample
  __shared__ unsigned long long sh_ib, sh_ia;
  __shared__ int sh_bfirst, sh_bsecond;
  const int tid = threadIdx.x;
  uint64_t rng = st->rng;
  if (mode == 1 && tid == 0) st->c += 1;  // kpp_d2 of this round has read it; the next round adds c + 1
  if (mode == 0) {
    if (tid == 0) {
      st->pick = (int64_t)kt::rng_below(rng, (uint64_t)N);
      st->rng = rng;
    }
    return;
  }
  const int64_t nch = (N + kChunk - 1) / kChunk;
  // total estimate + positivity (d2 >= 0, so total_ref > 0 iff some d2 > 0)
  double part = 0.0;
  for (int64_t b = tid; b < nch; b += blockDim.x) part = kt::dadd(part, chunk_sum[b]);
  const double tot = block_sum(part, red);
  if (tid == 0) {
    sh_tot = tot;
    // Any positive d2 <=> every chunk sum of non-negatives is 0 otherwise.
    sh_branch = tot > 0.0 ? 1 : 0;
    if (!force_exact) {
      if (sh_branch == 0) {
        st->pick = (int64_t)kt::rng_below(rng, (uint64_t)N);
        st->rng = rng;
      } else {
        sh_u = kt::rng_uniform01(rng);
        st->rng = rng;
      }
    }
  }
  __syncthreads();
  if (force_exact) {  // the exact replay decides (kpp_x_* kernels, launched next)
    if (tid == 0) {
      st->need_exact = 1;
      st->rng_fb = rng;
    }
    return;
  }
  if (sh_branch == 0) return;
  const double u = sh_u, T = sh_tot;
  // slack for the tree/warp-scan order of the estimates (per-chunk tree + carry over nch/32 warps)
  const double lgN = (double)(64 - __clzll((unsigned long long)N)) + 24.0 + (double)(nch / 32);
  const double eT = gamma_bound((double)(N / 4) + lgN) * T;
  const double r_est = kt::dmul(u, T);
  const double r_err = kt::dadd(kt::dmul(u, eT), gamma_bound(4.0) * r_est);
  const double r_lo = kt::dsub(r_est, r_err), r_hi = kt::dadd(r_est, r_err);
  // chunk exclusive prefix (sequential per 1024-chunk slice, tree-free and
  // simple: thread 0 scans up to nch chunk sums into scratch)
  if (tid < 32) {
    for (int64_t b = tid; b < nch; b += 32) scratch[b] = chunk_sum[b];
    __syncwarp();
    warp_exclusive_scan(scratch, nch, 1);
  }
  if (tid == 0) {
    sh_bfirst = -1;
    sh_bsecond = -1;
    sh_ib = ~0ull;
    sh_ia = ~0ull;
  }
  __syncthreads();
  // locate chunks: b_first = first chunk whose max (C_i + e_i) may exceed r_lo,
  // b_second = first chunk whose end certainly exceeds r_hi.
  for (int64_t b0 = 0; b0 < nch; b0 += blockDim.x) {
    const int64_t b = b0 + tid;
    if (b < nch) {
      const double hi_val = kt::dadd(scratch[b], chunk_sum[b]);
      const double e = gamma_bound((double)std::min<int64_t>(N, (b + 1) * kChunk) + lgN + 16.0) * hi_val;
      if (kt::dadd(hi_val, e) > r_lo) atomicMin(&sh_ib, (unsigned long long)b);
      if (kt::dsub(hi_val, e) > r_hi) atomicMin(&sh_ia, (unsigned long long)b);
    }
    __syncthreads();
  }
  if (tid == 0) {
    sh_bfirst = sh_ib == ~0ull ? -1 : (int)sh_ib;
    sh_bsecond = sh_ia == ~0ull ? -1 : (int)sh_ia;
    sh_ib = ~0ull;
    sh_ia = ~0ull;
  }
  __syncthreads();
  const int bfirst = sh_bfirst, bsecond = sh_bsecond;
  bool certified = false;
  int64_t pick = N - 1;
  if (bfirst < 0) {
    certified = true;  // cum never exceeds r: default N-1 (sampling.cpp:81)
  } else if (bsecond < 0 || bsecond - bfirst <= 1) {
    const int blast = bsecond < 0 ? bfirst : bsecond;
    for (int b = bfirst; b <= blast; ++b) {
      const int64_t i = (int64_t)b * kChunk + tid;
      double v = i < N ? d2[i] : 0.0;
      // inclusive block scan (Hillis-Steele through shared memory)
      __shared__ double sc[1024];
      sc[tid] = v;
      __syncthreads();
      for (int o = 1; o < 1024; o <<= 1) {
        const double add = tid >= o ? sc[tid - o] : 0.0;
        __syncthreads();
        sc[tid] = kt::dadd(sc[tid], add);
        __syncthreads();
      }
      if (i < N) {
        const double C = kt::dadd(scratch[b], sc[tid]);
        const double e = gamma_bound((double)(i + 1) + lgN + 16.0) * C;
        if (kt::dadd(C, e) > r_lo) atomicMin(&sh_ib, (unsigned long long)i);
        if (kt::dsub(C, e) > r_hi) atomicMin(&sh_ia, (unsigned long long)i);
      }
      __syncthreads();
    }
    if (sh_ia != ~0ull && sh_ib == sh_ia) {
      certified = true;
      pick = (int64_t)sh_ia;
    }
  }
  if (certified) {
    if (tid == 0) st->pick = pick;
    return;
  }
  // undecided: the exact parallel replay of the reference order decides (kpp_x_*
  // kernels, launched next), from the rng state rewound to before the uniform01 draw
  if (tid == 0) {
    st->need_exact = 1;
    st->rng_fb = st->rng - 0x9E3779B97F4A7C15ULL;  // the branch is identical, the draw is repeated
  }
}

// ------------------------------------------------------------------ assign (K3)
// Exact argmin over centroids (strict <, lowest index wins ties,
// sampling.cpp:39-54); writes d2 of the chosen centroid, the number of
// changed assignments and per-chunk loss partial sums.
template <class IdxT, int DM>
__global__ void __launch_bounds__(kBT) assign_kernel(KtSpaceParams sp, int lut_total,
                                                     const IdxT* __restrict__ pts, int64_t N,
                                                     const double* __restrict__ cent, int k,
                                                     const int32_t* __restrict__ prev,
                                                     int32_t* __restrict__ asg,
                                                     double* __restrict__ d2,
                                                     double* __restrict__ chunk_sum,
                                                     unsigned long long* __restrict__ changed,
                                                     int64_t chunk0) {
  extern __shared__ double sdyn[];
  __shared__ double red[32];
  const int D = sp.D;
  double* s_cent = sdyn;
  double* s_lut = sdyn + k * D;
  for (int i = threadIdx.x; i < k * D; i += blockDim.x) s_cent[i] = cent[i];
  const double* lut = stage_lut(sp, s_lut, lut_total);
  __syncthreads();
  const int64_t cidx = chunk0 + blockIdx.x;  // this rank's shard starts at chunk chunk0
  const int64_t base = cidx * kChunk;
  double part = 0.0;
  int nchg = 0;
  for (int j = 0; j < kChunk / kBT; ++j) {
    const int64_t i = base + j * kBT + threadIdx.x;
    if (i < N) {
      double x[DM];  // DM >= D, compile-time: the features stay in registers
      load_feats<IdxT, DM>(sp, lut, pts + i * D, D, x);
      double best = INFINITY;
      int bc = 0;
      for (int c = 0; c < k; ++c) {
        const double* cc = s_cent + c * D;
        double t = kt::dsub(x[0], cc[0]);
        double s = kt::dmul(t, t);
#pragma unroll
        for (int d = 1; d < DM; ++d) {
          if (d < D) {
            t = kt::dsub(x[d], cc[d]);
            s = kt::dadd(s, kt::dmul(t, t));
          }
        }
        if (s < best) {
          best = s;
          bc = c;
        }
      }
      asg[i] = bc;
      d2[i] = best;
      part = kt::dadd(part, best);
      if (prev && prev[i] != bc) ++nchg;
    }
  }
  const double s = block_sum(part, red);
  if (threadIdx.x == 0) chunk_sum[cidx] = s;
  if (prev) {
    for (int o = 16; o > 0; o >>= 1) nchg += __shfl_down_sync(0xffffffff, nchg, o);
    if ((threadIdx.x & 31) == 0 && nchg) atomicAdd(changed, (unsigned long long)nchg);
  }
}

// ------------------------------------------------------------------ certified Lloyd (mode B)
// Speculative iterations on centroids computed from EXACT INTEGER sums of knob
// indices: c_B = RN(S / (count * (card - 1))) is within 2^-53 relative of the
// exact mean, and the reference's sequential fp64 centroid (sampling.cpp:112-121)
// is within (count + 4) 2^-53 relative of it, so |c_B - c_ref| <= delta. Every
// assignment is certified against that bound (the winner's d2 interval must not
// overlap any other cluster's); an uncertain point or an empty cluster aborts the
// speculation and the run restarts in the exact-order mode A, so the assignment
// sequence is the reference's either way. The run's final centroids and d2 are
// recomputed exactly (mode A) after convergence.

// Segmented warp sums: lanes with the same cluster reduce their knob indices
// and count; the group leader adds them into the block's shared sums.
template <class IdxT>
__device__ __forceinline__ void warp_cluster_sums(bool live, int c, const IdxT* row, int D, int32_t* s_sum,
                                                  int32_t* s_cnt) {
  const int lane = threadIdx.x & 31;
  unsigned todo = __ballot_sync(0xffffffffu, live);
  while (todo) {
    const int leader = __ffs(todo) - 1;
    const int cl = __shfl_sync(0xffffffffu, c, leader);
    const unsigned m = __ballot_sync(0xffffffffu, live && c == cl) & todo;
    if ((m >> lane) & 1u) {
      for (int d = 0; d < D; ++d) {
        const unsigned v = __reduce_add_sync(m, (unsigned)row[d]);
        if (lane == leader) atomicAdd(&s_sum[cl * D + d], (int32_t)v);
      }
      if (lane == leader) atomicAdd(&s_cnt[cl], __popc(m));
    }
    todo &= ~m;
  }
}

// Adds the block's (possibly negative) integer sums into the global ones (two's complement).
__device__ __forceinline__ void flush_cluster_sums(int k, int D, const int32_t* s_sum, const int32_t* s_cnt,
                                                   unsigned long long* g_sum, unsigned long long* g_cnt) {
  for (int i = threadIdx.x; i < k * D; i += blockDim.x)
    if (s_sum[i]) atomicAdd(&g_sum[i], (unsigned long long)(long long)s_sum[i]);
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&g_cnt[i], (unsigned long long)(long long)s_cnt[i]);
}

// Integer sums of an (exact) assignment.
template <class IdxT>
__global__ void __launch_bounds__(kBT) cluster_sums_kernel(const IdxT* __restrict__ pts, int64_t N, int D, int k,
                                                           const int32_t* __restrict__ asg,
                                                           unsigned long long* __restrict__ g_sum,
                                                           unsigned long long* __restrict__ g_cnt) {
  __shared__ int32_t s_sum[kt::kMaxK * kt::kMaxKnobs];
  __shared__ int32_t s_cnt[kt::kMaxK];
  for (int i = threadIdx.x; i < k * D; i += blockDim.x) s_sum[i] = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  // grid-stride over the chunks: a few blocks per SM, so that the k (D + 1) global atomics of the
  // flush are paid per block, not per 1024 points (27k blocks contended on the same words at 27.7M)
  const int64_t nch = (N + kChunk - 1) / kChunk;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int64_t base = ch * kChunk;
    for (int j = 0; j < kChunk / kBT; ++j) {
      const int64_t i = base + j * kBT + threadIdx.x;
      const bool live = i < N;
      warp_cluster_sums(live, live ? asg[i] : 0, pts + (live ? i : 0) * D, D, s_sum, s_cnt);
    }
  }
  __syncthreads();
  flush_cluster_sums(k, D, s_sum, s_cnt, g_sum, g_cnt);
}

// c_B and its bound delta from the integer sums; counts empty clusters.
__global__ void centroids_from_sums_kernel(KtSpaceParams sp, int k, const unsigned long long* __restrict__ g_sum,
                                           const unsigned long long* __restrict__ g_cnt, double* __restrict__ cB,
                                           double* __restrict__ dB, unsigned long long* __restrict__ empty,
                                           double bound_scale = 1.0) {
  const int D = sp.D;
  for (int i = threadIdx.x; i < k * D; i += blockDim.x) {
    const int c = i / D, d = i % D;
    const unsigned long long cnt = g_cnt[c];
    double v = 0.0, del = 0.0;
    if (cnt > 0 && sp.card[d] > 1) {
      v = kt::ddiv((double)g_sum[i], kt::dmul((double)cnt, (double)(sp.card[d] - 1)));
      del = ((double)cnt + 4.0) * 0x1.0p-53 * v * (1.0 + 0x1.0p-20);
    }
    cB[i] = v;
    dB[i] = del;
  }
  __syncthreads();
  // per-cluster bound of |d2(x, c_B) - d2(x, c_ref)| without the rounding term: features and
  // centroids lie in [0, 1], so |x_d - c_d| <= 1 and sum_d delta_d (2|x_d - c_d| + delta_d)
  // <= sum_d delta_d (2 + delta_d)
  if (threadIdx.x < k) {
    double e = 0.0;
    for (int d = 0; d < D; ++d) {
      const double del = dB[threadIdx.x * D + d];
      e += del * (2.0 + del);
    }
    dB[kt::kMaxK * kt::kMaxKnobs + threadIdx.x] = e * (1.0 + 0x1.0p-20) * bound_scale;  // scale: tests only
    if (g_cnt[threadIdx.x] == 0) atomicAdd(empty, 1ull);
  }
}

// Sharded certified Lloyd: every rank adds the all-reduced deltas of the points that
// moved (integer sums: exact and order-free) to its replica of the sums.
__global__ void add_sums_kernel(unsigned long long* __restrict__ cs, const unsigned long long* __restrict__ delta,
                                int n) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) cs[i] += delta[i];
}

// Certified assignment against c_B: d2 in the reference's operation order with
// c_B, a rigorous interval per cluster, the winner only if its interval is
// strictly below every other cluster's. Fused: the integer sums are updated in
// place by the points that changed cluster (block-aggregated deltas), plus the
// changed / uncertain counts and the loss estimate.
// 128-thread blocks (8 points per thread per 1024-point chunk): twice the resident blocks
// of the 256-thread layout, so 1M points (1024 chunks) run in one wave instead of 1.7
constexpr int kCertBT = 128;
// dynamic shared memory of assign_cert_kernel<IdxT, DM> for k clusters (layout in the kernel)
inline size_t cert_smem_bytes(int k, int D, int DM, size_t lut_bytes) {
  const size_t dbl = (size_t)((k * D + kt::kMaxK + 1) & ~1) * 8;
  const size_t ints = (size_t)k * DM * 4 + (size_t)k * D * 4 + (size_t)(((k + 1) & ~1) + ((k * D) & 1)) * 4;
  return dbl + ints + lut_bytes + 16;
}
template <class IdxT, int DM>
__global__ void __launch_bounds__(kCertBT) assign_cert_kernel(
    KtSpaceParams sp, int lut_total, const IdxT* __restrict__ pts, int64_t N, const double* __restrict__ cB,
    const double* __restrict__ dB, int k, const int32_t* __restrict__ prev, int32_t* __restrict__ asg,
    double* __restrict__ d2, double* __restrict__ chunk_sum, unsigned long long* __restrict__ counters,
    unsigned long long* __restrict__ g_sum, unsigned long long* __restrict__ g_cnt, int64_t chunk0) {
  extern __shared__ __align__(16) double sdyn[];
  __shared__ double red[32];
  __shared__ float s_amax;
  const int D = sp.D;
  // dynamic layout sized by k (cert_smem_bytes): c_B (fp64), E_c, c_B rows in fp32 zero-padded to
  // DM (16-byte aligned for float4), the block's integer-sum deltas and counts, the feature table
  double* s_c = sdyn;  // knob-major [d][c]: lanes reading different clusters' coordinate d hit distinct banks
  double* s_e = sdyn + k * D;  // per-cluster centroid-difference bound E_c
  float* s_c32 = reinterpret_cast<float*>(sdyn + ((k * D + kt::kMaxK + 1) & ~1));  // [k][DM]
  int32_t* s_sum = reinterpret_cast<int32_t*>(s_c32 + k * DM);
  int32_t* s_cnt = s_sum + k * D;
  double* s_lut = reinterpret_cast<double*>(s_cnt + ((k + 1) & ~1) + ((k * D) & 1));
  // fp32 screening bound |s32 - d2_ref| <= A + R s32 for every cluster (features and
  // centroids in [0, 1]): conversions and the difference cost <= 1.5 ulp(1) per knob,
  // squaring <= 2x that, the FMA chain D 2^-24 relative; A also carries max_c E_c and
  // both are doubled for the fp32 arithmetic of the test itself.
  const float R32 = (float)(2 * D + 8) * 0x1.0p-24f;
  const double A32 = (double)(12 * D + 4) * 0x1.0p-24;
  for (int i = threadIdx.x; i < k * D; i += blockDim.x) {
    s_c[(i % D) * k + i / D] = cB[i];
    s_sum[i] = 0;
  }
  for (int i = threadIdx.x; i < k * DM; i += blockDim.x) {
    const int c = i / DM, d = i % DM;
    s_c32[i] = d < D ? (float)cB[c * D + d] : 0.f;
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) s_e[i] = dB[kt::kMaxK * kt::kMaxKnobs + i];
  if (threadIdx.x == 0) {
    double emax = 0.0;
    for (int c = 0; c < k; ++c) emax = fmax(emax, dB[kt::kMaxK * kt::kMaxKnobs + c]);
    s_amax = __double2float_ru(A32 + 2.0 * emax);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) s_cnt[i] = 0;
  const double* lut = stage_lut(sp, s_lut, lut_total);
  __syncthreads();
  const int64_t base = (chunk0 + blockIdx.x) * kChunk;  // this launch's chunk range (a rank's shard)
  double part = 0.0;
  int nchg = 0, nunc = 0;
  const double grow = (double)(2 * D + 4) * 0x1.0p-53;
  // 8-knob rows: the next point's row and previous assignment are loaded one iteration ahead
  // (their global-load latency was the kernel's top stall at small k)
  const bool row8 = DM == 8 && D == 8;
  uint4 raw_n = make_uint4(0u, 0u, 0u, 0u);
  int prev_n = 0;
  if (row8 && base + threadIdx.x < N) {
    raw_n = load_row8<IdxT>(pts + (base + threadIdx.x) * 8);
    if (prev) prev_n = __ldg(prev + base + threadIdx.x);
  }
  for (int j = 0; j < kChunk / kCertBT; ++j) {
    const int64_t i = base + j * kCertBT + threadIdx.x;
    const bool live = i < N;
    int bc = 0;
    const uint4 raw = raw_n;
    const int prev_i = prev_n;
    if (row8 && j + 1 < kChunk / kCertBT && i + kCertBT < N) {
      raw_n = load_row8<IdxT>(pts + (i + kCertBT) * 8);
      if (prev) prev_n = __ldg(prev + i + kCertBT);
    }
    if (live) {
      // (1) fp32 screening: the winner is certified if the runner-up's interval lies
      // strictly above the winner's: s2 (1 - R) - A > s1 (1 + R) + A
      double x[DM];  // DM >= D, compile-time: the features stay in registers
      if (row8) feats_row8<IdxT, DM>(sp, lut, raw, x);
      else load_feats<IdxT, DM>(sp, lut, pts + i * D, D, x);
      float xf[DM];
#pragma unroll
      for (int d = 0; d < DM; ++d) xf[d] = (float)x[d];  // padded knobs add 0 exactly
      float s1 = INFINITY, s2 = INFINITY;
      int w32 = 0;
      for (int c = 0; c < k; ++c) {
        const float4* cc = reinterpret_cast<const float4*>(s_c32 + c * DM);
        float s32 = 0.f;
#pragma unroll
        for (int q = 0; q < DM / 4; ++q) {
          const float4 v = cc[q];
          float t = xf[4 * q] - v.x;
          s32 = fmaf(t, t, s32);
          t = xf[4 * q + 1] - v.y;
          s32 = fmaf(t, t, s32);
          t = xf[4 * q + 2] - v.z;
          s32 = fmaf(t, t, s32);
          t = xf[4 * q + 3] - v.w;
          s32 = fmaf(t, t, s32);
        }
        if (s32 < s1) {
          s2 = s1;
          s1 = s32;
          w32 = c;
        } else {
          s2 = fminf(s2, s32);
        }
      }
      const float amax = s_amax;
      double best = INFINITY;
      if (fmaf(-R32, s2, s2) - amax > fmaf(R32, s1, s1) + amax) {  // (2a) the winner's d2 against c_B in the reference order
        const double* cc = s_c + w32;  // coordinate d at cc[d * k]
        double t = kt::dsub(x[0], cc[0]);
        best = kt::dmul(t, t);
#pragma unroll
        for (int d = 1; d < DM; ++d) {
          if (d < D) {
            t = kt::dsub(x[d], cc[d * k]);
            best = kt::dadd(best, kt::dmul(t, t));
          }
        }
        bc = w32;
      } else {  // (2b) near tie: the full fp64 scan with its own certificate
        double best_e = 0.0, lo_others = INFINITY;
        for (int c = 0; c < k; ++c) {
          const double* cc = s_c + c;
          double t = kt::dsub(x[0], cc[0]);
          double s = kt::dmul(t, t);
#pragma unroll
          for (int d = 1; d < DM; ++d) {
            if (d < D) {
              t = kt::dsub(x[d], cc[d * k]);
              s = kt::dadd(s, kt::dmul(t, t));
            }
          }
          // |d2_ref - s| <= E_c (centroid difference) + the rounding of both evaluations
          const double e = (s_e[c] + grow * (s + s_e[c])) * (1.0 + 0x1.0p-20) + 1e-300;
          if (s < best) {  // strict <: lowest index on ties, as the reference
            if (best < INFINITY) lo_others = fmin(lo_others, best - best_e);
            best = s;
            best_e = e;
            bc = c;
          } else {
            lo_others = fmin(lo_others, s - e);
          }
        }
        // certified only if no other cluster's interval reaches the winner's
        if (!(lo_others > best + best_e)) ++nunc;
      }
      asg[i] = bc;
      d2[i] = best;
      part = kt::dadd(part, best);
      const int pc = prev ? (row8 ? prev_i : prev[i]) : bc;
      if (pc != bc) {  // move this point's indices between the clusters' integer sums
        ++nchg;
        if (g_sum) {
          for (int d = 0; d < D; ++d) {
            const int v = (int)pts[i * D + d];
            if (v) {
              atomicAdd(&s_sum[bc * D + d], v);
              atomicAdd(&s_sum[pc * D + d], -v);
            }
          }
          atomicAdd(&s_cnt[bc], 1);
          atomicAdd(&s_cnt[pc], -1);
        }
      }
    }
  }
  const double s = block_sum(part, red);
  if (threadIdx.x == 0) chunk_sum[chunk0 + blockIdx.x] = s;
  for (int o = 16; o > 0; o >>= 1) {
    nchg += __shfl_down_sync(0xffffffff, nchg, o);
    nunc += __shfl_down_sync(0xffffffff, nunc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nchg) atomicAdd(counters, (unsigned long long)nchg);
    if (nunc) atomicAdd(counters + 2, (unsigned long long)nunc);
  }
  __syncthreads();
  if (g_sum) flush_cluster_sums(k, D, s_sum, s_cnt, g_sum, g_cnt);
}

// ------------------------------------------------------------------ assign on tcgen05 (K3 fast path)
// Screening GEMM on the 5th-gen tensor cores: for a tile of 128 points,
//   dot[p][c] = sum_d idx[p][d] * (2^10 * c[c][d] / (card_d - 1))
// with A = [idx | idx] (fp16, exact for idx < 2048) and B = [hi | lo] (the
// fp16 split of the scaled centroid coordinate), K = 32, fp32 accumulation in
// TMEM, so dot = sum_d x_d c_d to ~2^-21. score_c = |c|^2 - 2 dot ranks the
// clusters like the exact d2 (|x|^2 is common). A rigorous per-cluster bound
// E_c certifies the winner; the winner's d2 is then recomputed EXACTLY in the
// reference order (sequential over knobs, fp64, no FMA), and any uncertain
// point falls back to the full exact scan — assignments and d2 stay bit-exact.
constexpr int kTcPts = 128;
constexpr int kTcK = 32;   // 2 x 16 knobs
constexpr int kTcMaxN = 64;
// Below this k the exact SIMT scan (3kD fp64 ops per point) beats the tcgen05 screening
// pass, whose per-tile MMA round trip dominates (measured at N = 1M: 45 vs 161 us for k = 8).
constexpr int kTcMinK = 24;

template <class IdxT>
__global__ void __launch_bounds__(kTcPts) assign_tc_kernel(
    KtSpaceParams sp, int lut_total, const IdxT* __restrict__ pts, int64_t N, const double* __restrict__ cent,
    int k, const int32_t* __restrict__ prev, int32_t* __restrict__ asg, double* __restrict__ d2,
    double* __restrict__ tile_sum, unsigned long long* __restrict__ counters, int64_t tile_begin,
    int64_t tile_end) {
  extern __shared__ __align__(128) unsigned char tsm[];
  unsigned char* sA = tsm;                              // 128 x 32 fp16 = 8 KB
  unsigned char* sB = sA + kTcPts * kTcK * 2;           // 64 x 32 fp16 = 4 KB
  double* s_cent = reinterpret_cast<double*>(sB + kTcMaxN * kTcK * 2);  // k x D
  double* s_cn2 = s_cent + kt::kMaxK * kt::kMaxKnobs;   // k
  double* s_lut = s_cn2 + kt::kMaxK;                    // feature LUT
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  __shared__ double red[32];
  const int D = sp.D, t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int NN = (k + 15) & ~15;  // MMA N (multiple of 16 for M = 128)
  for (int i = t; i < k * D; i += kTcPts) s_cent[i] = cent[i];
  const double* lut = stage_lut(sp, s_lut, lut_total);
  __syncthreads();
  // B = [hi | lo] of v = 2^10 * c / (card - 1)
  for (int i = t; i < NN * 16; i += kTcPts) {
    const int c = i / 16, d = i % 16;
    __half hi = __float2half(0.f), lo = __float2half(0.f);
    if (c < k && d < D && sp.card[d] > 1) {
      const double v = kt::dmul(kt::ddiv(s_cent[c * D + d], (double)(sp.card[d] - 1)), 1024.0);
      hi = __double2half(v);
      lo = __double2half(kt::dsub(v, (double)__half2float(hi)));
    }
    *reinterpret_cast<__half*>(sB + kt::tc::kmajor_offset(c, d, kTcK)) = hi;
    *reinterpret_cast<__half*>(sB + kt::tc::kmajor_offset(c, 16 + d, kTcK)) = lo;
  }
  if (t < k) {  // |c|^2, sequential
    double s = 0.0;
    for (int d = 0; d < D; ++d) s = kt::dadd(s, kt::dmul(s_cent[t * D + d], s_cent[t * D + d]));
    s_cn2[t] = s;
  }
  if (w == 0) kt::tc::tmem_alloc(&tbase, 64);
  if (t == 0) {
    kt::tc::mbar_init(&mbar, 1);
    kt::tc::fence_mbar_init();
  }
  kt::tc::fence_before();
  __syncthreads();
  kt::tc::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = kt::tc::idesc_f16_f32(kTcPts, NN);
  const double eps_rel = (double)(2 * D + 4) * 0x1.0p-23;
  uint32_t phase = 0;
  double part = 0.0;
  unsigned nchg = 0, nunc = 0;
  for (int64_t tile = tile_begin + blockIdx.x; tile < tile_end; tile += gridDim.x) {
    const int64_t p = tile * kTcPts + t;
    const bool live = p < N;
    int ix[16];
    int sidx = 0;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      ix[d] = (live && d < D) ? (int)pts[p * D + d] : 0;
      sidx += ix[d];
      const __half h = __int2half_rn(ix[d]);
      *reinterpret_cast<__half*>(sA + kt::tc::kmajor_offset(t, d, kTcK)) = h;
      *reinterpret_cast<__half*>(sA + kt::tc::kmajor_offset(t, 16 + d, kTcK)) = h;
    }
    kt::tc::fence_proxy_async();
    kt::tc::fence_before();
    __syncthreads();
    kt::tc::fence_after();
    if (t == 0) {
#pragma unroll
      for (int kb = 0; kb < kTcK / 16; ++kb) {
        const uint64_t ad = kt::tc::smem_desc(kt::tc::smem_u32(sA + kb * 256), 128, (kTcK / 8) * 128);
        const uint64_t bd = kt::tc::smem_desc(kt::tc::smem_u32(sB + kb * 256), 128, (kTcK / 8) * 128);
        kt::tc::mma_f16(tmem, ad, bd, idesc, kb > 0);
      }
      kt::tc::commit(&mbar);
    }
    kt::tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    kt::tc::fence_after();
    float dotf[kTcMaxN];
#pragma unroll
    for (int c0 = 0; c0 < kTcMaxN; c0 += 16) {
      if (c0 < NN) {
        uint32_t r[16];
        kt::tc::ld_32x32b_x16(tmem + ((uint32_t)(32 * w) << 16) + (uint32_t)c0, r);
        kt::tc::ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) dotf[c0 + j] = __uint_as_float(r[j]);
      }
    }
    if (live) {
      // screening: best score and the tightest competitor, with per-cluster bounds
      const double abs_term = (double)sidx * 0x1.0p-35 + 1e-15;
      double best = INFINITY, best_e = 0.0, lb_others = INFINITY;
      int bc = 0;
#pragma unroll
      for (int c = 0; c < kTcMaxN; ++c) {
        if (c < k) {
          const double dot = (double)dotf[c] * 0x1.0p-10;
          const double sc = s_cn2[c] - 2.0 * dot;
          const double e = 2.0 * (eps_rel * (fabs(dot) * 1.001 + 1e-12) + abs_term) + 1e-12 +
                           1e-15 * (s_cn2[c] + 2.0 * fabs(dot));
          if (sc < best) {
            if (best < INFINITY) lb_others = fmin(lb_others, best - best_e);
            best = sc;
            best_e = e;
            bc = c;
          } else {
            lb_others = fmin(lb_others, sc - e);
          }
        }
      }
      double x[16];
#pragma unroll
      for (int d = 0; d < 16; ++d) x[d] = d < D ? lut[sp.lut_off[d] + ix[d]] : 0.0;
      double bestd;
      if (lb_others > best + best_e) {  // certified: exact d2 of the winner only
        double tt = kt::dsub(x[0], s_cent[bc * D]);
        bestd = kt::dmul(tt, tt);
        for (int d = 1; d < D; ++d) {
          tt = kt::dsub(x[d], s_cent[bc * D + d]);
          bestd = kt::dadd(bestd, kt::dmul(tt, tt));
        }
      } else {  // uncertain: the full exact scan (sampling.cpp:39-54)
        ++nunc;
        bestd = INFINITY;
        bc = 0;
        for (int c = 0; c < k; ++c) {
          double tt = kt::dsub(x[0], s_cent[c * D]);
          double s = kt::dmul(tt, tt);
          for (int d = 1; d < D; ++d) {
            tt = kt::dsub(x[d], s_cent[c * D + d]);
            s = kt::dadd(s, kt::dmul(tt, tt));
          }
          if (s < bestd) {
            bestd = s;
            bc = c;
          }
        }
      }
      asg[p] = bc;
      d2[p] = bestd;
      part = kt::dadd(part, bestd);
      if (prev && prev[p] != bc) ++nchg;
    }
    const double ts = block_sum(live ? part : 0.0, red);
    if (t == 0) tile_sum[tile] = ts;
    part = 0.0;
    kt::tc::fence_before();
    __syncthreads();
    kt::tc::fence_after();
  }
  for (int o = 16; o > 0; o >>= 1) {
    nchg += __shfl_down_sync(0xffffffff, nchg, o);
    nunc += __shfl_down_sync(0xffffffff, nunc, o);
  }
  if (lane == 0) {
    if (nchg) atomicAdd(counters, (unsigned long long)nchg);
    if (nunc) atomicAdd(counters + 2, (unsigned long long)nunc);
  }
  kt::tc::fence_before();
  __syncthreads();
  if (w == 0) kt::tc::tmem_dealloc(tmem, 64);
}

// ------------------------------------------------------------------ centroid update (K4)
// Stable counting sort of point ids by cluster (ascending point order inside
// each cluster), then one thread per (cluster, knob) sums its members' features
// in that order (sampling.cpp:110-121).
__global__ void __launch_bounds__(kBT) hist_kernel(const int32_t* __restrict__ asg, int64_t N, int k,
                                                   int32_t* __restrict__ blockcounts) {
  __shared__ int cnt[kt::kMaxK];
  for (int c = threadIdx.x; c < k; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int j = threadIdx.x; j < kChunk; j += blockDim.x) {
    const int64_t i = base + j;
    if (i < N) atomicAdd(&cnt[asg[i]], 1);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) blockcounts[(int64_t)blockIdx.x * k + c] = cnt[c];
}

// Exclusive scan over blocks per cluster; cluster totals, starts and the
// per-cluster segment bases of the exact-sum machinery (csb[k+1]).
// One 1024-thread block per cluster: exclusive scan of its per-block counts (strided by k).
__global__ void __launch_bounds__(1024) scan_counts_kernel(int32_t* __restrict__ blockcounts, int64_t nblocks,
                                                           int k, int32_t* __restrict__ counts) {
  const int c = blockIdx.x;
  const int t = block_exclusive_scan<int32_t>(blockcounts + c, nblocks, k, [](int32_t a, int32_t b) { return a + b; });
  if (threadIdx.x == 0) counts[c] = t;
}

// Cluster starts and segment starts from the cluster totals.
__global__ void cluster_starts_kernel(const int32_t* __restrict__ counts, int k, int32_t* __restrict__ cstart,
                                      int32_t* __restrict__ csb) {
  if (threadIdx.x != 0) return;
  int sum = 0, sb = 0;
  for (int j = 0; j < k; ++j) {
    cstart[j] = sum;
    csb[j] = sb;
    sum += counts[j];
    sb += (counts[j] + kt::xsum::kSeg - 1) / kt::xsum::kSeg;
  }
  csb[k] = sb;
}

// Stable scatter: warp w of the block owns points [base + w*128, base + (w+1)*128).
// Writes member ids and the members' knob-index rows in cluster-major,
// ascending-point order (the reference's summation order, sampling.cpp:112-116).
template <class IdxT>
__global__ void __launch_bounds__(kBT) scatter_kernel(const int32_t* __restrict__ asg, int64_t N, int k,
                                                      int D, const IdxT* __restrict__ pts,
                                                      const int32_t* __restrict__ blockoffs,
                                                      const int32_t* __restrict__ cstart,
                                                      int32_t* __restrict__ members,
                                                      IdxT* __restrict__ sorted) {
  constexpr int kWarps = kBT / 32;
  constexpr int kPerWarp = kChunk / kWarps;  // 128 points = 4 rounds of 32
  __shared__ int wcnt[kWarps][kt::kMaxK];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = lane; c < k; c += 32) wcnt[w][c] = 0;
  __syncwarp();
  const int64_t wbase = (int64_t)blockIdx.x * kChunk + w * kPerWarp;
  for (int r = 0; r < kPerWarp / 32; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    if (i < N) atomicAdd(&wcnt[w][asg[i]], 1);
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int c = threadIdx.x;
    int run = 0;
    for (int ww = 0; ww < kWarps; ++ww) {
      const int v = wcnt[ww][c];
      wcnt[ww][c] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int r = 0; r < kPerWarp / 32; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool ok = i < N;
    const int c = ok ? asg[i] : -1 - lane;
    const unsigned m = __match_any_sync(0xffffffff, c);
    const int before = __popc(m & ((1u << lane) - 1));
    if (ok) {
      const int64_t pos = cstart[c] + blockoffs[(int64_t)blockIdx.x * k + c] + wcnt[w][c] + before;
      members[pos] = (int32_t)i;
      if (D == 8) {  // the 8-knob row as one vector (8 or 16 bytes) instead of 8 scattered stores
        if constexpr (sizeof(IdxT) == 1)
          *reinterpret_cast<uint2*>(sorted + pos * 8) = __ldg(reinterpret_cast<const uint2*>(pts + i * 8));
        else
          *reinterpret_cast<uint4*>(sorted + pos * 8) = __ldg(reinterpret_cast<const uint4*>(pts + i * 8));
      } else {
        for (int d = 0; d < D; ++d) sorted[pos * D + d] = pts[i * D + d];
      }
    }
    __syncwarp();
    if (ok && before == 0) wcnt[w][c] += __popc(m);
    __syncwarp();
  }
}

// ---- exact centroid sums over the sorted rows (exactsum.cuh) ----------------
// thread (cluster-segment g, knob d); g indexes segments of all clusters (csb).
__device__ __forceinline__ int cluster_of_segment(const int32_t* csb, int k, int g) {
  int c = 0;
  while (c + 1 < k && csb[c + 1] <= g) ++c;
  return c;
}

template <class IdxT>
__global__ void xs_partial_kernel(KtSpaceParams sp, const IdxT* __restrict__ sorted,
                                  const int32_t* __restrict__ counts, const int32_t* __restrict__ cstart,
                                  const int32_t* __restrict__ csb, int k, int max_segs,
                                  double* __restrict__ approx) {
  const int D = sp.D;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = (int)(t / D), d = (int)(t % D);
  if (g >= max_segs || g >= csb[k]) return;
  const int c = cluster_of_segment(csb, k, g);
  const int j = g - csb[c];
  const int n = counts[c];
  const int lo = j * kt::xsum::kSeg, hi = min(n, lo + kt::xsum::kSeg);
  const double* lut = sp.lut + sp.lut_off[d];
  const IdxT* rows = sorted + (int64_t)cstart[c] * D + d;
  double s = 0.0;
  for (int i = lo; i < hi; ++i) s = kt::dadd(s, __ldg(lut + (int)rows[(int64_t)i * D]));
  approx[(int64_t)g * D + d] = s;
}

// warp per (cluster c, knob d): exclusive prefix of the approximate segment sums.
// One 1024-thread block per (cluster, knob): the APPROXIMATE segment prefix (it only predicts the
// binade each segment map is built for; a wrong prediction falls back to the plain chain).
__global__ void __launch_bounds__(1024) xs_prefix_kernel(int D, const int32_t* __restrict__ csb, int k,
                                                         double* __restrict__ approx) {
  const int c = blockIdx.x / D, d = blockIdx.x % D;
  block_exclusive_scan<double>(approx + (int64_t)csb[c] * D + d, csb[c + 1] - csb[c], D,
                               [](double a, double b) { return kt::dadd(a, b); });
}

template <class IdxT>
__global__ void xs_map_kernel(KtSpaceParams sp, const IdxT* __restrict__ sorted,
                              const int32_t* __restrict__ counts, const int32_t* __restrict__ cstart,
                              const int32_t* __restrict__ csb, int k, int max_segs,
                              const double* __restrict__ prefix, kt::xsum::SegMap* __restrict__ maps) {
  const int D = sp.D;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = (int)(t / D), d = (int)(t % D);
  if (g >= max_segs || g >= csb[k]) return;
  const int c = cluster_of_segment(csb, k, g);
  const int j = g - csb[c];
  const int n = counts[c];
  const int lo = j * kt::xsum::kSeg, hi = min(n, lo + kt::xsum::kSeg);
  const double pre = prefix[(int64_t)g * D + d];
  const double* lut = sp.lut + sp.lut_off[d];
  const IdxT* rows = sorted + (int64_t)cstart[c] * D + d;
  auto at = [&](int i) { return __ldg(lut + (int)rows[(int64_t)(lo + i) * D]); };
  const kt::xsum::SegMap m = pre > 0.0 ? kt::xsum::segment_map(at, hi - lo, kt::xsum::binade_of(pre))
                                       : kt::xsum::zero_segment_map(at, hi - lo);
  maps[(int64_t)g * D + d] = m;
}

// Warp-cooperative exact chain over one segment: every lane holds the same
// running sum (uniform control flow); lanes fetch 32 elements at a time and
// the chain consumes them in order through shuffles.
template <class At>
__device__ __forceinline__ double warp_seq_segment(double s, At at, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  constexpr int kAhead = 4;  // batches in flight: the loads overlap the chain
  double v[kAhead];
#pragma unroll
  for (int b = 0; b < kAhead; ++b) {
    const int i = lo + b * 32 + lane;
    v[b] = i < hi ? at(i) : 0.0;
  }
  for (int i0 = lo; i0 < hi; i0 += 32 * kAhead) {
#pragma unroll
    for (int b = 0; b < kAhead; ++b) {
      const int base = i0 + b * 32;
      const double cur = v[b];
      const int nx = base + kAhead * 32 + lane;  // refill this slot for the next round
      v[b] = nx < hi ? at(nx) : 0.0;
      if (base < hi) {
        if (hi - base >= 32) {
#pragma unroll
          for (int q = 0; q < 32; ++q) s = kt::dadd(s, __shfl_sync(0xffffffff, cur, q));
        } else {
          for (int q = 0; q < hi - base; ++q) s = kt::dadd(s, __shfl_sync(0xffffffff, cur, q));
        }
      }
    }
  }
  return s;
}

// Warp-cooperative composition of a chain's segment maps (maps prefetched 32 at a time).
template <class At, class MapAt>
__device__ __forceinline__ double warp_compose(At at, MapAt map_at, int nseg, int n, int* nseq_out) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;  // MatrixXd::Zero / loss = 0.0 then += in order
  int nseq = 0;
  for (int g0 = 0; g0 < nseg; g0 += 32) {
    kt::xsum::SegMap mine{0, 0, 0, 0};
    if (g0 + lane < nseg) mine = map_at(g0 + lane);
    const int mcount = min(32, nseg - g0);
    // Fast path: all maps of this batch valid for one binade -> compose the
    // 32 maps with a warp scan (m -> m + F(m mod 2) is closed under
    // composition) and apply the whole batch in one step.
    const unsigned real = __ballot_sync(0xffffffff, lane < mcount && mine.ok != 2);  // non-identity maps
    if (real == 0) continue;  // whole batch is identity (all-zero segments)
    const int e0 = __shfl_sync(0xffffffff, mine.e, __ffs(real) - 1);
    const bool uniform = __all_sync(0xffffffff, lane >= mcount || mine.ok == 2 || (mine.ok == 1 && mine.e == e0));
    if (uniform && s > 0.0) {
      uint64_t c0 = mine.F0, c1 = mine.F1;  // inclusive composition f_0 .. f_lane
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t p0 = __shfl_up_sync(0xffffffff, c0, off);
        const uint64_t p1 = __shfl_up_sync(0xffffffff, c1, off);
        if (lane >= off) {  // earlier maps (p) then mine (c)
          const uint64_t n0 = p0 + ((p0 & 1u) ? c1 : c0);
          const uint64_t n1 = p1 + (((1u + p1) & 1u) ? c1 : c0);
          c0 = n0;
          c1 = n1;
        }
      }
      kt::xsum::SegMap all;
      all.F0 = __shfl_sync(0xffffffff, c0, mcount - 1);
      all.F1 = __shfl_sync(0xffffffff, c1, mcount - 1);
      all.e = e0;
      all.ok = all.F0 < (1ull << 53) && all.F1 < (1ull << 53);
      if (kt::xsum::apply_map(s, all)) continue;
    }
    for (int q = 0; q < mcount; ++q) {
      kt::xsum::SegMap m;
      m.F0 = __shfl_sync(0xffffffff, mine.F0, q);
      m.F1 = __shfl_sync(0xffffffff, mine.F1, q);
      m.e = __shfl_sync(0xffffffff, mine.e, q);
      m.ok = __shfl_sync(0xffffffff, mine.ok, q);
      if (kt::xsum::apply_map(s, m)) continue;
      const int g = g0 + q;
      const int lo = g * kt::xsum::kSeg, hi = min(n, lo + kt::xsum::kSeg);
      ++nseq;
      s = warp_seq_segment(s, at, lo, hi);
    }
  }
  *nseq_out = nseq;
  return s;
}

// Block-cooperative (1024 threads) version of warp_compose with bit-identical results: per round
// of 1024 segment maps, the 32 warps compose their 32-map batches in parallel (the same scan and
// uniform-binade test as warp_compose), then warp 0 walks the 32 batch results in order, taking
// exactly warp_compose's per-batch decisions (identity batch, composed map, else per-segment maps
// and sequential segments). The serial part drops from one warp scan + map load per 32 segments
// to one apply per 32 segments.
template <class At, class MapAt>
__device__ double block_compose(At at, MapAt map_at, int nseg, int n, int* nseq_out) {
  __shared__ kt::xsum::SegMap smaps[1024];
  __shared__ kt::xsum::SegMap wmap[32];
  __shared__ int wflag[32];  // 0: identity batch, 1: uniform (wmap valid to try), 2: per-segment
  __shared__ double s_sh;
  __shared__ int nseq_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_sh = 0.0;  // MatrixXd::Zero / loss = 0.0 then += in order
    nseq_sh = 0;
  }
  for (int sb0 = 0; sb0 < nseg; sb0 += 1024) {
    {
      const int g0 = sb0 + 32 * w;
      const int mcount = min(32, nseg - g0);
      kt::xsum::SegMap mine{0, 0, 0, 0};
      if (lane < mcount) mine = map_at(g0 + lane);
      smaps[32 * w + lane] = mine;
      const unsigned real = __ballot_sync(0xffffffff, lane < mcount && mine.ok != 2);
      int flag = 0;
      if (real != 0) {
        const int e0 = __shfl_sync(0xffffffff, mine.e, __ffs(real) - 1);
        const bool uniform = __all_sync(0xffffffff, lane >= mcount || mine.ok == 2 || (mine.ok == 1 && mine.e == e0));
        flag = 2;
        if (uniform) {
          uint64_t c0 = mine.F0, c1 = mine.F1;
          for (int off = 1; off < 32; off <<= 1) {
            const uint64_t p0 = __shfl_up_sync(0xffffffff, c0, off);
            const uint64_t p1 = __shfl_up_sync(0xffffffff, c1, off);
            if (lane >= off) {
              const uint64_t n0 = p0 + ((p0 & 1u) ? c1 : c0);
              const uint64_t n1 = p1 + (((1u + p1) & 1u) ? c1 : c0);
              c0 = n0;
              c1 = n1;
            }
          }
          const uint64_t f0 = __shfl_sync(0xffffffff, c0, max(mcount, 1) - 1);
          const uint64_t f1 = __shfl_sync(0xffffffff, c1, max(mcount, 1) - 1);
          if (lane == 0) wmap[w] = kt::xsum::SegMap{f0, f1, e0, (f0 < (1ull << 53) && f1 < (1ull << 53)) ? 1 : 0};
          flag = 1;
        }
      }
      if (lane == 0) wflag[w] = mcount > 0 ? flag : 0;
    }
    __syncthreads();
    if (w == 0) {
      double s = s_sh;
      int nseq = 0;
      __syncwarp();  // every lane holds the round's start value before lane 0 may overwrite it
      for (int b = 0; b < 32; ++b) {
        const int g0 = sb0 + 32 * b;
        if (g0 >= nseg) break;
        const int fl = wflag[b];
        if (fl == 0) continue;  // whole batch is identity (all-zero segments)
        if (fl == 1 && s > 0.0 && kt::xsum::apply_map(s, wmap[b])) continue;
        const int mcount = min(32, nseg - g0);
        for (int q = 0; q < mcount; ++q) {
          if (kt::xsum::apply_map(s, smaps[32 * b + q])) continue;
          const int lo = (g0 + q) * kt::xsum::kSeg, hi = min(n, lo + kt::xsum::kSeg);
          ++nseq;
          s = warp_seq_segment(s, at, lo, hi);
        }
      }
      if (lane == 0) {
        s_sh = s;
        nseq_sh += nseq;
      }
    }
    __syncthreads();
  }
  *nseq_out = nseq_sh;
  return s_sh;
}

// ---- kmeans++ exact replay (sampling.cpp:65-96), in parallel. Taken when the
// certified pick is undecided (more likely at tens of millions of points, where the
// rigorous bound of the parallel prefix grows like N u) or when forced. The reference
// draws r = uniform01 * total with total = d2.sum() in Eigen's 4-lane order
// (eigen_shim: lane v sums d2[v + 4j] sequentially, then (l0 + l2) + (l1 + l3), tail),
// and picks the first i whose SEQUENTIAL cum exceeds r. Views 0..3 are the four
// strided lanes, view 4 the natural order; each is summed exactly with the segment
// maps of exactsum.cuh (approximate prefix -> binade -> maps -> warp composition).
constexpr int kKppViews = 5;
struct KppView {
  const double* x;
  int64_t off, stride, n;
  __device__ double operator()(int64_t i) const { return x[off + stride * i]; }
};
__device__ __forceinline__ KppView kpp_view(const double* d2, int64_t N, int v) {
  return v < 4 ? KppView{d2, v, 4, N >= 4 ? N / 4 : 0} : KppView{d2, 0, 1, N};
}

__global__ void kpp_x_partial_kernel(const double* __restrict__ d2, int64_t N, int64_t S, const KppState* st,
                                     double* __restrict__ approx) {
  if (!st->need_exact) return;
  const KppView x = kpp_view(d2, N, blockIdx.y);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = g * kt::xsum::kSeg;
  if (lo >= x.n) return;
  const int64_t hi = min(x.n, lo + kt::xsum::kSeg);
  double s = 0.0;
  for (int64_t i = lo; i < hi; ++i) s = kt::dadd(s, x(i));
  approx[blockIdx.y * S + g] = s;
}

__global__ void kpp_x_prefix_kernel(int64_t N, int64_t S, const KppState* st, double* __restrict__ approx) {
  if (!st->need_exact) return;
  const int v = threadIdx.x >> 5;
  if (v >= kKppViews) return;
  const int64_t n = v < 4 ? (N >= 4 ? N / 4 : 0) : N;
  warp_exclusive_scan(approx + v * S, (n + kt::xsum::kSeg - 1) / kt::xsum::kSeg, 1);
}

__global__ void kpp_x_map_kernel(const double* __restrict__ d2, int64_t N, int64_t S, const KppState* st,
                                 const double* __restrict__ prefix, kt::xsum::SegMap* __restrict__ maps) {
  if (!st->need_exact) return;
  const KppView x = kpp_view(d2, N, blockIdx.y);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = g * kt::xsum::kSeg;
  if (lo >= x.n) return;
  const int len = (int)(min(x.n, lo + kt::xsum::kSeg) - lo);
  auto at = [&](int i) { return x(lo + i); };
  const double p = prefix[blockIdx.y * S + g];
  maps[blockIdx.y * S + g] = p > 0.0 ? kt::xsum::segment_map(at, len, kt::xsum::binade_of(p))
                                     : kt::xsum::zero_segment_map(at, len);
}

// 4 warps: the exact lane sums -> total -> r; then warp 0 walks the natural-order
// composition batch by batch and, in the batch where the exact running sum first
// exceeds r, segment by segment, then element by element.
__global__ void __launch_bounds__(128) kpp_x_pick_kernel(const double* __restrict__ d2, int64_t N, int64_t S,
                                                         KppState* st, const kt::xsum::SegMap* __restrict__ maps) {
  __shared__ double lanes[4];
  __shared__ double sh_r;
  __shared__ int sh_case;  // 0: below(N) already picked, 1: search cum > r
  if (!st->need_exact) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const KppView x = kpp_view(d2, N, w);
    const int64_t nseg = (x.n + kt::xsum::kSeg - 1) / kt::xsum::kSeg;
    int nseq = 0;
    const double s = x.n > 0 ? warp_compose([&](int i) { return x(i); }, [&](int g) { return maps[w * S + g]; },
                                            (int)nseg, (int)x.n, &nseq)
                             : 0.0;
    if (lane == 0) lanes[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Eigen's vectorised sum (the shim's pinned order, see oracle/eigen_shim/Eigen/Core)
    const int64_t aligned2 = (N / 4) * 4, aligned = (N / 2) * 2;
    double total;
    if (aligned == 0) {
      total = d2[0];
      for (int64_t i = 1; i < N; ++i) total = kt::dadd(total, d2[i]);
    } else {
      double a0 = d2[0], a1 = d2[1];
      if (aligned > 2) {
        a0 = kt::dadd(lanes[0], lanes[2]);
        a1 = kt::dadd(lanes[1], lanes[3]);
        if (aligned > aligned2) {
          a0 = kt::dadd(a0, d2[aligned2]);
          a1 = kt::dadd(a1, d2[aligned2 + 1]);
        }
      }
      total = kt::dadd(a0, a1);
      for (int64_t i = aligned; i < N; ++i) total = kt::dadd(total, d2[i]);
    }
    uint64_t rng = st->rng_fb;
    if (total <= 0.0) {
      st->pick = (int64_t)kt::rng_below(rng, (uint64_t)N);
      sh_case = 0;
    } else {
      sh_r = kt::dmul(kt::rng_uniform01(rng), total);
      sh_case = 1;
    }
    st->rng = rng;
    st->fallbacks += 1;
  }
  __syncthreads();
  if (w != 0 || sh_case == 0) {
    if (threadIdx.x == 0) st->need_exact = 0;
    return;
  }
  const double r = sh_r;
  const KppView x = kpp_view(d2, N, 4);
  const kt::xsum::SegMap* m4 = maps + 4 * S;
  const int nseg = (int)((N + kt::xsum::kSeg - 1) / kt::xsum::kSeg);
  double s = 0.0;  // cum = 0.0, then += in order
  int64_t pick = N - 1;
  bool found = false;
  for (int g0 = 0; g0 < nseg && !found; g0 += 32) {
    const int mcount = min(32, nseg - g0);
    kt::xsum::SegMap mine{0, 0, 0, 2};
    if (lane < mcount) mine = m4[g0 + lane];
    // whole batch at once when every map is valid in one binade and the batch ends <= r
    const unsigned real = __ballot_sync(0xffffffff, lane < mcount && mine.ok != 2);
    if (real == 0) continue;  // all-zero segments: cum unchanged
    const int e0 = __shfl_sync(0xffffffff, mine.e, __ffs(real) - 1);
    const bool uniform = __all_sync(0xffffffff, lane >= mcount || mine.ok == 2 || (mine.ok == 1 && mine.e == e0));
    if (uniform && s > 0.0) {
      uint64_t c0 = mine.ok == 2 ? 0 : mine.F0, c1 = mine.ok == 2 ? 0 : mine.F1;
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t p0 = __shfl_up_sync(0xffffffff, c0, off);
        const uint64_t p1 = __shfl_up_sync(0xffffffff, c1, off);
        if (lane >= off) {
          const uint64_t n0 = p0 + ((p0 & 1u) ? c1 : c0);
          const uint64_t n1 = p1 + (((1u + p1) & 1u) ? c1 : c0);
          c0 = n0;
          c1 = n1;
        }
      }
      kt::xsum::SegMap all;
      all.F0 = __shfl_sync(0xffffffff, c0, mcount - 1);
      all.F1 = __shfl_sync(0xffffffff, c1, mcount - 1);
      all.e = e0;
      all.ok = all.F0 < (1ull << 53) && all.F1 < (1ull << 53);
      double s_end = s;
      if (kt::xsum::apply_map(s_end, all) && !(s_end > r)) {
        s = s_end;
        continue;
      }
    }
    for (int q = 0; q < mcount && !found; ++q) {
      kt::xsum::SegMap m;
      m.F0 = __shfl_sync(0xffffffff, mine.F0, q);
      m.F1 = __shfl_sync(0xffffffff, mine.F1, q);
      m.e = __shfl_sync(0xffffffff, mine.e, q);
      m.ok = __shfl_sync(0xffffffff, mine.ok, q);
      const int lo = (g0 + q) * kt::xsum::kSeg, hi = (int)(N < (int64_t)lo + kt::xsum::kSeg ? N : (int64_t)lo + kt::xsum::kSeg);
      double s_next = s;
      if (!kt::xsum::apply_map(s_next, m)) s_next = warp_seq_segment(s, [&](int i) { return x(i); }, lo, hi);
      if (s_next > r) {  // the first i with cum > r lies in this segment
        double c = s;
        for (int i = lo; i < hi; ++i) {
          c = kt::dadd(c, x(i));
          if (c > r) {
            pick = i;
            break;
          }
        }
        found = true;
      }
      s = s_next;
    }
  }
  if (lane == 0) {
    st->pick = pick;
    st->need_exact = 0;
  }
}

// 1024-thread block per (cluster c, knob d): compose the segment maps from s = 0 exactly;
// centroid = s / count (sampling.cpp:110-121).
template <class IdxT>
__global__ void __launch_bounds__(1024) xs_compose_kernel(KtSpaceParams sp, const IdxT* __restrict__ sorted,
                                                          const int32_t* __restrict__ counts,
                                                          const int32_t* __restrict__ cstart,
                                                          const int32_t* __restrict__ csb, int k,
                                                          const kt::xsum::SegMap* __restrict__ maps,
                                                          double* __restrict__ cent, int32_t* __restrict__ seq_segments) {
  const int D = sp.D;
  const int c = blockIdx.x / D, d = blockIdx.x % D;
  const int n = counts[c];
  if (n == 0) return;  // empty cluster: reseeded
  const double* lut = sp.lut + sp.lut_off[d];
  const IdxT* rows = sorted + (int64_t)cstart[c] * D + d;
  const int gb = csb[c], nseg = csb[c + 1] - csb[c];
  int nseq = 0;
  const double s = block_compose([&](int i) { return __ldg(lut + (int)rows[(int64_t)i * D]); },
                                 [&](int g) { return maps[(int64_t)(gb + g) * D + d]; }, nseg, n, &nseq);
  if (threadIdx.x == 0) {
    cent[c * D + d] = kt::ddiv(s, (double)n);
    if (nseq) atomicAdd(seq_segments, nseq);
  }
}

// ---- exact loss: the sequential sum of per-point d2 (sampling.cpp:56-63) -----
__global__ void xs_loss_partial_kernel(const double* __restrict__ x, int64_t N, double* __restrict__ approx) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = g * kt::xsum::kSeg;
  if (lo >= N) return;
  const int64_t hi = min(N, lo + kt::xsum::kSeg);
  double s = 0.0;
  for (int64_t i = lo; i < hi; ++i) s = kt::dadd(s, x[i]);
  approx[g] = s;
}

__global__ void xs_loss_map_kernel(const double* __restrict__ x, int64_t N, const double* __restrict__ prefix,
                                   kt::xsum::SegMap* __restrict__ maps) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = g * kt::xsum::kSeg;
  if (lo >= N) return;
  const int len = (int)(min(N, lo + kt::xsum::kSeg) - lo);
  auto at = [&](int i) { return x[lo + i]; };
  maps[g] = prefix[g] > 0.0 ? kt::xsum::segment_map(at, len, kt::xsum::binade_of(prefix[g]))
                            : kt::xsum::zero_segment_map(at, len);
}

__global__ void __launch_bounds__(1024) xs_loss_compose_kernel(const double* __restrict__ x, int64_t N,
                                                               const double* __restrict__ approx,
                                                               double* __restrict__ prefix,
                                                               const kt::xsum::SegMap* __restrict__ maps, int phase,
                                                               double* out) {
  const int64_t nseg = (N + kt::xsum::kSeg - 1) / kt::xsum::kSeg;
  if (phase == 0) {  // exclusive prefix of the approximate segment sums
    for (int64_t g = threadIdx.x; g < nseg; g += blockDim.x) prefix[g] = approx[g];
    __syncthreads();
    block_exclusive_scan<double>(prefix, nseg, 1, [](double a, double b) { return kt::dadd(a, b); });
    return;
  }
  int nseq = 0;
  const double s = block_compose([&](int i) { return x[i]; }, [&](int g) { return maps[g]; }, (int)nseg, (int)N, &nseq);
  if (threadIdx.x == 0) *out = s;
}

// Empty clusters (sampling.cpp:122-136): in cluster order, the unclaimed
// point farthest from its OLD centroid (strict >, first index on ties).
template <class IdxT>
__global__ void __launch_bounds__(1024) reseed_kernel(KtSpaceParams sp,
                                                      const IdxT* __restrict__ pts, int64_t N,
                                                      const int32_t* __restrict__ counts, int k,
                                                      const double* __restrict__ d2_old,
                                                      double* __restrict__ cent,
                                                      int32_t* __restrict__ nempty) {
  __shared__ int64_t claimed[kt::kMaxK];
  __shared__ int nclaimed;
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  const int D = sp.D;
  if (threadIdx.x == 0) nclaimed = 0;
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    if (counts[c] > 0) continue;
    double best = -1.0;
    int64_t besti = 0;
    bool have = false;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
      bool cl = false;
      for (int q = 0; q < nclaimed; ++q) cl |= claimed[q] == i;
      if (cl) continue;
      const double v = d2_old[i];
      if (!have || v > best) {  // per-thread indices ascend, so first max kept
        best = v;
        besti = i;
        have = true;
      }
    }
    if (!have) {
      best = -INFINITY;
      besti = INT64_MAX;
    }
    // (value desc, index asc) reduction
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffff, best, o);
      const int64_t oi = __shfl_down_sync(0xffffffff, besti, o);
      if (ov > best || (ov == best && oi < besti)) {
        best = ov;
        besti = oi;
      }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
      bv[w] = best;
      bi[w] = besti;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = bv[0];
      int64_t ii = bi[0];
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (bv[q] > b || (bv[q] == b && bi[q] < ii)) {
          b = bv[q];
          ii = bi[q];
        }
      // worst starts at -1.0 with strict >: all d2 >= 0, the first unclaimed point qualifies
      claimed[nclaimed++] = ii;
      for (int d = 0; d < D; ++d) cent[c * D + d] = sp.lut[sp.lut_off[d] + (int)pts[ii * D + d]];
      atomicAdd(nempty, 1);
    }
    __syncthreads();
  }
}

__global__ void sum_chunks_kernel(const double* __restrict__ cs, int64_t n, double* out) {
  __shared__ double red[32];
  double p = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) p = kt::dadd(p, cs[i]);
  const double s = block_sum(p, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void count_diff_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                                  int64_t N, unsigned long long* out) {
  int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    c += a[i] != b[i];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffff, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// ------------------------------------------------------------------ snap (K6)
// Eigen contiguous squaredNorm over D.
__device__ double eigen_sqnorm_diff(const double* x, const double* c, int n) {
  auto f = [&](int i) {
    const double t = kt::dsub(x[i], c[i]);
    return kt::dmul(t, t);
  };
  const int a2 = (n / 4) * 4, a = (n / 2) * 2;
  if (a == 0) {
    double s = f(0);
    for (int i = 1; i < n; ++i) s = kt::dadd(s, f(i));
    return s;
  }
  double p0 = f(0), p1 = f(1);
  if (a > 2) {
    double q0 = f(2), q1 = f(3);
    for (int i = 4; i < a2; i += 4) {
      p0 = kt::dadd(p0, f(i));
      p1 = kt::dadd(p1, f(i + 1));
      q0 = kt::dadd(q0, f(i + 2));
      q1 = kt::dadd(q1, f(i + 3));
    }
    p0 = kt::dadd(p0, q0);
    p1 = kt::dadd(p1, q1);
    if (a > a2) {
      p0 = kt::dadd(p0, f(a2));
      p1 = kt::dadd(p1, f(a2 + 1));
    }
  }
  double s = kt::dadd(p0, p1);
  for (int i = a; i < n; ++i) s = kt::dadd(s, f(i));
  return s;
}

// Rounding (sampling.cpp:209-214) + validity; flags[c] = 1 when a fallback is needed.
__global__ void snap_round_kernel(KtSpaceParams sp, const double* __restrict__ cent, int k,
                                  int32_t* __restrict__ out, int32_t* __restrict__ need) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  const int D = sp.D;
  for (int d = 0; d < D; ++d) {
    const int card = sp.card[d];
    int v = (int)floor(kt::dadd(kt::dmul(cent[c * D + d], (double)(card - 1)), 0.5));
    v = v < 0 ? 0 : (v > card - 1 ? card - 1 : v);
    out[c * D + d] = v;
  }
  const int32_t* row = out + c * D;
  need[c] = kt::rule_eval(sp, [&](int d) { return (int)row[d]; }) ? 0 : 1;
}

struct SnapKey {
  unsigned long long hi;  // (invalid << 63) | (d2 bits >> 1) -- d2 >= 0 so bit 63 is 0
  unsigned long long lo;  // (d2 bit 0 << 63) | id >> 1 ... packed below
};

// Per (centroid, block): best (invalid, d2, id) candidate; lexicographic min.
template <class IdxT>
__global__ void __launch_bounds__(kBT) snap_fallback_kernel(KtSpaceParams sp, int lut_total,
                                                            const double* __restrict__ cent,
                                                            const int32_t* __restrict__ need,
                                                            const IdxT* __restrict__ cand,
                                                            const uint64_t* __restrict__ ids,
                                                            int64_t N,
                                                            unsigned long long* __restrict__ part) {
  extern __shared__ double sdyn[];
  const int c = blockIdx.y;
  const int D = sp.D;
  unsigned long long* outp = part + ((int64_t)c * gridDim.x + blockIdx.x) * 4;
  if (!need[c]) {
    if (threadIdx.x == 0) outp[0] = outp[1] = outp[2] = outp[3] = ~0ull;
    return;
  }
  const double* lut = stage_lut(sp, sdyn, lut_total);
  __shared__ double cc[kt::kMaxKnobs];
  if (threadIdx.x < D) cc[threadIdx.x] = cent[c * D + threadIdx.x];
  __syncthreads();
  // key (invalid, d2 bits, id) and the row it came from (ids are unique: the key decides)
  unsigned long long b0 = ~0ull, b1 = ~0ull, b2 = ~0ull, b3 = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const IdxT* row = cand + i * D;
    const bool valid = kt::rule_eval(sp, [&](int d) { return (int)row[d]; });
    double x[kt::kMaxKnobs];
    for (int d = 0; d < D; ++d) x[d] = lut[sp.lut_off[d] + (int)row[d]];
    const double d2 = eigen_sqnorm_diff(x, cc, D);
    const unsigned long long k0 = valid ? 0ull : 1ull;
    const unsigned long long k1 = (unsigned long long)__double_as_longlong(d2);
    const unsigned long long k2 = ids[i];
    if (k0 < b0 || (k0 == b0 && (k1 < b1 || (k1 == b1 && k2 < b2)))) {
      b0 = k0;
      b1 = k1;
      b2 = k2;
      b3 = (unsigned long long)i;
    }
  }
  __shared__ unsigned long long s0[kBT], s1[kBT], s2[kBT], s3[kBT];
  s0[threadIdx.x] = b0;
  s1[threadIdx.x] = b1;
  s2[threadIdx.x] = b2;
  s3[threadIdx.x] = b3;
  __syncthreads();
  for (int o = kBT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const int q = threadIdx.x + o;
      if (s0[q] < s0[threadIdx.x] ||
          (s0[q] == s0[threadIdx.x] && (s1[q] < s1[threadIdx.x] || (s1[q] == s1[threadIdx.x] && s2[q] < s2[threadIdx.x])))) {
        s0[threadIdx.x] = s0[q];
        s1[threadIdx.x] = s1[q];
        s2[threadIdx.x] = s2[q];
        s3[threadIdx.x] = s3[q];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    outp[0] = s0[0];
    outp[1] = s1[0];
    outp[2] = s2[0];
    outp[3] = s3[0];
  }
}

template <class IdxT>
__global__ void snap_reduce_kernel(KtSpaceParams sp, const int32_t* __restrict__ need,
                                   const unsigned long long* __restrict__ part, int nblk,
                                   const IdxT* __restrict__ cand, const uint64_t* __restrict__ ids,
                                   int64_t N, int32_t* __restrict__ out) {
  const int c = blockIdx.x;
  if (!need[c] || threadIdx.x != 0) return;
  const unsigned long long* p = part + (int64_t)c * nblk * 4;
  unsigned long long b0 = ~0ull, b1 = ~0ull, b2 = ~0ull, b3 = ~0ull;
  for (int q = 0; q < nblk; ++q) {
    const unsigned long long k0 = p[4 * q], k1 = p[4 * q + 1], k2 = p[4 * q + 2];
    if (k0 < b0 || (k0 == b0 && (k1 < b1 || (k1 == b1 && k2 < b2)))) {
      b0 = k0;
      b1 = k1;
      b2 = k2;
      b3 = p[4 * q + 3];
    }
  }
  if (b0 == ~0ull) return;  // no candidates: keep the rounding (sampling.cpp:233)
  for (int d = 0; d < sp.D; ++d) out[c * sp.D + d] = (int32_t)cand[(int64_t)b3 * sp.D + d];
}

// ------------------------------------------------------------------ host orchestration
struct Run {
  // device
  double* cent;      // k x D
  int32_t* asg;
  double* d2;
  double loss_est;   // parallel estimate
  double loss_exact; // NaN unless computed
  std::vector<double> iter_losses;
};

struct IterReadback {
  double loss;
  unsigned long long changed;
  int32_t seq, segs;
  unsigned long long unc;
  unsigned long long empty;  // certified mode: empty clusters seen by centroids_from_sums
};
// Collects an iteration's scalars for one host readback and clears the
// sequential-segment counter for the next centroid update.
__global__ void gather_readback_kernel(const double* dscal, const unsigned long long* ull, int32_t* seqcnt,
                                       const int32_t* segs, IterReadback* outs, int* slot = nullptr) {
  IterReadback* out = slot ? outs + (*slot)++ : outs;
  out->loss = dscal[0];
  out->changed = ull[0];
  out->seq = *seqcnt;
  out->segs = *segs;
  out->unc = ull[2];
  out->empty = ull[3];
  *seqcnt = 0;
}

// Certified iteration tail in one launch: the loss estimate over the chunk sums, the
// iteration's readback, then the counters cleared for the next iteration.
__global__ void __launch_bounds__(1024) sum_gather_kernel(const double* __restrict__ cs, int64_t n, double* dscal,
                                                          unsigned long long* ull, int32_t* seqcnt,
                                                          const int32_t* segs, IterReadback* outs, int* slot) {
  __shared__ double red[32];
  double p = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) p = kt::dadd(p, cs[i]);
  const double s = block_sum(p, red);
  if (threadIdx.x == 0) {
    dscal[0] = s;
    IterReadback* out = outs + (*slot)++;
    out->loss = s;
    out->changed = ull[0];
    out->seq = *seqcnt;
    out->segs = *segs;
    out->unc = ull[2];
    out->empty = ull[3];
    *seqcnt = 0;
    ull[0] = ull[1] = ull[2] = ull[3] = 0;
  }
}

// CUDA graph capture is illegal on the legacy default stream (a context bound to
// torch's default stream); those runs take the uncaptured paths.
inline bool capturable(cudaStream_t st) { return st != nullptr && st != cudaStreamLegacy; }

// Ends an open stream capture if an error unwinds through it, so that a failed
// capture does not leave the stream (and, in thread-local mode, the thread) capturing.
struct CaptureGuard {
  cudaStream_t s;
  bool open = true;
  void end(cudaGraph_t* g) {
    open = false;
    KT_CUDA(cudaStreamEndCapture(s, g));
  }
  ~CaptureGuard() {
    if (!open) return;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
};

template <class IdxT>
struct KMeans {
  ktune_ctx* ctx;
  const ktune_space* sp;
  const IdxT* pts;  // device
  int64_t N;
  int D;
  int lut_total;
  int64_t nchunks;
  size_t lut_smem;
  // workspace
  double* d2;         // kmeans++ d2
  double* chunk;      // chunk sums
  double* scratch;    // chunk prefix
  KppState* kst;
  int32_t* asg_a;     // current assignment
  int32_t* asg_b;     // next assignment
  double* d2_a;       // per-point d2 of current assignment
  double* d2_b;
  int32_t* members;
  int32_t* blockcounts;
  int32_t* counts;    // [k] + cstart [k] + nempty
  double* cent_a;
  double* cent_b;
  unsigned long long* isum[2] = {nullptr, nullptr};  // certified mode: integer sums [k*D] + counts [k]
  double* cB = nullptr;  // certified mode: centroids from the integer sums and their bounds
  double* dB = nullptr;
  int* rb_slot = nullptr;           // next readback slot of a batched certified run
  IterReadback* rb_dev = nullptr;   // per-iteration scalars (device) ...
  IterReadback* rb_host = nullptr;  // ... and their pinned host copy
  unsigned long long* ull;  // [0] changed, [1] diff
  double* dscal;      // [0] loss sum, [1] exact loss
  // best-of-restarts and previous-k best (for exact fallbacks)
  int32_t* best_asg;
  double* best_d2;
  double* best_cent;
  int32_t* prev_asg;
  double* prev_d2;
  // exact-sum machinery
  IdxT* sorted;       // members' rows, cluster-major, ascending point order
  double* xs_approx;  // per (segment, knob) approximate sums / prefixes
  kt::xsum::SegMap* xs_maps;
  int max_segs;
  int32_t* csb;       // per-cluster segment bases [k+1]
  int32_t* seqcnt;    // segments summed sequentially (stat)
  int world = 1, rank = 0;
  bool sharded = false;  // per-point state all-gathered over NCCL (world > 1, or forced for tests)
  int64_t shard_chunks = 0, cap = 0;
  double* tile_sum = nullptr;  // tcgen05 assign: per-128-point-tile loss partials
  bool use_tc = false;         // tcgen05 screening assignment (KTUNE_OPT_KMEANS_MODE = 3; measured slower)
  double* dzero = nullptr;      // all-zero bound block: assign_cert_kernel against exact centroids
  size_t screen_smem = 0;

  void setup(ktune_ctx* c, const ktune_space* s, const IdxT* p, int64_t n) {
    ctx = c;
    sp = s;
    pts = p;
    N = n;
    D = s->D;
    lut_total = s->lut_total;
    nchunks = kt::ceil_div(N, kChunk);
    // multi-GPU: rank r assigns chunks [r*shard_chunks, (r+1)*shard_chunks); the
    // per-point results are all-gathered so every rank holds the full state.
    world = ctx->world;
    rank = ctx->rank;
    sharded = world > 1 || (ctx->opt_force_sharded && ctx->nccl);
    shard_chunks = kt::ceil_div(nchunks, world);
    cap = (int64_t)world * shard_chunks * kChunk;
    lut_smem = sizeof(double) * lut_total;
    d2 = (double*)ctx->dev(kt::WS_D2, sizeof(double) * N);
    chunk = (double*)ctx->dev(kt::WS_BLOCK, sizeof(double) * world * shard_chunks);
    scratch = (double*)ctx->dev(kt::WS_BLOCK2, sizeof(double) * nchunks);
    kst = (KppState*)ctx->dev(kt::WS_KPP, sizeof(KppState));
    asg_a = (int32_t*)ctx->dev(kt::WS_ASSIGN, sizeof(int32_t) * cap);
    asg_b = (int32_t*)ctx->dev(kt::WS_ASSIGN2, sizeof(int32_t) * cap);
    d2_a = (double*)ctx->dev(kt::WS_D2B, sizeof(double) * cap * 2);
    d2_b = d2_a + cap;
    members = (int32_t*)ctx->dev(kt::WS_MEMBERS, sizeof(int32_t) * N);
    blockcounts = (int32_t*)ctx->dev(kt::WS_SCRATCH, sizeof(int32_t) * nchunks * kt::kMaxK);
    counts = (int32_t*)ctx->dev(kt::WS_SCRATCH2, sizeof(int32_t) * (4 * kt::kMaxK + 16));
    csb = counts + 2 * kt::kMaxK + 8;
    seqcnt = csb + kt::kMaxK + 4;
    max_segs = (int)(kt::ceil_div(N, kt::xsum::kSeg) + kt::kMaxK);
    tile_sum = (double*)ctx->dev(kt::WS_TILESUM, sizeof(double) * (size_t)world * shard_chunks * (kChunk / kTcPts));
    use_tc = ctx->opt_kmeans_mode == 3 && D <= 16 &&
             (size_t)lut_total * 8 + kTcPts * kTcK * 2 + kTcMaxN * kTcK * 2 + (kt::kMaxK * kt::kMaxKnobs + kt::kMaxK) * 8 <= 200 * 1024;
    for (int d = 0; d < D; ++d) use_tc = use_tc && s->card[d] <= 2048;  // idx exact in fp16
    sorted = (IdxT*)ctx->dev(kt::WS_SORTED, sizeof(IdxT) * N * D);
    xs_approx = (double*)ctx->dev(kt::WS_XS_APPROX, sizeof(double) * (size_t)max_segs * D);
    xs_maps = (kt::xsum::SegMap*)ctx->dev(kt::WS_XS_MAPS, sizeof(kt::xsum::SegMap) * (size_t)max_segs * D);
    KT_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (4 * kt::kMaxK + 16), ctx->stream));
    cent_a = (double*)ctx->dev(kt::WS_CENT, sizeof(double) * kt::kMaxK * D * 3);
    cent_b = cent_a + kt::kMaxK * D;
    best_cent = cent_b + kt::kMaxK * D;
    ull = (unsigned long long*)ctx->dev(kt::WS_VALID, 64);
    rb_dev = (IterReadback*)ctx->dev(kt::WS_XS_RB, sizeof(IterReadback) * 8 + 64);
    rb_slot = reinterpret_cast<int*>(rb_dev + 8);
    {
      const size_t words = (size_t)kt::kMaxK * (kt::kMaxKnobs + 1);
      const size_t nb = kt::kMaxK * kt::kMaxKnobs + kt::kMaxK;  // bound block: [k x D] deltas, [kMaxK] E_c
      unsigned long long* w = (unsigned long long*)ctx->dev(
          kt::WS_KM_CERT, sizeof(unsigned long long) * words * 2 + sizeof(double) * (kt::kMaxK * kt::kMaxKnobs + 2 * nb));
      isum[0] = w;
      isum[1] = w + words;
      cB = reinterpret_cast<double*>(w + 2 * words);
      dB = cB + kt::kMaxK * kt::kMaxKnobs;  // [k x D] deltas, then [kMaxK] per-cluster bounds
      dzero = dB + nb;                      // exact centroids: every bound 0
      KT_CUDA(cudaMemsetAsync(dzero, 0, sizeof(double) * nb, ctx->stream));
    }
    screen_smem = cert_smem_bytes(kt::kMaxK, D, D <= 8 ? 8 : (D <= 16 ? 16 : kt::kMaxKnobs), lut_smem);
    KT_DISPATCH_DM(D, KT_CUDA(cudaFuncSetAttribute(assign_cert_kernel<IdxT, DM_>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)screen_smem)));
    rb_host = (IterReadback*)ctx->host(3, sizeof(IterReadback) * 8);
    dscal = (double*)ctx->dev(kt::WS_SNAP, 64);
    best_asg = (int32_t*)ctx->dev(kt::WS_BEST_ASSIGN, sizeof(int32_t) * N);
    best_d2 = (double*)ctx->dev(kt::WS_BEST_D2, sizeof(double) * N);
    prev_asg = (int32_t*)ctx->dev(kt::WS_PREV_ASSIGN, sizeof(int32_t) * N);
    prev_d2 = (double*)ctx->dev(kt::WS_PREV_D2, sizeof(double) * N);
  }

  cudaStream_t s() const { return ctx->stream; }
  // cluster_sums_kernel grid: a few blocks per SM, at most 1024 chunks (1M points) per block so that
  // its int32 shared-memory sums (<= 2^20 x 2047) cannot overflow
  unsigned sums_grid() const {
    return (unsigned)std::max<int64_t>(std::min<int64_t>(nchunks, (int64_t)kt::sm_count(ctx) * 8),
                                       kt::ceil_div(nchunks, 1024));
  }
  int grid_pts() const { return (int)nchunks; }

  // exact-replay workspace of kmeans++ (allocated before any capture: no cudaMalloc while capturing)
  double* kpp_x_buffer() {
    const int64_t S = kt::ceil_div(N, kt::xsum::kSeg);
    return (double*)ctx->dev(kt::WS_KPP_X, (sizeof(double) + sizeof(kt::xsum::SegMap)) * kKppViews * S);
  }

  // One kmeans++ round: the distance update for centroid st->c, then (if another pick follows)
  // the certified pick and its exact replay (a no-op unless kpp_select left the pick undecided).
  // Nothing in it depends on the host, so it is captured once per KMeans object and replayed.
  void kpp_round(bool pick) {
    kpp_d2_kernel<IdxT><<<grid_pts(), kBT, lut_smem, s()>>>(sp->params, lut_total, pts, N, kst, cent_a, d2, chunk);
    kt::check_launch(ctx, "kpp_d2");
    if (!pick) return;
    kpp_select_kernel<<<1, 1024, 0, s()>>>(d2, chunk, N, kst, 1, (int)ctx->opt_force_exact, scratch);
    const int64_t S = kt::ceil_div(N, kt::xsum::kSeg);
    double* xa = kpp_x_buffer();
    kt::xsum::SegMap* xm = reinterpret_cast<kt::xsum::SegMap*>(xa + kKppViews * S);
    const dim3 gv((unsigned)kt::ceil_div(S, 128), kKppViews);
    kpp_x_partial_kernel<<<gv, 128, 0, s()>>>(d2, N, S, kst, xa);
    kpp_x_prefix_kernel<<<1, 32 * kKppViews, 0, s()>>>(N, S, kst, xa);
    kpp_x_map_kernel<<<gv, 128, 0, s()>>>(d2, N, S, kst, xa, xm);
    kpp_x_pick_kernel<<<1, 128, 0, s()>>>(d2, N, S, kst, xm);
    kt::check_launch(ctx, "kpp_select", 5);
  }

  // captured rounds, one per centroid buffer (cent_a and cent_b swap roles between restarts;
  // every other pointer of the round is fixed for this object)
  cudaGraphExec_t kpp_graph[2] = {nullptr, nullptr};
  const double* kpp_graph_cent[2] = {nullptr, nullptr};
  int64_t kpp_graph_force_exact[2] = {0, 0};
  KMeans() = default;
  KMeans(const KMeans&) = delete;
  KMeans& operator=(const KMeans&) = delete;
  ~KMeans() {
    for (auto& g : kpp_graph)
      if (g) cudaGraphExecDestroy(g);
  }

  void kmeanspp(int k, uint64_t rng_seed) {
    KppState h{rng_seed, 0, 0, 0, 0, 0, 0};
    KT_CUDA(cudaMemcpyAsync(kst, &h, sizeof(h), cudaMemcpyHostToDevice, s()));
    kpp_select_kernel<<<1, 1024, 0, s()>>>(d2, chunk, N, kst, 0, 0, scratch);
    kt::check_launch(ctx, "kpp_select");
    // the host launch rate (6 launches per round) bounds an uncaptured kmeans++ round
    const bool use_graph = !ctx->opt_profile && capturable(s()) && k > 2;
    const int gi = kpp_graph_cent[0] == cent_a ? 0 : (kpp_graph_cent[1] == cent_a ? 1 : (kpp_graph[0] ? 1 : 0));
    if (use_graph && kpp_graph[gi] &&
        (kpp_graph_cent[gi] != cent_a || kpp_graph_force_exact[gi] != ctx->opt_force_exact)) {
      cudaGraphExecDestroy(kpp_graph[gi]);
      kpp_graph[gi] = nullptr;
    }
    for (int c = 0; c < k; ++c) {
      if (c + 1 < k && use_graph) {
        if (!kpp_graph[gi]) {
          kpp_x_buffer();
          cudaGraph_t graph;
          KT_CUDA(cudaStreamBeginCapture(s(), cudaStreamCaptureModeThreadLocal));
          CaptureGuard cg{s()};
          kpp_round(true);
          cg.end(&graph);
          KT_CUDA(cudaGraphInstantiate(&kpp_graph[gi], graph, 0));
          cudaGraphDestroy(graph);
          kpp_graph_cent[gi] = cent_a;
          kpp_graph_force_exact[gi] = ctx->opt_force_exact;
        }
        KT_CUDA(cudaGraphLaunch(kpp_graph[gi], s()));
      } else {
        kpp_round(c + 1 < k);
      }
      if (c + 1 < k) ctx->stats[KTUNE_STAT_KPP_PICKS] += 1;
    }
  }

  // assignment against cent; returns loss estimate; changed count if prev != null
  double assign(const double* cent, int k, const int32_t* prev, int32_t* asg, double* dd,
                unsigned long long* changed_out) {
    enqueue_assign(cent, k, prev, asg, dd);
    return finish_assign(prev, changed_out);
  }

  // Stream work of one assignment pass (no host synchronisation: capturable into a
  // CUDA graph), ending with the iteration's scalars copied into pinned memory.
  void enqueue_assign(const double* cent, int k, const int32_t* prev, int32_t* asg, double* dd) {
    KT_CUDA(cudaMemsetAsync(ull, 0, 32, s()));  // changed, -, uncertain, empty (all read back)
    const size_t smem = sizeof(double) * (k * D) + lut_smem;
    if (use_tc && k <= kTcMaxN && k >= kTcMinK) {
      // tcgen05 screening + certified exact winner (this rank's chunk range)
      const int64_t c0 = (int64_t)rank * shard_chunks;
      const int64_t cend = std::min<int64_t>(nchunks, c0 + shard_chunks);
      const int64_t t0 = c0 * (kChunk / kTcPts), t1 = std::min<int64_t>(kt::ceil_div(N, kTcPts), cend * (kChunk / kTcPts));
      const size_t tsmem = kTcPts * kTcK * 2 + kTcMaxN * kTcK * 2 + (kt::kMaxK * kt::kMaxKnobs + kt::kMaxK) * 8 + lut_smem;
      if (t1 > t0) {
        kt::ProfScope prof(ctx, KTUNE_STAT_ASSIGN_NS);
        KT_CUDA(cudaFuncSetAttribute(assign_tc_kernel<IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
        const int grid = (int)std::min<int64_t>(t1 - t0, (int64_t)kt::sm_count(ctx) * 4);
        assign_tc_kernel<IdxT><<<grid, kTcPts, tsmem, s()>>>(sp->params, lut_total, pts, N, cent, k, prev, asg, dd,
                                                             tile_sum, ull, t0, t1);
        kt::check_launch(ctx, "assign_tc");
        sum_chunks_kernel<<<1, 1024, 0, s()>>>(tile_sum + t0, t1 - t0, dscal);
      } else {
        KT_CUDA(cudaMemsetAsync(dscal, 0, 8, s()));
      }
      if (sharded) {
        const int64_t S = shard_chunks * kChunk;
        kt::allgather(ctx, asg + rank * S, asg, sizeof(int32_t) * S);
        kt::allgather(ctx, dd + rank * S, dd, sizeof(double) * S);
        kt::allreduce_sum(ctx, ull, 1, false);
        kt::allreduce_sum(ctx, dscal, 1, true);
      }
    } else if (ctx->opt_kmeans_mode != 1) {
      // fp32 screening against the exact centroids (zero centroid bounds), the winner's d2
      // and near ties in the reference's fp64 order: exact assignment, d2 and chunk sums
      const int64_t c0 = sharded ? (int64_t)rank * shard_chunks : 0;
      const int64_t nloc = sharded ? std::max<int64_t>(0, std::min<int64_t>(nchunks, c0 + shard_chunks) - c0) : nchunks;
      if (nloc > 0) {
        kt::ProfScope prof(ctx, KTUNE_STAT_ASSIGN_NS);
        KT_DISPATCH_DM(D, assign_cert_kernel<IdxT, DM_><<<(unsigned)nloc, kCertBT, cert_smem_bytes(k, D, DM_, lut_smem), s()>>>(
                              sp->params, lut_total, pts, N, cent, dzero, k, prev, asg, dd, chunk, ull, nullptr,
                              nullptr, c0));
        kt::check_launch(ctx, "assign_screen");
      }
      if (sharded) {
        if (nloc < shard_chunks)  // zero the padding chunks of the last shard
          KT_CUDA(cudaMemsetAsync(chunk + c0 + nloc, 0, sizeof(double) * (shard_chunks - nloc), s()));
        const int64_t S = shard_chunks * kChunk;
        kt::allgather(ctx, asg + rank * S, asg, sizeof(int32_t) * S);
        kt::allgather(ctx, dd + rank * S, dd, sizeof(double) * S);
        kt::allgather(ctx, chunk + c0, chunk, sizeof(double) * shard_chunks);
        kt::allreduce_sum(ctx, ull, 1, false);
      }
      KT_CUDA(cudaMemsetAsync(ull + 2, 0, 8, s()));  // near ties were resolved by the exact scan
    } else if (!sharded) {
      kt::ProfScope prof(ctx, KTUNE_STAT_ASSIGN_NS);
      KT_DISPATCH_DM(D, assign_kernel<IdxT, DM_><<<grid_pts(), kBT, smem, s()>>>(sp->params, lut_total, pts, N, cent,
                                                                                 k, prev, asg, dd, chunk, ull, 0));
      kt::check_launch(ctx, "assign");
    } else {
      const int64_t c0 = (int64_t)rank * shard_chunks;
      const int64_t nloc = std::max<int64_t>(0, std::min<int64_t>(nchunks, c0 + shard_chunks) - c0);
      if (nloc > 0) {
        kt::ProfScope prof(ctx, KTUNE_STAT_ASSIGN_NS);
        KT_DISPATCH_DM(D, assign_kernel<IdxT, DM_><<<(unsigned)nloc, kBT, smem, s()>>>(
                              sp->params, lut_total, pts, N, cent, k, prev, asg, dd, chunk, ull, c0));
        kt::check_launch(ctx, "assign");
      }
      if (nloc < shard_chunks)  // zero the padding chunks of the last shard
        KT_CUDA(cudaMemsetAsync(chunk + c0 + nloc, 0, sizeof(double) * (shard_chunks - nloc), s()));
      const int64_t S = shard_chunks * kChunk;
      kt::allgather(ctx, asg + rank * S, asg, sizeof(int32_t) * S);
      kt::allgather(ctx, dd + rank * S, dd, sizeof(double) * S);
      kt::allgather(ctx, chunk + c0, chunk, sizeof(double) * shard_chunks);
      kt::allreduce_sum(ctx, ull, 1, false);
    }
    if (!(use_tc && k <= kTcMaxN && k >= kTcMinK)) sum_chunks_kernel<<<1, 1024, 0, s()>>>(chunk, nchunks, dscal);
    kt::check_launch(ctx, "sum_chunks");
    // one gather + one pinned readback per iteration (instead of five pageable copies)
    gather_readback_kernel<<<1, 1, 0, s()>>>(dscal, ull, seqcnt, csb + k, rb_dev);
    kt::check_launch(ctx, "gather_readback");
    KT_CUDA(cudaMemcpyAsync(rb_host, rb_dev, sizeof(IterReadback), cudaMemcpyDeviceToHost, s()));
  }

  double finish_assign(const int32_t* prev, unsigned long long* changed_out) {
    KT_CUDA(cudaStreamSynchronize(s()));
    const IterReadback& h = *rb_host;
    if (prev) {
      ctx->stats[KTUNE_STAT_XS_SEQUENTIAL] += h.seq;
      ctx->stats[KTUNE_STAT_XS_SEGMENTS] += (int64_t)h.segs * D;
    }
    ctx->stats[KTUNE_STAT_ASSIGN_FALLBACKS] += (int64_t)h.unc;
    if (changed_out) *changed_out = h.changed;
    return h.loss;
  }

  void update_centroids(int k, const int32_t* asg, const double* d2_old, double* next) {
    int32_t* cstart = counts + kt::kMaxK;
    hist_kernel<<<grid_pts(), kBT, 0, s()>>>(asg, N, k, blockcounts);
    scan_counts_kernel<<<k, 1024, 0, s()>>>(blockcounts, nchunks, k, counts);
    cluster_starts_kernel<<<1, 32, 0, s()>>>(counts, k, cstart, csb);
    scatter_kernel<IdxT><<<grid_pts(), kBT, 0, s()>>>(asg, N, k, D, pts, blockcounts, cstart, members, sorted);
    // exact in-order centroid sums (exactsum.cuh)
    const int th = 256;
    const int gseg = (int)kt::ceil_div((int64_t)max_segs * D, th);
    xs_partial_kernel<IdxT><<<gseg, th, 0, s()>>>(sp->params, sorted, counts, cstart, csb, k, max_segs, xs_approx);
    xs_prefix_kernel<<<k * D, 1024, 0, s()>>>(D, csb, k, xs_approx);
    xs_map_kernel<IdxT><<<gseg, th, 0, s()>>>(sp->params, sorted, counts, cstart, csb, k, max_segs, xs_approx, xs_maps);
    xs_compose_kernel<IdxT><<<k * D, 1024, 0, s()>>>(sp->params, sorted, counts, cstart, csb, k, xs_maps, next,
                                                     seqcnt);
    KT_CUDA(cudaMemsetAsync(counts + 2 * kt::kMaxK, 0, 4, s()));
    reseed_kernel<IdxT><<<1, 1024, 0, s()>>>(sp->params, pts, N, counts, k, d2_old, next,
                                             counts + 2 * kt::kMaxK);
    kt::check_launch(ctx, "centroid update", 9);
  }

  // The reference's sequential loss (sampling.cpp:56-63), bit-exact, in parallel.
  double exact_loss(const double* dd) {
    const int64_t nseg = kt::ceil_div(N, kt::xsum::kSeg);
    const int g = (int)kt::ceil_div(nseg, 128);
    xs_loss_partial_kernel<<<g, 128, 0, s()>>>(dd, N, xs_approx);
    xs_loss_compose_kernel<<<1, 1024, 0, s()>>>(dd, N, xs_approx, xs_approx + nseg, xs_maps, 0, dscal + 1);
    xs_loss_map_kernel<<<g, 128, 0, s()>>>(dd, N, xs_approx + nseg, xs_maps);
    xs_loss_compose_kernel<<<1, 1024, 0, s()>>>(dd, N, xs_approx, xs_approx + nseg, xs_maps, 1, dscal + 1);
    kt::check_launch(ctx, "exact loss", 4);
    double v;
    KT_CUDA(cudaMemcpyAsync(&v, dscal + 1, 8, cudaMemcpyDeviceToHost, s()));
    KT_CUDA(cudaStreamSynchronize(s()));
    return v;
  }

  double loss_err(double L) const { return (double)(N + 80) * kU * 1.0625 * L; }

  bool same_assign(const int32_t* a, const int32_t* b) {
    KT_CUDA(cudaMemsetAsync(ull + 1, 0, 8, s()));
    count_diff_kernel<<<std::min<int64_t>(kt::ceil_div(N, 256), 1024), 256, 0, s()>>>(a, b, N, ull + 1);
    kt::check_launch(ctx, "count_diff");
    unsigned long long v;
    KT_CUDA(cudaMemcpyAsync(&v, ull + 1, 8, cudaMemcpyDeviceToHost, s()));
    KT_CUDA(cudaStreamSynchronize(s()));
    return v == 0;
  }

  // Lloyd from kmeans++ (sampling.cpp:98-153). Result left in (cent_a, asg_a, d2_a).
  double lloyd(int k, uint64_t rng_seed, int max_iters, std::vector<double>& iter_losses) {
    kmeanspp(k, rng_seed);
    double loss = assign(cent_a, k, nullptr, asg_a, d2_a, nullptr);
    iter_losses.assign(1, loss);
    return lloyd_loop(k, 0, max_iters, loss, iter_losses);
  }

  // Exact Lloyd iterations it0 .. max_iters-1 from the exact state (asg_a, d2_a).
  double lloyd_loop(int k, int it0, int max_iters, double loss, std::vector<double>& iter_losses,
                    bool* converged = nullptr) {
    if (converged) *converged = false;
    // Single-GPU iterations replay a captured CUDA graph (centroid update + assignment +
    // readback: ~20 launches): the loop is launch-bound at N = 1M. Two graphs, one per
    // parity of the a/b buffer swap.
    // no graphs on the legacy default stream (capture is illegal there) or while profiling
    const bool use_graph = !sharded && !ctx->opt_profile && capturable(s());
    cudaGraphExec_t gx[2] = {nullptr, nullptr};
    struct GraphGuard {
      cudaGraphExec_t* g;
      ~GraphGuard() {
        for (int i = 0; i < 2; ++i)
          if (g[i]) cudaGraphExecDestroy(g[i]);
      }
    } guard{gx};
    for (int it = it0; it < max_iters; ++it) {
      unsigned long long changed = 0;
      if (use_graph) {
        cudaGraphExec_t& g = gx[it & 1];
        if (!g) {
          cudaGraph_t graph;
          KT_CUDA(cudaStreamBeginCapture(s(), cudaStreamCaptureModeThreadLocal));
          CaptureGuard cg{s()};
          update_centroids(k, asg_a, d2_a, cent_b);
          enqueue_assign(cent_b, k, asg_a, asg_b, d2_b);
          cg.end(&graph);
          KT_CUDA(cudaGraphInstantiate(&g, graph, 0));
          cudaGraphDestroy(graph);
        }
        KT_CUDA(cudaGraphLaunch(g, s()));
      } else {
        update_centroids(k, asg_a, d2_a, cent_b);
        enqueue_assign(cent_b, k, asg_a, asg_b, d2_b);
      }
      const double nl = finish_assign(asg_a, &changed);
      ctx->stats[KTUNE_STAT_LLOYD_ITERS] += 1;
      if (nl > loss + 1e-9 + loss_err(loss) + loss_err(nl))
        kt::fail(KTUNE_ERR_LOGIC, "kmeans: Lloyd loss increased, which should be impossible");
      std::swap(cent_a, cent_b);
      std::swap(asg_a, asg_b);
      std::swap(d2_a, d2_b);
      loss = nl;
      iter_losses.push_back(nl);
      if (changed == 0) {
        if (converged) *converged = true;
        break;
      }
    }
    return loss;
  }

  // Certified speculative Lloyd (mode B, see assign_cert_kernel): returns false
  // (the caller reruns the exact mode A) on an uncertain point or an empty
  // cluster. On success the final centroids and d2 are recomputed exactly from
  // the last two assignments, as the reference's loop leaves them.
  bool lloyd_cert(int k, uint64_t rng_seed, int max_iters, std::vector<double>& iter_losses) {
    kmeanspp(k, rng_seed);
    double loss = assign(cent_a, k, nullptr, asg_a, d2_a, nullptr);  // exact
    iter_losses.assign(1, loss);
    const size_t words = (size_t)kt::kMaxK * (kt::kMaxKnobs + 1);
    const size_t tsmem = cert_smem_bytes(k, D, D <= 8 ? 8 : (D <= 16 ? 16 : kt::kMaxKnobs), lut_smem);  // <= screen_smem
    int cur = 0;
    KT_CUDA(cudaMemsetAsync(isum[cur], 0, sizeof(unsigned long long) * words, s()));
    cluster_sums_kernel<IdxT><<<sums_grid(), kBT, 0, s()>>>(pts, N, D, k, asg_a, isum[cur],
                                                                  isum[cur] + (size_t)kt::kMaxK * kt::kMaxKnobs);
    kt::check_launch(ctx, "cluster_sums");
    // Iterations run in batches of kCertBatch replayed CUDA graphs (one per parity of the
    // a/b swap) with ONE readback per batch. Iterations past convergence are idempotent
    // (same assignment, same sums), so overshooting inside a batch changes no state.
    constexpr int kCertBatch = 4;
    unsigned long long* cs = isum[cur];  // sums of asg_a; updated in place to those of asg_b
    cudaGraphExec_t gx[2] = {nullptr, nullptr};
    struct GraphGuard {
      cudaGraphExec_t* g;
      ~GraphGuard() {
        for (int i = 0; i < 2; ++i)
          if (g[i]) cudaGraphExecDestroy(g[i]);
      }
    } guard{gx};
    // sharded: this rank's chunks only; the moved-point deltas of the integer sums, the
    // changed/uncertain counters and the loss estimate are all-reduced (O(k D) words per
    // iteration), assignments stay rank-local until the exact finalisation
    const int64_t c0 = sharded ? (int64_t)rank * shard_chunks : 0;
    const int64_t nloc = sharded ? std::max<int64_t>(0, std::min<int64_t>(nchunks, c0 + shard_chunks) - c0) : nchunks;
    unsigned long long* dsum = isum[1];
    if (!sharded) KT_CUDA(cudaMemsetAsync(ull, 0, 32, s()));  // then cleared by each iteration's tail
    auto enqueue_iter = [&]() {
      if (sharded) KT_CUDA(cudaMemsetAsync(ull, 0, 32, s()));
      centroids_from_sums_kernel<<<1, 1024, 0, s()>>>(sp->params, k, cs, cs + (size_t)kt::kMaxK * kt::kMaxKnobs, cB,
                                                      dB, ull + 3, std::ldexp(1.0, (int)ctx->opt_kmeans_bound_log2));
      unsigned long long* tgt = sharded ? dsum : cs;
      if (sharded) KT_CUDA(cudaMemsetAsync(dsum, 0, sizeof(unsigned long long) * words, s()));
      if (nloc > 0)
        KT_DISPATCH_DM(D, assign_cert_kernel<IdxT, DM_><<<(unsigned)nloc, kCertBT, tsmem, s()>>>(
                              sp->params, lut_total, pts, N, cB, dB, k, asg_a, asg_b, d2_b, chunk, ull, tgt,
                              tgt + (size_t)kt::kMaxK * kt::kMaxKnobs, c0));
      kt::check_launch(ctx, "assign_cert", 2);
      if (!sharded) {
        sum_gather_kernel<<<1, 1024, 0, s()>>>(chunk, nloc, dscal, ull, seqcnt, csb + k, rb_dev, rb_slot);
        kt::check_launch(ctx, "sum_gather");
        return;
      }
      if (nloc > 0) sum_chunks_kernel<<<1, 1024, 0, s()>>>(chunk + c0, nloc, dscal);
      else KT_CUDA(cudaMemsetAsync(dscal, 0, 8, s()));
      if (sharded) {
        kt::allreduce_sum(ctx, dsum, words, false);
        add_sums_kernel<<<(int)kt::ceil_div((int64_t)words, 256), 256, 0, s()>>>(cs, dsum, (int)words);
        kt::allreduce_sum(ctx, ull, 3, false);
        kt::allreduce_sum(ctx, dscal, 1, true);
      }
      gather_readback_kernel<<<1, 1, 0, s()>>>(dscal, ull, seqcnt, csb + k, rb_dev, rb_slot);
    };
    int iters = 0;
    bool done = false;
    const bool graphs = capturable(s()) && !sharded;  // legacy stream / NCCL calls: the same work, uncaptured
    // Rescue instead of restart: the state at each batch start is certified, so an
    // uncertain point or an empty cluster inside a batch continues EXACTLY (mode A) from
    // there. Snapshot: the exact initial (assignment, d2) before the first batch, the
    // previous assignment before later ones (its exact centroids reproduce the current one).
    int32_t* snap_asg = (int32_t*)ctx->dev(kt::WS_CERT_SNAP, (sizeof(int32_t) + sizeof(double)) * N);
    double* snap_d2 = reinterpret_cast<double*>(snap_asg + N);
    // A rescue runs EXACT iterations from the batch start: one batch's worth, after which the
    // integer sums are rebuilt from the exact assignment and certified batches resume (large
    // lattice sets meet a near tie within the centroid bound now and then, not every
    // iteration); from the third rescue of a run on, exactly to the end.
    int rescues = 0;
    constexpr int kMaxRescues = 3;  // caps 3, 5, 8 measured alike on C3 (<= 3 rescues per run)
    auto rescue = [&](int t, int upto, double at_loss, bool* finished) {
      ctx->stats[KTUNE_STAT_KMEANS_ABORTS] += 1;
      ++rescues;
      if (t == 0) {  // back to the exact initial assignment
        KT_CUDA(cudaMemcpyAsync(asg_a, snap_asg, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s()));
        KT_CUDA(cudaMemcpyAsync(d2_a, snap_d2, sizeof(double) * N, cudaMemcpyDeviceToDevice, s()));
      } else {  // exact centroids of the previous assignment (certified: no empty cluster), exact assign
        KT_CUDA(cudaMemcpyAsync(asg_b, snap_asg, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s()));
        if (sharded) {  // certified iterations keep assignments rank-local: every rank needs all of them
          const int64_t S = shard_chunks * kChunk;
          kt::allgather(ctx, asg_b + rank * S, asg_b, sizeof(int32_t) * S);
        }
        update_centroids(k, asg_b, d2_b, cent_a);
        assign(cent_a, k, nullptr, asg_a, d2_a, nullptr);
      }
      const int limit = rescues >= kMaxRescues ? max_iters : std::min(max_iters, t + upto);
      bool conv = false;
      const size_t n0 = iter_losses.size();
      const double l = lloyd_loop(k, t, limit, at_loss, iter_losses, &conv);
      const int ran = (int)(iter_losses.size() - n0);
      *finished = conv || t + ran >= max_iters;
      return std::make_pair(t + ran, l);
    };
    while (iters < max_iters && !done) {
      const int it0 = iters;
      const int nb = std::min(kCertBatch, max_iters - it0);
      if (iters == 0) {
        KT_CUDA(cudaMemcpyAsync(snap_asg, asg_a, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s()));
        KT_CUDA(cudaMemcpyAsync(snap_d2, d2_a, sizeof(double) * N, cudaMemcpyDeviceToDevice, s()));
      } else {
        KT_CUDA(cudaMemcpyAsync(snap_asg, asg_b, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s()));
      }
      const int t_batch = iters;
      const double loss_batch = loss;
      const size_t nl_batch = iter_losses.size();
      KT_CUDA(cudaMemsetAsync(rb_slot, 0, sizeof(int), s()));
      int32_t* sa = asg_a;  // the device-side view of the swaps inside this batch
      int32_t* sb = asg_b;
      double* da = d2_a;
      double* db = d2_b;
      for (int j = 0; j < nb; ++j) {
        if (!graphs) {
          enqueue_iter();
        } else {
          cudaGraphExec_t& g = gx[(it0 + j) & 1];
          if (!g) {
            cudaGraph_t graph;
            KT_CUDA(cudaStreamBeginCapture(s(), cudaStreamCaptureModeThreadLocal));
            CaptureGuard cg{s()};
            enqueue_iter();
            cg.end(&graph);
            KT_CUDA(cudaGraphInstantiate(&g, graph, 0));
            cudaGraphDestroy(graph);
          }
          KT_CUDA(cudaGraphLaunch(g, s()));
        }
        std::swap(asg_a, asg_b);
        std::swap(d2_a, d2_b);
      }
      asg_a = sa;
      asg_b = sb;
      d2_a = da;
      d2_b = db;
      KT_CUDA(cudaMemcpyAsync(rb_host, rb_dev, sizeof(IterReadback) * nb, cudaMemcpyDeviceToHost, s()));
      KT_CUDA(cudaStreamSynchronize(s()));
      for (int j = 0; j < nb; ++j) {
        const IterReadback h = rb_host[j];
        if (h.empty || h.unc) {  // speculation off: continue exactly from the batch start
          asg_a = sa;
          asg_b = sb;
          d2_a = da;
          d2_b = db;
          iter_losses.resize(nl_batch);
          bool finished = false;
          const auto [t_next, l_next] = rescue(t_batch, kCertBatch, loss_batch, &finished);
          if (finished) return true;  // exact to the end (the state lloyd_loop leaves)
          // resume certified batches from the exact state: integer sums of asg_a, snapshot of
          // asg_b (the previous assignment) at the next batch start
          KT_CUDA(cudaMemsetAsync(isum[cur], 0, sizeof(unsigned long long) * words, s()));
          cluster_sums_kernel<IdxT><<<sums_grid(), kBT, 0, s()>>>(pts, N, D, k, asg_a, isum[cur],
                                                                        isum[cur] + (size_t)kt::kMaxK * kt::kMaxKnobs);
          kt::check_launch(ctx, "cluster_sums");
          if (!sharded) KT_CUDA(cudaMemsetAsync(ull, 0, 32, s()));
          iters = t_next;
          loss = l_next;
          break;
        }
        ctx->stats[KTUNE_STAT_LLOYD_ITERS] += 1;
        if (h.loss > loss * (1.0 + 1e-9) + 1e-9 + loss_err(loss) + loss_err(h.loss))
          kt::fail(KTUNE_ERR_LOGIC, "kmeans: Lloyd loss increased, which should be impossible");
        std::swap(asg_a, asg_b);
        std::swap(d2_a, d2_b);
        loss = h.loss;
        iter_losses.push_back(h.loss);
        ++iters;
        if (h.changed == 0) {
          done = true;
          break;
        }
      }
    }
    if (iters > 0) {
      if (sharded) {  // every rank needs both full assignments for the exact finalisation
        const int64_t S = shard_chunks * kChunk;
        kt::allgather(ctx, asg_a + rank * S, asg_a, sizeof(int32_t) * S);
        kt::allgather(ctx, asg_b + rank * S, asg_b, sizeof(int32_t) * S);
      }
      // exact final state: centroids from the previous assignment (asg_b), then the exact
      // d2 against them; the certified assignment must be reproduced exactly
      update_centroids(k, asg_b, d2_b, cent_b);
      assign(cent_b, k, nullptr, asg_b, d2_b, nullptr);
      if (!same_assign(asg_a, asg_b)) return false;
      std::swap(cent_a, cent_b);
      std::swap(asg_a, asg_b);
      std::swap(d2_a, d2_b);
    }
    return true;
  }

  struct Result {
    double loss, loss_exact;
    std::vector<double> iter_losses;
  };

  // kmeans_run (sampling.cpp:157-175): best of restarts into best_* buffers.
  // Restart losses are the reference's exact sequential sums, so the strict
  // "<" (earliest restart wins ties) is decided exactly.
  Result run(int k, uint64_t seed, int max_iters, int restarts) {
    Result best{0.0, NAN, {}};
    bool have = false;
    for (int r = 0; r < std::max(1, restarts); ++r) {
      std::vector<double> il;
      const uint64_t rs = kt::seed_combine(seed, (uint64_t)r);
      const bool spec = !ctx->opt_force_exact && ctx->opt_kmeans_mode != 1 && ctx->opt_kmeans_mode != 3;
      if (!spec || !lloyd_cert(k, rs, max_iters, il)) {
        if (spec) ctx->stats[KTUNE_STAT_KMEANS_ABORTS] += 1;
        lloyd(k, rs, max_iters, il);
      }
      int32_t nfb = 0;  // kmeans++ picks decided by the exact replay (this restart)
      KT_CUDA(cudaMemcpyAsync(&nfb, &kst->fallbacks, sizeof(nfb), cudaMemcpyDeviceToHost, s()));
      KT_CUDA(cudaStreamSynchronize(s()));
      ctx->stats[KTUNE_STAT_KPP_FALLBACKS] += nfb;
      const double Lx = exact_loss(d2_a);
      il.back() = Lx;
      if (!have || Lx < best.loss_exact) {
        have = true;
        best.loss = Lx;
        best.loss_exact = Lx;
        best.iter_losses = il;
        KT_CUDA(cudaMemcpyAsync(best_asg, asg_a, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s()));
        KT_CUDA(cudaMemcpyAsync(best_d2, d2_a, sizeof(double) * N, cudaMemcpyDeviceToDevice, s()));
        KT_CUDA(cudaMemcpyAsync(best_cent, cent_a, sizeof(double) * k * D, cudaMemcpyDeviceToDevice, s()));
      }
    }
    return best;
  }
};

template <class IdxT>
void snap_device(ktune_ctx* ctx, const ktune_space* sp, const double* d_cent, int k,
                 const IdxT* d_cand, const uint64_t* d_ids, int64_t N, int32_t* d_out) {
  int32_t* need = (int32_t*)ctx->dev(kt::WS_OUT4, sizeof(int32_t) * kt::kMaxK);
  snap_round_kernel<<<1, 64, 0, ctx->stream>>>(sp->params, d_cent, k, d_out, need);
  kt::check_launch(ctx, "snap_round");
  if (N <= 0) return;
  const int nblk = (int)std::min<int64_t>(kt::ceil_div(N, kBT), 256);
  unsigned long long* part = (unsigned long long*)ctx->dev(kt::WS_OUT3, sizeof(unsigned long long) * 4 * nblk * k);
  dim3 grid(nblk, k);
  snap_fallback_kernel<IdxT><<<grid, kBT, sizeof(double) * sp->lut_total, ctx->stream>>>(
      sp->params, sp->lut_total, d_cent, need, d_cand, d_ids, N, part);
  snap_reduce_kernel<IdxT><<<k, 32, 0, ctx->stream>>>(sp->params, need, part, nblk, d_cand, d_ids, N, d_out);
  kt::check_launch(ctx, "snap", 2);
}

void check_lut(const ktune_space* sp) {
  if ((size_t)sp->lut_total * 8 + kt::kMaxK * kt::kMaxKnobs * 8 > 200 * 1024)
    kt::fail(KTUNE_ERR_CONFIG, "k-means: feature table too large for shared memory");
}

template <class IdxT>
void kmeans_impl(ktune_ctx* ctx, const ktune_space* space, const void* idx, int64_t N, int k,
                 uint64_t seed, int max_iters, int restarts, ktune_kmeans_out* out, bool dev) {
  const int D = space->D;
  const IdxT* d_pts = (const IdxT*)kt::stage_in(ctx, kt::WS_IN0, idx, sizeof(IdxT) * N * D, dev);
  KMeans<IdxT> km;
  km.setup(ctx, space, d_pts, N);
  auto res = km.run(k, seed, max_iters, restarts);
  const double loss = std::isnan(res.loss_exact) ? res.loss : res.loss_exact;
  if (dev) {
    if (out->centroids) KT_CUDA(cudaMemcpyAsync(out->centroids, km.best_cent, sizeof(double) * k * D, cudaMemcpyDeviceToDevice, ctx->stream));
    if (out->assignments) KT_CUDA(cudaMemcpyAsync(out->assignments, km.best_asg, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    if (out->l2_loss) KT_CUDA(cudaMemcpyAsync(out->l2_loss, &loss, 8, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    if (out->centroids) KT_CUDA(cudaMemcpyAsync(out->centroids, km.best_cent, sizeof(double) * k * D, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->assignments) KT_CUDA(cudaMemcpyAsync(out->assignments, km.best_asg, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->l2_loss) *out->l2_loss = loss;
  }
  if (out->iteration_losses) {
    for (size_t i = 0; i < res.iter_losses.size(); ++i) out->iteration_losses[i] = res.iter_losses[i];
    if (!res.iter_losses.empty() && !std::isnan(res.loss_exact))
      out->iteration_losses[res.iter_losses.size() - 1] = res.loss_exact;
  }
  if (out->num_losses) *out->num_losses = (int32_t)res.iter_losses.size();
  KT_CUDA(cudaStreamSynchronize(ctx->stream));
}

template <class IdxT>
void sweep_impl(ktune_ctx* ctx, const ktune_space* space, const void* idx, const uint64_t* ids,
                int64_t N, const ktune_sampling_params* p, uint64_t rng_seed, ktune_sweep_out* out,
                bool dev) {
  const int D = space->D;
  const IdxT* d_pts = (const IdxT*)kt::stage_in(ctx, kt::WS_IN0, idx, sizeof(IdxT) * N * D, dev);
  const uint64_t* d_ids = (const uint64_t*)kt::stage_in(ctx, kt::WS_IN1, ids, sizeof(uint64_t) * N, dev);
  KMeans<IdxT> km;
  km.setup(ctx, space, d_pts, N);
  const int k_lo = (int)std::min<int64_t>(p->k_min, N);
  const int k_hi = (int)std::min<int64_t>(p->k_max_exclusive - 1, N);
  double prev = INFINITY;
  bool have_prev = false;
  int chosen = k_lo;
  double chosen_loss = 0.0;
  std::vector<double> klosses;
  double* d_chosen_cent = (double*)ctx->dev(kt::WS_OUT2, sizeof(double) * kt::kMaxK * D);
  for (int k = k_lo; k <= k_hi; ++k) {
    auto res = km.run(k, kt::seed_combine(rng_seed, (uint64_t)k), p->max_iters, p->restarts);
    chosen = k;
    chosen_loss = std::isnan(res.loss_exact) ? res.loss : res.loss_exact;
    KT_CUDA(cudaMemcpyAsync(d_chosen_cent, km.best_cent, sizeof(double) * k * D, cudaMemcpyDeviceToDevice, ctx->stream));
    // break test: threshold * L_k >= L_{k-1} on exact losses (sampling.cpp:444)
    const bool brk = have_prev && p->threshold * res.loss_exact >= prev;
    klosses.push_back(chosen_loss);
    if (brk) break;
    prev = res.loss_exact;
    have_prev = true;
  }
  // snap the chosen centroids (sampling.cpp:448-452)
  int32_t* d_snap = (int32_t*)ctx->dev(kt::WS_OUT1, sizeof(int32_t) * kt::kMaxK * D);
  snap_device<IdxT>(ctx, space, d_chosen_cent, chosen, d_pts, d_ids, N, d_snap);
  const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (out->centroids) KT_CUDA(cudaMemcpyAsync(out->centroids, d_chosen_cent, sizeof(double) * chosen * D, kind, ctx->stream));
  if (out->assignments) KT_CUDA(cudaMemcpyAsync(out->assignments, km.best_asg, sizeof(int32_t) * N, kind, ctx->stream));
  if (out->snapped) KT_CUDA(cudaMemcpyAsync(out->snapped, d_snap, sizeof(int32_t) * chosen * D, kind, ctx->stream));
  KT_CUDA(cudaStreamSynchronize(ctx->stream));
  *out->k = chosen;
  if (out->l2_loss) *out->l2_loss = chosen_loss;
  if (out->k_losses)
    for (size_t i = 0; i < klosses.size(); ++i) out->k_losses[i] = klosses[i];
  if (out->num_k) *out->num_k = (int32_t)klosses.size();
}

}  // namespace

extern "C" {

int ktune_kmeans_run(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                     int64_t N, int k, uint64_t seed, int max_iters, int restarts,
                     ktune_kmeans_out* out, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_kmeans_run");
    if (N == 0) kt::fail(KTUNE_ERR_CONFIG, "kmeans: empty point set");
    if (k < 1 || k > N)
      kt::fail(KTUNE_ERR_CONFIG, "kmeans: k=" + std::to_string(k) + " out of range for " + std::to_string(N) + " points");
    if (k > kt::kMaxK) kt::fail(KTUNE_ERR_CONFIG, "kmeans: k > 64 unsupported on the device path");
    if (idx_bytes != 1 && idx_bytes != 2) kt::fail(KTUNE_ERR_CONFIG, "idx_bytes must be 1 or 2");
    if (N > INT32_MAX) kt::fail(KTUNE_ERR_CONFIG, "kmeans: at most 2^31-1 points");
    if (max_iters < 0) max_iters = 0;
    check_lut(space);
    cudaSetDevice(ctx->device);
    if (idx_bytes == 1)
      kmeans_impl<uint8_t>(ctx, space, idx, N, k, seed, max_iters, restarts, out, flags & KTUNE_F_DEVICE);
    else
      kmeans_impl<uint16_t>(ctx, space, idx, N, k, seed, max_iters, restarts, out, flags & KTUNE_F_DEVICE);
  });
}

int ktune_adaptive_sweep(ktune_ctx* ctx, const ktune_space* space, const void* idx, int idx_bytes,
                         const uint64_t* ids, int64_t N, const ktune_sampling_params* p,
                         uint64_t rng_seed, ktune_sweep_out* out, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_adaptive_sweep");
    if (N == 0) kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: empty candidate set");
    if (p->k_min >= p->k_max_exclusive || p->k_min < 1)
      kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: need 1 <= k_min < k_max_exclusive");
    if (p->threshold <= 1.0) kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: threshold must exceed 1");
    if (p->k_max_exclusive - 1 > kt::kMaxK) kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: k > 64 unsupported on the device path");
    if (idx_bytes != 1 && idx_bytes != 2) kt::fail(KTUNE_ERR_CONFIG, "idx_bytes must be 1 or 2");
    if (N > INT32_MAX) kt::fail(KTUNE_ERR_CONFIG, "adaptive_sample: at most 2^31-1 candidates");
    check_lut(space);
    cudaSetDevice(ctx->device);
    if (idx_bytes == 1)
      sweep_impl<uint8_t>(ctx, space, idx, ids, N, p, rng_seed, out, flags & KTUNE_F_DEVICE);
    else
      sweep_impl<uint16_t>(ctx, space, idx, ids, N, p, rng_seed, out, flags & KTUNE_F_DEVICE);
  });
}

int ktune_snap(ktune_ctx* ctx, const ktune_space* space, const double* centroids, int k,
               const void* cand_idx, int idx_bytes, const uint64_t* cand_ids, int64_t N,
               int32_t* out_idx, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_snap");
    if (k < 0 || k > kt::kMaxK) kt::fail(KTUNE_ERR_CONFIG, "snap: 0 <= k <= 64");
    if (k == 0) return;
    if (idx_bytes != 1 && idx_bytes != 2) kt::fail(KTUNE_ERR_CONFIG, "idx_bytes must be 1 or 2");
    const bool dev = flags & KTUNE_F_DEVICE;
    const int D = space->D;
    const double* d_c = (const double*)kt::stage_in(ctx, kt::WS_IN2, centroids, sizeof(double) * k * D, dev);
    const void* d_cand = kt::stage_in(ctx, kt::WS_IN0, cand_idx, (size_t)idx_bytes * N * D, dev);
    const uint64_t* d_ids = (const uint64_t*)kt::stage_in(ctx, kt::WS_IN1, cand_ids, sizeof(uint64_t) * N, dev);
    int32_t* d_out = (int32_t*)kt::out_buf(ctx, kt::WS_OUT0, out_idx, sizeof(int32_t) * k * D, dev);
    if (idx_bytes == 1)
      snap_device<uint8_t>(ctx, space, d_c, k, (const uint8_t*)d_cand, d_ids, N, d_out);
    else
      snap_device<uint16_t>(ctx, space, d_c, k, (const uint16_t*)d_cand, d_ids, N, d_out);
    kt::stage_out(ctx, out_idx, d_out, sizeof(int32_t) * k * D, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
