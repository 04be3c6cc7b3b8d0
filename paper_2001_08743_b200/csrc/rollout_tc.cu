// K2 on the 5th-generation tensor cores: the batched Adaptive-Exploration
// rollout (run_episodes; ActorCritic::forward,
// actor_critic.hpp:18-64) with CERTIFIED sampling.
//
// Per config-step the actor-critic MLP runs as three tcgen05.mma GEMMs with
// fp32 accumulators in TMEM:
//   L1  h0  = tanh(W0 x + b0)        A = [idx | idx] (fp16, exact integers)
//                                    B = [hi | lo] of W0/(card-1) * 2^e1
//   L2  [hp|hv] = tanh(W h0 + b)     A = h0 * 2^14 split hi/lo (fp16),
//                                    B = [Wp1;Wv1] * 2^e2 split hi/lo,
//                                    3 products hi*hi + hi*lo + lo*hi
//   L3  logits = Wp2 hp + bp2        same split, N = roundup16(3n)
// (fp16 pairs carry 22 significant bits; products are exact in fp32), so the
// logits agree with the exact fp64 forward to ~1e-6. The value head
// (wv2 . hv + bv2) is an fp32 dot product in the L2 epilogue.
//
// Sampling is CERTIFIED: the fast probabilities p0 = P(dec), c1 = P(dec) +
// P(stay) decide the action only when the draw u is farther than delta from
// both (|u - p0| > delta and |u - c1| > delta); otherwise the warp recomputes
// that row's forward EXACTLY in fp64 (the same operations as the exact kernel
// and the oracle: DFMA chains in ascending input order, the portable tanh/
// exp/log of DESIGN.md §5.3) and decides with the exact probabilities.
// Knob indices, actions and therefore every visited configuration are
// bit-identical to the exact path; log-probabilities and values are fp32-
// accurate (north star: 1e-5 relative).
//
// Layout: one persistent CTA per SM (384 threads = 3 slots x 4 warps). A slot
// is a tile of up to 128 episodes (one TMEM lane and one thread per episode,
// 128 TMEM columns per slot); its configurations live in the owning threads'
// registers for the whole episode. Weights are staged once per CTA into shared
// memory as fp16 hi/lo (UMMA K-major, no swizzle); each slot has a 32 KB
// operand buffer reused by every layer (L2 runs in two K halves). Slots run
// independently (named barrier + mbarrier per slot), so one slot's MMAs
// overlap the other slots' SIMT epilogues.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "device.cuh"
#include "internal.cuh"
#include "tcgen05.cuh"

namespace {

constexpr int kH = 128, kG = 64;  // hidden sizes of the tensor-core path
constexpr int kSlots = 3;  // 3 x 128 episodes per SM: 384 threads, up to 168 registers each
constexpr int kThr = kSlots * 128;
constexpr int kMaxWarps = kSlots * 4;
constexpr int kTcMaxN = 21;       // 3n <= 64: the L3 accumulator stays clear of hv's TMEM columns
constexpr int kMaxTcTasks = 12;
constexpr float kActScale = 16384.f;  // 2^14 activation scale inside the fp16 operands

struct TcTask {
  int32_t card[kt::kMaxKnobs];
  int32_t foff[kt::kMaxKnobs];  // feature LUT offsets: x_d = flut[foff[d] + idx_d] (design_space.cpp:195-197)
  const double* flut;
  const double* params;  // fp64 flat layout (actor_critic.hpp:52-53)
  int32_t n, T;
  int64_t E, episode_offset;
  uint64_t seed;
  const uint16_t* init_idx;
  uint16_t* idx;
  int8_t* actions;
  double* logp;
  double* value;
  float* logp32;
  float* value32;
  int64_t sE, sT, aE, aT;          // trajectory layout (rows), see RolloutWork
  int32_t cta_base, ctas, warps;  // CTAs [cta_base, cta_base + ctas) share warps = ceil(E/32)
  int32_t e1, e2, e3;             // power-of-two weight scales of L1, L2, L3
  // fused cost-model scoring (K1 in the epilogue; gnode == nullptr: scored by a separate K1 launch)
  const uint32_t* gnode;  // complete trees: (feature << 24) | t1 (ktune_gbt::d_inode_idx)
  const double* gleaf;
  int32_t ntrees, depth;
  double gbase, glr;
  double* score;  // E x (T+1)
  // compact outputs written by the rollout itself (host-buffer calls; NULL: not requested)
  uint8_t* idx8;   // rows as uint8 knob indices (idx layout, n bytes per row)
  uint32_t* ids;   // rows as configuration ids id_of (score layout)
  uint8_t* act2;   // steps as 2-bit direction codes, ceil(n/4) bytes per step (actions layout)
};

struct TcLaunch {
  int32_t num_tasks;
  int32_t t_begin, t_end;  // steps [t_begin, t_end) of a T-step episode (segmented launches)
  int32_t check;
  float delta;
  unsigned long long* counters;  // [fallbacks, checked, mismatches, max err (float bits)]
  // streamed host-buffer rollouts: the episode's steps form nseg segments, segment s = steps
  // [ceil(s T / nseg), ceil((s+1) T / nseg)); every slot adds 1 to progress[s] when its rows
  // have finished segment s, so the copy stream can wait for progress[s] to reach the slot
  // count (cuStreamWaitValue32) while the kernel runs on
  unsigned int* progress;
  int32_t nseg;
  TcTask task[kMaxTcTasks];
};

// Shared-memory carve-up (bytes).
constexpr uint32_t kOffB2 = 0;             // [128 x 256] fp16: [Wp1;Wv1] hi (K 0..127) | lo
constexpr uint32_t kOffA = 65536;          // kSlots x [128 x 128] fp16 operand buffers
constexpr uint32_t kABytes = 32768;
constexpr uint32_t kOffB1 = kOffA + kSlots * kABytes;
__host__ __device__ inline int nk_of(int n) { return (n + 7) & ~7; }
__host__ __device__ inline int n3_of(int n) { return (3 * n + 15) & ~15; }
__host__ __device__ inline uint32_t off_b3(int n) { return kOffB1 + 128u * 2 * nk_of(n) * 2; }
__host__ __device__ inline uint32_t off_f32(int n) { return off_b3(n) + (uint32_t)n3_of(n) * 256; }
constexpr int kNF32 = 128 + 64 + 64 + 64 + 64 + 4;  // b0 bp1 bv1 wv2 bp2 bv2
// D <= 8: the step's counter-RNG draws are parked in shared memory (two float4 per thread,
// thread-contiguous) between the L2 MMA window that computes them and the L3 epilogue.
__host__ __device__ inline uint32_t off_draw(int n) { return (off_f32(n) + kNF32 * 4 + 15) & ~15u; }
__host__ __device__ inline uint32_t draw_bytes(int n) { return n <= 8 ? 2u * 16u * kThr : 0u; }
__host__ __device__ inline uint32_t off_gbt(int n) { return off_draw(n) + draw_bytes(n); }
// + fused GBT: leaves f64 [ntrees][2^depth], node words u32 [ntrees][2^depth - 1], then the
// thread-private knob columns int32 [n][kThr] the tree walks index (conflict-free).
__host__ __device__ inline uint32_t gbt_leaf_bytes(int ntrees, int depth) { return (uint32_t)ntrees * (8u << depth); }
__host__ __device__ inline uint32_t gbt_node_bytes(int ntrees, int depth) {
  return ((uint32_t)ntrees * 4u * ((1u << depth) - 1) + 15) & ~15u;
}
__host__ __device__ inline uint32_t tc_smem_bytes(int n, int ntrees, int depth) {
  const uint32_t g = ntrees > 0 ? gbt_leaf_bytes(ntrees, depth) + gbt_node_bytes(ntrees, depth) + (uint32_t)n * kThr * 4 : 0;
  return off_gbt(n) + g + 1024;
}

// Partial GBT walk over trees [t0, t1): s += leaf_t(x) in tree order. The full
// score base + lr * s is bit-exact with cost_model.cpp:179-187 and K1.
// col: this thread's knob column (col[d * kThr]); node word = (byte offset of column d) << 16 | t1.
__device__ __forceinline__ double gbt_walk(double s, const uint32_t* __restrict__ s_node,
                                           const double* __restrict__ s_leaf, const unsigned char* col, int t0,
                                           int t1, int depth) {
  const int NI = (1 << depth) - 1, NL = 1 << depth;
#pragma unroll 2
  for (int tr = t0; tr < t1; ++tr) {
    const uint32_t* tn = s_node + tr * NI;
    int nd = 0;
    for (int l = 0; l < depth; ++l) {
      const uint32_t w = tn[nd];
      const int v = *reinterpret_cast<const int*>(col + (w >> 16));
      nd = 2 * nd + 1 + (v >= (int)(w & 0xFFFFu) ? 1 : 0);
    }
    s = kt::dadd(s, s_leaf[tr * NL + (nd - NI)]);
  }
  return s;
}

// ---------------------------------------------------------------- fast math
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// S * tanh(x) from y = -2 log2(e) x (the scale is folded into the
// pre-activation FMA): e = exp(-2x), S tanh(x) = 2S/(1 + e) - S. A PAIR of
// units shares one reciprocal: with d = 1 + e, 1/d_a = d_b / (d_a d_b), so a
// pair costs two ex2 and one rcp on the SFU (3 MUFU instead of 4) and the rest
// runs as packed f32x2 FMA-pipe instructions. y is clamped at 63 so that
// d_a d_b <= 2^126 stays finite (tanh(-21.8) = -1 to 2^-62). Absolute error
// <= ~5e-7 * S (ex2 2^-22.7, rcp 2^-23.3, three roundings).
constexpr float kK2L = -2.8853900817779268f;  // -2 log2(e)
__device__ __forceinline__ float2 act2(float2 y, float S) {
  const float ea = ex2f(fminf(y.x, 63.f)), eb = ex2f(fminf(y.y, 63.f));
  const float2 d = __fadd2_rn(make_float2(ea, eb), make_float2(1.f, 1.f));
  const float R = rcpf(d.x * d.y);
  const float2 r = __fmul2_rn(make_float2(d.y, d.x), make_float2(R, R));
  return __ffma2_rn(r, make_float2(2.f * S, 2.f * S), make_float2(-S, -S));
}
// Pre-activation pair: acc * sc + b (b from shared memory, 8-byte aligned).
__device__ __forceinline__ float2 pre2(uint32_t a0, uint32_t a1, float sc, const float* b) {
  return __ffma2_rn(make_float2(__uint_as_float(a0), __uint_as_float(a1)), make_float2(sc, sc),
                    *reinterpret_cast<const float2*>(b));
}

__device__ __forceinline__ uint32_t h2bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// fp16 hi/lo split of a pair: hi = RN_f16(v), lo = RN_f16(v - hi) (v - hi is exact).
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 f = __half22float2(h);
  hi = h2bits(h);
  lo = h2bits(__float22half2_rn(__fadd2_rn(make_float2(a, b), make_float2(-f.x, -f.y))));
}

// Eight consecutive K values of row r (already scaled): hi at column k0, lo
// at column 64 + k0 of a [128 x 128] K-major operand buffer.
__device__ __forceinline__ void store8_split(unsigned char* Ab, int r, int k0, const float* v) {
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) split2(v[2 * p], v[2 * p + 1], hi[p], lo[p]);
  *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, k0, 128)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, 64 + k0, 128)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// 16 units (TMEM columns already loaded into v) -> S*tanh -> fp16 hi/lo -> operand columns c0..c0+15.
__device__ __forceinline__ void act_store16(unsigned char* Ab, int r, int c0, const uint32_t* v, float sc,
                                            const float* bias) {
  float hv[16];
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 h = act2(pre2(v[j], v[j + 1], sc, bias + j), kActScale);
    hv[j] = h.x;
    hv[j + 1] = h.y;
  }
  store8_split(Ab, r, c0, hv);
  store8_split(Ab, r, c0 + 8, hv + 8);
}
__device__ __forceinline__ void sync_slot(int slot, int nthreads = 128) {
  kt::tc::fence_proxy_async();
  kt::tc::fence_before();
  kt::tc::named_bar(1 + slot, nthreads);
}

// Three-product split GEMM over 4 K chunks of 16: hi*hi + hi*lo + lo*hi.
// Descriptors are precomputed: +16 in the address field = +256 bytes.
// A: hi chunk kb at +kb*16, lo at +64 (1024 B); B: chunk c at +c*16, lo at +blo16.
__device__ __forceinline__ void mma_split4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t blo16, int c0,
                                           uint32_t idesc, bool accumulate) {
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    const uint64_t ahi = adesc + 16 * kb, alo = adesc + 64 + 16 * kb;
    const uint64_t bhi = bdesc + 16 * (c0 + kb), bl = bdesc + blo16 + 16 * (c0 + kb);
    kt::tc::mma_f16(d, ahi, bhi, idesc, (accumulate || kb > 0) ? 1u : 0u);
    kt::tc::mma_f16(d, ahi, bl, idesc, 1u);
    kt::tc::mma_f16(d, alo, bhi, idesc, 1u);
  }
}

// Packed configuration (two uint16 knob indices per register).
template <int NMAX>
struct Cfg {
  uint32_t w[NMAX / 2];
  __device__ __forceinline__ int get(int d) const { return (int)((w[d >> 1] >> ((d & 1) * 16)) & 0xFFFFu); }
  __device__ __forceinline__ void set(int d, int v) {
    const int sh = (d & 1) * 16;
    w[d >> 1] = (w[d >> 1] & ~(0xFFFFu << sh)) | ((uint32_t)v << sh);
  }
};

// Configuration id (design_space.cpp:158-167: mixed radix, last knob fastest); knobs >= n
// have cardinality 1 and index 0, so the Horner chain runs branch-free over NMAX.
template <int NMAX>
__device__ __forceinline__ uint32_t cfg_id(const Cfg<NMAX>& c, const int* card) {
  uint32_t id = 0;
#pragma unroll
  for (int d = 0; d < NMAX; ++d) id = id * (uint32_t)card[d] + (uint32_t)c.get(d);
  return id;
}

template <int NMAX>
__device__ __forceinline__ void store_row_u8(uint8_t* dst, const Cfg<NMAX>& c, int n) {
  if ((n & 7) == 0) {
#pragma unroll
    for (int q = 0; q < NMAX / 8; ++q)
      if (8 * q < n) {
        const uint32_t lo = __byte_perm(c.w[4 * q], c.w[4 * q + 1], 0x6420);
        const uint32_t hi = __byte_perm(c.w[4 * q + 2], c.w[4 * q + 3], 0x6420);
        reinterpret_cast<uint2*>(dst)[q] = make_uint2(lo, hi);
      }
  } else {
#pragma unroll
    for (int d = 0; d < NMAX; ++d)
      if (d < n) dst[d] = (uint8_t)c.get(d);
  }
}

// 2-bit direction codes (direction + 1) of one step: the low 2n bits of the decision word.
__device__ __forceinline__ void store_act2(uint8_t* dst, uint64_t acts, int n) {
  if (n == 8) {
    *reinterpret_cast<uint16_t*>(dst) = (uint16_t)acts;
  } else {
    for (int b = 0; 4 * b < n; ++b) {
      const int k = min(4, n - 4 * b);
      dst[b] = (uint8_t)((acts >> (8 * b)) & ((1u << (2 * k)) - 1u));
    }
  }
}

template <int NMAX>
__device__ __forceinline__ void store_row_idx(uint16_t* dst, const Cfg<NMAX>& c, int n) {
  if ((n & 7) == 0) {
#pragma unroll
    for (int q = 0; q < NMAX / 8; ++q)
      if (8 * q < n)
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(c.w[4 * q], c.w[4 * q + 1], c.w[4 * q + 2], c.w[4 * q + 3]);
  } else if ((n & 1) == 0) {
#pragma unroll
    for (int q = 0; q < NMAX / 2; ++q)
      if (2 * q < n) reinterpret_cast<uint32_t*>(dst)[q] = c.w[q];
  } else {
#pragma unroll
    for (int d = 0; d < NMAX; ++d)
      if (d < n) dst[d] = (uint16_t)c.get(d);
  }
}

// Exact fp64 re-decision of row `L`'s flagged knobs by the whole warp (same
// operations and order as the exact kernel's forward_tile and the oracle).
// cfg is each lane's own configuration (row L's is shuffled from lane L); fastp[2d],
// fastp[2d+1] are lane L's fast p0 and c1 (or the planted draw) of knob d.
// Returns, in lane L, the exact actions (2 bits per knob) and the sum of the
// exact log-probabilities of the flagged knobs; check-mode statistics too.
struct Redecided {
  uint64_t acts;
  float lp;
};

template <int NMAX>
__device__ __noinline__ Redecided exact_redecide(const TcTask& tk, int t, int L, uint32_t fm, Cfg<NMAX> cfg,
                                                 const int* scard, double* sh0, double* shp, double* slg,
                                                 int64_t ge_L, uint64_t acts, const float* fastp, uint32_t fast_cert,
                                                 unsigned long long* stats, int check) {
  // Latency-bound by construction (a few dependent fp64 chains per lane), so every stage
  // issues its global weight loads in batches ahead of the chains that consume them, and
  // the independent chains of a lane are interleaved.
  const int lane = threadIdx.x & 31;
  const int n = tk.n;
  const double* __restrict__ P = tk.params;
  const int ob0 = kH * n, owp1 = ob0 + kH, obp1 = owp1 + kG * kH, owp2 = obp1 + kG, obp2 = owp2 + 3 * n * kG;
  double x[NMAX];
#pragma unroll
  for (int d = 0; d < NMAX; ++d) {
    const int c = (int)((__shfl_sync(0xffffffffu, cfg.w[d >> 1], L) >> ((d & 1) * 16)) & 0xFFFFu);
    x[d] = d < n ? tk.flut[tk.foff[d] + c] : 0.0;  // = c / (card - 1) (0 if card = 1), host-divided
  }
  // h0 = tanh(W0 x + b0): W0 column-major (h x n); units lane + 32m, four chains interleaved
  {
    double acc[kH / 32], bias[kH / 32];
#pragma unroll
    for (int m = 0; m < kH / 32; ++m) {
      acc[m] = 0.0;
      bias[m] = P[ob0 + lane + 32 * m];
    }
#pragma unroll
    for (int i = 0; i < NMAX; ++i)
      if (i < n) {
        double w[kH / 32];
#pragma unroll
        for (int m = 0; m < kH / 32; ++m) w[m] = P[i * kH + lane + 32 * m];
#pragma unroll
        for (int m = 0; m < kH / 32; ++m) acc[m] = __fma_rn(w[m], x[i], acc[m]);
      }
#pragma unroll
    for (int m = 0; m < kH / 32; ++m) sh0[lane + 32 * m] = kt::kt_tanh_bf(kt::dadd(acc[m], bias[m]));
  }
  __syncwarp();
  // hp = tanh(Wp1 h0 + bp1): Wp1 column-major (g x h); units lane, lane + 32 as two interleaved
  // 128-long chains, weights loaded 16 rows ahead
  {
    constexpr int B = 8;
    double a0 = 0.0, a1 = 0.0;
    double w0[B], w1[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      w0[j] = P[owp1 + j * kG + lane];
      w1[j] = P[owp1 + j * kG + lane + 32];
    }
#pragma unroll 1
    for (int i0 = 0; i0 < kH; i0 += B) {
      double n0[B], n1[B];
      const int i1 = i0 + B < kH ? i0 + B : i0;  // next batch (reloads the last one at the end)
#pragma unroll
      for (int j = 0; j < B; ++j) {
        n0[j] = P[owp1 + (i1 + j) * kG + lane];
        n1[j] = P[owp1 + (i1 + j) * kG + lane + 32];
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const double h = sh0[i0 + j];
        a0 = __fma_rn(w0[j], h, a0);
        a1 = __fma_rn(w1[j], h, a1);
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        w0[j] = n0[j];
        w1[j] = n1[j];
      }
    }
    const double b0v = P[obp1 + lane], b1v = P[obp1 + lane + 32];
    shp[lane] = kt::kt_tanh_bf(kt::dadd(a0, b0v));
    shp[lane + 32] = kt::kt_tanh_bf(kt::dadd(a1, b1v));
  }
  __syncwarp();
  // logits of the flagged knobs: item it -> (k-th flagged knob, a); weights loaded up front
  const int nf = __popc(fm);
  for (int it = lane; it < 3 * nf; it += 32) {
    uint32_t mm = fm;
    for (int q = 0; q < it / 3; ++q) mm &= mm - 1;
    const int a = 3 * (__ffs(mm) - 1) + it % 3;
    double acc = 0.0;
#pragma unroll
    for (int j0 = 0; j0 < kG; j0 += 16) {
      double w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = P[owp2 + (j0 + j) * 3 * n + a];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc = __fma_rn(w[j], shp[j0 + j], acc);
    }
    slg[it] = kt::dadd(acc, P[obp2 + a]);
  }
  __syncwarp();
  // the flagged knobs' exact softmax, draw and decision, one knob per lane, folded into lane L
  const uint64_t acts_L = __shfl_sync(0xffffffffu, acts, L);
  const uint32_t cert_L = __shfl_sync(0xffffffffu, fast_cert, L);
  int ae = 0, dk = 0;
  float lpk = 0.f;
  if (lane < nf) {
    uint32_t mm = fm;
    for (int q = 0; q < lane; ++q) mm &= mm - 1;
    dk = __ffs(mm) - 1;
    const kt::Knob3 k3 = kt::softmax3(slg[3 * lane], slg[3 * lane + 1], slg[3 * lane + 2]);
    // check mode 5 (planted draws): u was placed 2 delta from a FAST CDF value (fastp[2d+1])
    const uint64_t ge = (uint64_t)ge_L;
    const double u = check == 5 ? (double)fastp[2 * dk + 1]
                                : kt::hash01(tk.seed, (ge * (uint64_t)tk.T + (uint64_t)t) * (uint64_t)n + (uint64_t)dk);
    const double c1 = kt::dadd(k3.p[0], k3.p[1]);
    ae = u < k3.p[0] ? 0 : (u < c1 ? 1 : 2);
    // margin monitor (every re-decided knob, every mode): max |p_fast - p_exact| of the
    // decision's CDF values, so production runs keep measuring the certificate's margin
    const float e0 = fabsf((float)(fastp[2 * dk] - k3.p[0]));
    const float err = check == 5 ? e0 : fmaxf(e0, fabsf((float)(fastp[2 * dk + 1] - c1)));
    atomicMax(reinterpret_cast<unsigned int*>(stats + 3), __float_as_uint(err));
    if ((check == 1 || check == 5) && ((cert_L >> dk) & 1u)) {  // compare against the fast decision
      const int af = (int)((acts_L >> (2 * dk)) & 3u);
      if (af != ae) atomicAdd(stats + 2, 1ull);
    }
    lpk = (float)k3.lp[ae];
  }
  float lp_exact = 0.f;
  for (int j = 0; j < nf; ++j) {  // knob order (the joint log-probability is summed in that order)
    const int aj = __shfl_sync(0xffffffffu, ae, j), dj = __shfl_sync(0xffffffffu, dk, j);
    const float lj = __shfl_sync(0xffffffffu, lpk, j);
    if (lane == L) {
      acts = (acts & ~(3ull << (2 * dj))) | ((uint64_t)aj << (2 * dj));
      lp_exact += lj;
    }
  }
  __syncwarp();
  return {acts, lp_exact};
}

// Prologue shared by both kernels: the actor-critic weights -> fp16 hi/lo UMMA operands
// (power-of-two scaled), biases (and the value head) -> fp32 in shared memory.
__device__ __forceinline__ void stage_weights(const TcTask& tk, unsigned char* sm, const int* scard, int tid, int nthr) {
  const int n = tk.n, nk = nk_of(n), K1 = 2 * nk, N3 = n3_of(n);
  const double* __restrict__ P = tk.params;
  const int ob0 = kH * n, owp1 = ob0 + kH, obp1 = owp1 + kG * kH, owp2 = obp1 + kG, obp2 = owp2 + 3 * n * kG,
            owv1 = obp2 + 3 * n, obv1 = owv1 + kG * kH, owv2 = obv1 + kG, obv2 = owv2 + kG;
  unsigned char* B2 = sm + kOffB2;
  unsigned char* B1 = sm + kOffB1;
  unsigned char* B3 = sm + off_b3(n);
  float* f32 = reinterpret_cast<float*>(sm + off_f32(n));
  {
    const double s1 = ldexp(1.0, tk.e1), s2 = ldexp(1.0, tk.e2), s3 = ldexp(1.0, tk.e3);
    for (int i = tid; i < 128 * K1; i += nthr) {
      const int j = i / K1, k = i % K1, part = k >= nk, kk = part ? k - nk : k;
      double v = 0.0;
      if (kk < n && scard[kk] > 1) v = kt::dmul(kt::ddiv(P[kk * kH + j], (double)(scard[kk] - 1)), s1);
      const __half hi = __double2half(v);
      const __half o = part ? __double2half(kt::dsub(v, (double)__half2float(hi))) : hi;
      *reinterpret_cast<__half*>(B1 + kt::tc::kmajor_offset(j, k, K1)) = o;
    }
    for (int i = tid; i < 128 * 256; i += nthr) {
      const int u = i >> 8, k = i & 255, part = k >> 7, kk = k & 127;
      const double wv = u < kG ? P[owp1 + kk * kG + u] : P[owv1 + kk * kG + (u - kG)];
      const double v = kt::dmul(wv, s2);
      const __half hi = __double2half(v);
      const __half o = part ? __double2half(kt::dsub(v, (double)__half2float(hi))) : hi;
      *reinterpret_cast<__half*>(B2 + kt::tc::kmajor_offset(u, k, 256)) = o;
    }
    for (int i = tid; i < N3 * 128; i += nthr) {
      const int a = i >> 7, k = i & 127, part = k >> 6, kk = k & 63;
      const double v = a < 3 * n ? kt::dmul(P[owp2 + kk * 3 * n + a], s3) : 0.0;
      const __half hi = __double2half(v);
      const __half o = part ? __double2half(kt::dsub(v, (double)__half2float(hi))) : hi;
      *reinterpret_cast<__half*>(B3 + kt::tc::kmajor_offset(a, k, 128)) = o;
    }
    for (int i = tid; i < kNF32; i += nthr) {
      float v = 0.f;
      if (i < 128) v = (float)(P[ob0 + i] * (double)kK2L);  // tanh layers: bias * -2log2(e)
      else if (i < 192) v = (float)(P[obp1 + i - 128] * (double)kK2L);
      else if (i < 256) v = (float)(P[obv1 + i - 192] * (double)kK2L);
      else if (i < 320) v = (float)P[owv2 + i - 256];
      else if (i < 384) v = i - 320 < 3 * n ? (float)P[obp2 + i - 320] : 0.f;
      else if (i == 384) v = (float)P[obv2];
      f32[i] = v;
    }
  }
}

// kStream: the streamed host-buffer variant (compact encodings written here, per-segment
// progress published); a separate instantiation so the device-buffer path keeps its registers.
template <int NMAX, bool kStream>
__global__ void __launch_bounds__(kThr, 1) rollout_tc_kernel(const __grid_constant__ TcLaunch L) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t mbar[kSlots];
  __shared__ uint32_t tbase_sh;
  __shared__ int scard[kt::kMaxKnobs];
  int ti = 0;
  while (ti + 1 < L.num_tasks && L.task[ti + 1].cta_base <= (int)blockIdx.x) ++ti;
  const TcTask& tk = L.task[ti];
  const int jc = (int)blockIdx.x - tk.cta_base;
  const int wbase = tk.warps / tk.ctas, wextra = tk.warps % tk.ctas;
  const int nw = wbase + (jc < wextra ? 1 : 0);  // live warps of this CTA
  const int64_t row0 = (int64_t)(jc * wbase + min(jc, wextra)) * 32;
  const int n = tk.n, T = tk.T, nk = nk_of(n), K1 = 2 * nk, N3 = n3_of(n);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const double* __restrict__ P = tk.params;
  const int ob0 = kH * n, owp1 = ob0 + kH, obp1 = owp1 + kG * kH, owp2 = obp1 + kG, obp2 = owp2 + 3 * n * kG,
            owv1 = obp2 + 3 * n, obv1 = owv1 + kG * kH, owv2 = obv1 + kG, obv2 = owv2 + kG;

  unsigned char* B2 = sm + kOffB2;
  unsigned char* B1 = sm + kOffB1;
  unsigned char* B3 = sm + off_b3(n);
  float* f32 = reinterpret_cast<float*>(sm + off_f32(n));
  float* sb0 = f32;
  float* sbp1 = sb0 + 128;
  float* sbv1 = sbp1 + 64;
  float* swv2 = sbv1 + 64;
  float* sbp2 = swv2 + 64;
  float* sbv2 = sbp2 + 64;

  // ---- prologue: weights -> fp16 hi/lo operands, biases -> fp32
  if (tid < kt::kMaxKnobs) scard[tid] = tk.card[tid];
  __syncthreads();
  stage_weights(tk, sm, scard, tid, kThr);
  double* s_leaf = reinterpret_cast<double*>(sm + off_gbt(n));
  uint32_t* s_node = reinterpret_cast<uint32_t*>(sm + off_gbt(n) + (tk.gnode ? gbt_leaf_bytes(tk.ntrees, tk.depth) : 0));
  int32_t* s_col = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(s_node) +
                                              (tk.gnode ? gbt_node_bytes(tk.ntrees, tk.depth) : 0));
  if (tk.gnode) {
    const int NI = (1 << tk.depth) - 1, NL = 1 << tk.depth;
    for (int i = tid; i < tk.ntrees * NL; i += kThr) s_leaf[i] = tk.gleaf[i];
    for (int i = tid; i < tk.ntrees * NI; i += kThr) {
      const uint32_t wd = tk.gnode[i];
      s_node[i] = ((uint32_t)((wd >> 24) * kThr * 4) << 16) | min(wd & 0xFFFFFFu, 0xFFFFu);
    }
  }
  if (w == 0) kt::tc::tmem_alloc(&tbase_sh, 512);
  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) kt::tc::mbar_init(&mbar[s], 1);
    kt::tc::fence_mbar_init();
  }
  kt::tc::fence_proxy_async();
  kt::tc::fence_before();
  __syncthreads();
  kt::tc::fence_after();

  const int slot = w >> 2, q = w & 3;
  const bool slot_used = 4 * slot < nw;
  if (slot_used) {
    const bool lw = w < nw;
    const int64_t e = row0 + 32 * w + lane;
    const bool lr = lw && e < tk.E;
    const int r = 32 * q + lane;  // TMEM lane / operand row
    unsigned char* Ab = sm + kOffA + slot * kABytes;
    const uint32_t a_addr = kt::tc::smem_u32(Ab);
    const uint32_t tcol = tbase_sh + ((uint32_t)(32 * q) << 16) + (uint32_t)(128 * slot);
    const uint32_t tslot = tbase_sh + (uint32_t)(128 * slot);
    const bool leader = q == 0 && lane == 0;
    uint64_t* mb = &mbar[slot];
    // pre-activation scales (with -2log2(e) folded in for the tanh layers)
    const float sc1 = ldexpf(kK2L, -tk.e1), sc2 = ldexpf(kK2L, -(14 + tk.e2)), sc3 = ldexpf(1.f, -(14 + tk.e3));
    const uint32_t id128 = kt::tc::idesc_f16_f32(128, 128), idn3 = kt::tc::idesc_f16_f32(128, N3);
    const uint64_t ad0 = kt::tc::smem_desc(a_addr, 128, 2048);
    const uint64_t b1d = kt::tc::smem_desc(kt::tc::smem_u32(B1), 128, (K1 / 8) * 128);
    const uint64_t b2d = kt::tc::smem_desc(kt::tc::smem_u32(B2), 128, 4096);
    const uint64_t b3d = kt::tc::smem_desc(kt::tc::smem_u32(B3), 128, 2048);
    const uint64_t ge = (uint64_t)(tk.episode_offset + e);
    // exact re-decision scratch: the warp's own 8 KB of the operand buffer (its
    // rows' row groups), free between the L3 MMA and the next step's L1 operand
    double* sh0 = reinterpret_cast<double*>(Ab + 8192 * q);
    double* shp = reinterpret_cast<double*>(Ab + 8192 * q + 1024);
    double* slg = reinterpret_cast<double*>(Ab + 8192 * q + 1536);

    Cfg<NMAX> cfg;
#pragma unroll
    for (int i = 0; i < NMAX / 2; ++i) cfg.w[i] = 0;
    if (lr) {
      if (L.t_begin == 0) {
#pragma unroll
        for (int d = 0; d < NMAX; ++d)
          if (d < n) cfg.set(d, tk.init_idx[e * n + d]);
        store_row_idx(tk.idx + e * tk.sE * n, cfg, n);
        if constexpr (kStream) {
          if (tk.idx8) store_row_u8(tk.idx8 + e * tk.sE * n, cfg, n);
          if (tk.ids) tk.ids[e * tk.sE] = cfg_id(cfg, scard);
        }
      } else {  // resume a segmented rollout from trajectory row t_begin
        const uint16_t* src = tk.idx + (e * tk.sE + L.t_begin * tk.sT) * n;
#pragma unroll
        for (int d = 0; d < NMAX; ++d)
          if (d < n) cfg.set(d, src[d]);
      }
    }
    const unsigned char* mycol = reinterpret_cast<const unsigned char*>(s_col + tid);
    if (tk.gnode) {
#pragma unroll
      for (int d = 0; d < NMAX; ++d)
        if (d < n) s_col[d * kThr + tid] = cfg.get(d);
    }
    const int gh = tk.ntrees / 2;  // the walk of row t runs in two halves inside step t's MMA waits
    uint32_t ph = 0;
    // streamed variant: the first step of the next segment (segment of step x = floor(x nseg / T),
    // so segment s starts at ceil(s T / nseg)); divisions only at the boundaries
    int seg_next = 0;
    if constexpr (kStream)
      seg_next = (int)((((uint32_t)L.t_begin * (uint32_t)L.nseg) / (uint32_t)T + 1) * (uint32_t)T +
                       (uint32_t)L.nseg - 1) / (uint32_t)L.nseg;
#if KT_TC_TRACE
    const bool trace_cta = L.check == 2 && blockIdx.x == 0 && q == 0 && lane == 0;
#endif
#if KT_TC_TRACE  // phase trace (check mode 2, tools/trace_tc.py): build with -DKT_TC_TRACE=1
#define TR(k)                                                                                  \
  if (trace_cta && (t == 200 || t == 201))                                                      \
    L.counters[4 + (slot * 2 + (t - 200)) * 16 + (k)] = (unsigned long long)clock64();
#else
#define TR(k)
#endif
    for (int t = L.t_begin; t < L.t_end; ++t) {
      TR(0)
      // ---- L1 operand: [idx | idx] as fp16 (exact integers)
      if (lw) {
#pragma unroll
        for (int c = 0; c < NMAX / 8; ++c) {
          if (8 * c < nk) {
            uint32_t pk[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int d = 8 * c + 2 * p;
              pk[p] = h2bits(__floats2half2_rn((float)cfg.get(d), (float)cfg.get(d + 1)));
            }
            const uint4 v = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, 8 * c, 128)) = v;
            *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, nk + 8 * c, 128)) = v;
          }
        }
      }
      sync_slot(slot);
      TR(1)
      if (leader) {
        kt::tc::fence_after();
        if (L.check != 3)
          for (int kb = 0; kb < K1 / 16; ++kb) kt::tc::mma_f16(tslot, ad0 + 16 * kb, b1d + 16 * kb, id128, kb > 0);
        kt::tc::commit(mb);
      }
      uint32_t raw[64];
      double gs = 0.0;
      float ufs[NMAX];  // this step's counter-RNG draws, computed while the L2 (K half 1) MMAs run
      if (lw) {
        if (tk.gnode) gs = gbt_walk(0.0, s_node, s_leaf, mycol, 0, gh, tk.depth);  // fused K1, row t
        kt::tc::mbar_wait(mb, ph);
        kt::tc::fence_after();
        TR(2)
        // ---- L1 epilogue, units 0..63: h0 = tanh(W0 x + b0) -> L2 operand (K half 0)
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t v[16];
          kt::tc::ld_32x32b_x16(tcol + c0, v);
          kt::tc::ld_wait();
          act_store16(Ab, r, c0, v, sc1, sb0 + c0);
        }
        // units 64..127: raw accumulators to registers before L2 overwrites the columns
        uint32_t* r0 = raw;
        kt::tc::ld_32x32b_x32(tcol + 64, *reinterpret_cast<uint32_t(*)[32]>(r0));
        kt::tc::ld_32x32b_x32(tcol + 96, *reinterpret_cast<uint32_t(*)[32]>(r0 + 32));
        kt::tc::ld_wait();
      }
      ph ^= 1;
      TR(3)
      sync_slot(slot);
      TR(4)
      if (leader) {  // L2, K half 0
        kt::tc::fence_after();
        if (L.check != 3) mma_split4(tslot, ad0, b2d, 128, 0, id128, false);
        kt::tc::commit(mb);
      }
      if (lw) {
        // units 64..127 while the L2 MMAs run: tanh + hi/lo split in registers
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          const float2 h = act2(pre2(raw[j], raw[j + 1], sc1, sb0 + 64 + j), kActScale);
          split2(h.x, h.y, raw[j], raw[j + 1]);  // raw[j] = hi pair, raw[j+1] = lo pair
        }
        TR(5)
        kt::tc::mbar_wait(mb, ph);
        kt::tc::fence_after();
        TR(6)
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, 8 * m, 128)) =
              make_uint4(raw[8 * m], raw[8 * m + 2], raw[8 * m + 4], raw[8 * m + 6]);
          *reinterpret_cast<uint4*>(Ab + kt::tc::kmajor_offset(r, 64 + 8 * m, 128)) =
              make_uint4(raw[8 * m + 1], raw[8 * m + 3], raw[8 * m + 5], raw[8 * m + 7]);
        }
      }
      ph ^= 1;
      sync_slot(slot);
      TR(8)
      if (leader) {  // L2, K half 1
        kt::tc::fence_after();
        if (L.check != 3) mma_split4(tslot, ad0, b2d, 128, 4, id128, true);
        kt::tc::commit(mb);
      }
      if (lw) {
#pragma unroll
        for (int d = 0; d < NMAX; ++d) {
          const uint64_t hsh = kt::mix64(tk.seed ^ kt::mix64((ge * (uint64_t)T + (uint64_t)t) * (uint64_t)n +
                                                             (uint64_t)d + 0x9E3779B97F4A7C15ULL));
          ufs[d] = (float)(uint32_t)(hsh >> 40) * 0x1.0p-24f;  // |uf - u| < 2^-24
          if constexpr (NMAX > 8) asm volatile("" : "+f"(ufs[d]));  // keep the draws inside the L2 MMA window
        }
        if constexpr (NMAX == 8) {  // park them in shared memory across the L2 epilogue (no spills)
          float4* sd = reinterpret_cast<float4*>(sm + off_draw(n));
          sd[tid] = make_float4(ufs[0], ufs[1], ufs[2], ufs[3]);
          sd[kThr + tid] = make_float4(ufs[4], ufs[5], ufs[6], ufs[7]);
        }
        if (tk.gnode) {  // fused K1, row t: second half of the walk while the L2 MMAs run
          gs = gbt_walk(gs, s_node, s_leaf, mycol, gh, tk.ntrees, tk.depth);
          if (lr) tk.score[e * tk.sE + t * tk.sT] = kt::dadd(tk.gbase, kt::dmul(tk.glr, gs));
        }
        kt::tc::mbar_wait(mb, ph);
        kt::tc::fence_after();
        TR(9)
        // ---- L2 epilogue (policy half): hp -> L3 operand
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t v[16];
          kt::tc::ld_32x32b_x16(tcol + c0, v);
          kt::tc::ld_wait();
          act_store16(Ab, r, c0, v, sc2, sbp1 + c0);
        }
      }
      ph ^= 1;
      sync_slot(slot);
      TR(11)
      if (leader) {  // L3 logits (accumulator columns 0..N3-1; hv stays in 64..127)
        kt::tc::fence_after();
        if (L.check != 3) mma_split4(tslot, ad0, b3d, 64, 0, idn3, false);
        kt::tc::commit(mb);
      }
      if (lw) {
        // ---- L2 epilogue (value half), overlapping the L3 MMAs: v = wv2 . tanh(.) + bv2
        float2 vs2 = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int c0 = 64; c0 < 128; c0 += 16) {
          uint32_t v[16];
          kt::tc::ld_32x32b_x16(tcol + c0, v);
          kt::tc::ld_wait();
#pragma unroll
          for (int j = 0; j < 16; j += 2)
            vs2 = __ffma2_rn(*reinterpret_cast<const float2*>(swv2 + c0 - 64 + j),
                             act2(pre2(v[j], v[j + 1], sc2, sbv1 + c0 - 64 + j), 1.f), vs2);
        }
        const float vs = vs2.x + vs2.y;
        if (lr && L.check != 4) {
          const float v = vs + sbv2[0];
          if (tk.value) tk.value[e * tk.aE + t * tk.aT] = (double)v;
          if (tk.value32) tk.value32[e * tk.aE + t * tk.aT] = v;
        }
        TR(12)
        kt::tc::mbar_wait(mb, ph);
        kt::tc::fence_after();
        TR(13)
        // ---- L3 epilogue: per-knob softmax, certified inverse-CDF draw, saturating move
        if constexpr (NMAX == 8) {
          const float4* sd = reinterpret_cast<const float4*>(sm + off_draw(n));
          const float4 u0 = sd[tid], u1 = sd[kThr + tid];
          ufs[0] = u0.x; ufs[1] = u0.y; ufs[2] = u0.z; ufs[3] = u0.w;
          ufs[4] = u1.x; ufs[5] = u1.y; ufs[6] = u1.z; ufs[7] = u1.w;
        }
        uint64_t acts = 0;
        uint32_t cert = 0;
        float lpj = 0.f;
        const float delta = L.delta;
        float* fastp = reinterpret_cast<float*>(Ab + 8192 * q + 2048);  // fast p0/c1 per (row, knob) for re-decisions
        float fp0[NMAX], fc1[NMAX];
        // Branch-free over all NMAX knobs (knobs >= n see zero logits and are masked), so the
        // per-knob dependent chains (ex2 -> rcp -> lg2) of all knobs interleave.
#pragma unroll
        for (int g = 0; g < NMAX / 8; ++g) {  // knob groups of 8: 24 logit columns
          if (8 * g < n) {
            uint32_t v[24];
            kt::tc::ld_32x32b_x16(tcol + 24 * g, *reinterpret_cast<uint32_t(*)[16]>(v));
            kt::tc::ld_32x32b_x8(tcol + 24 * g + 16, *reinterpret_cast<uint32_t(*)[8]>(v + 16));
            kt::tc::ld_wait();
#pragma unroll
            for (int dd = 0; dd < 8; ++dd) {
              const int d = 8 * g + dd;
              const float l0 = fmaf(__uint_as_float(v[3 * dd]), sc3, sbp2[3 * d]);
              const float l1 = fmaf(__uint_as_float(v[3 * dd + 1]), sc3, sbp2[3 * d + 1]);
              const float l2 = fmaf(__uint_as_float(v[3 * dd + 2]), sc3, sbp2[3 * d + 2]);
              const float m = fmaxf(l0, fmaxf(l1, l2));
              const float e0 = ex2f((l0 - m) * 1.4426950408889634f), e1 = ex2f((l1 - m) * 1.4426950408889634f),
                          e2 = ex2f((l2 - m) * 1.4426950408889634f);
              const float s = e0 + e1 + e2;
              const float rs = rcpf(s);
              const float p0 = e0 * rs, c1 = (e0 + e1) * rs;
              float uf = ufs[d];
              if (L.check == 5) {  // planted draw 2 delta below/above p0 or c1 (bits of the real draw)
                const float base = uf < 0.5f ? p0 : c1;
                uf = fminf(fmaxf(base + ((uf * 4.f - floorf(uf * 4.f)) < 0.5f ? -2.f : 2.f) * delta, 0.f),
                           0x1.fffffep-1f);
              }
              const int a = uf < p0 ? 0 : (uf < c1 ? 1 : 2);
              const bool ok = fabsf(uf - p0) > delta && fabsf(uf - c1) > delta && d < n;
              acts |= (uint64_t)a << (2 * d);
              fp0[d] = p0;
              fc1[d] = L.check == 5 ? uf : c1;
              const float lpa = (a == 0 ? l0 : (a == 1 ? l1 : l2)) - m - lg2f(s) * 0.69314718055994531f;
              cert |= ok ? 1u << d : 0u;
              lpj += ok ? lpa : 0.f;  // uncertain knobs add their exact log-probability later
            }
          } else {
#pragma unroll
            for (int dd = 0; dd < 8; ++dd) fp0[8 * g + dd] = fc1[8 * g + dd] = 0.f;
          }
        }
        uint32_t fb;
        TR(14)
        const uint32_t allk = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
        const bool chk = L.check == 1 || L.check == 5;  // every knob re-decided exactly
        fb = chk ? allk : (allk & ~cert);
        if (!lr) fb = 0;
        if (fb) {  // rare: the re-decision compares against (and monitors) the fast values
#pragma unroll
          for (int d = 0; d < NMAX; ++d) {
            fastp[(lane * NMAX + d) * 2] = fp0[d];
            fastp[(lane * NMAX + d) * 2 + 1] = fc1[d];
          }
        }
        unsigned pend = __ballot_sync(0xffffffffu, fb != 0);
        float lpx = 0.f;
        if (pend) {
          const unsigned nk = __reduce_add_sync(0xffffffffu, (unsigned)__popc(fb));
          if (lane == 0 && L.counters) atomicAdd(L.counters + (chk ? 1 : 0), (unsigned long long)nk);
        }
        while (pend) {
          const int Lr = __ffs(pend) - 1;
          pend &= pend - 1;
          const uint32_t fm = __shfl_sync(0xffffffffu, fb, Lr);
          const int64_t geL = __shfl_sync(0xffffffffu, (long long)ge, Lr);
          const Redecided rd = exact_redecide<NMAX>(tk, t, Lr, fm, cfg, scard, sh0, shp, slg, geL, acts,
                                                    fastp + Lr * NMAX * 2, cert, L.counters, L.check);
          if (lane == Lr) {
            acts = rd.acts;
            lpx = rd.lp;
          }
        }
        TR(7)
        if (chk) lpj = lpx;  // every knob re-decided: exact log-probabilities
        else lpj += lpx;
        // saturating move (design_space.cpp:175-187) and the trajectory writes
        uint32_t apk[(NMAX + 3) / 4];
#pragma unroll
        for (int i = 0; i < (NMAX + 3) / 4; ++i) apk[i] = 0;
#pragma unroll
        for (int d = 0; d < NMAX; ++d) {  // branch-free: knobs >= n have card 1, index 0, and stay 0
          const int a = (int)((acts >> (2 * d)) & 3u);
          int v = cfg.get(d) + a - 1;
          v = v < 0 ? 0 : (v > scard[d] - 1 ? scard[d] - 1 : v);
          cfg.set(d, v);
          apk[d >> 2] |= (uint32_t)(uint8_t)(int8_t)(a - 1) << (8 * (d & 3));
        }
        if (tk.gnode) {  // the new configuration (row t+1) for the next step's fused walk
#pragma unroll
          for (int d = 0; d < NMAX; ++d)
            if (d < n) s_col[d * kThr + tid] = cfg.get(d);
        }
        TR(10)
        if (lr && L.check != 4) {  // 4: timing experiment (no trajectory writes)
          store_row_idx(tk.idx + (e * tk.sE + (t + 1) * tk.sT) * n, cfg, n);
          if constexpr (kStream) {
            if (tk.idx8) store_row_u8(tk.idx8 + (e * tk.sE + (t + 1) * tk.sT) * n, cfg, n);
            if (tk.ids) tk.ids[e * tk.sE + (t + 1) * tk.sT] = cfg_id(cfg, scard);
            if (tk.act2) store_act2(tk.act2 + (e * tk.aE + t * tk.aT) * ((n + 3) / 4), acts, n);
          }
          if (tk.actions) {
            int8_t* ad = tk.actions + (e * tk.aE + t * tk.aT) * n;
            if ((n & 3) == 0) {
#pragma unroll
              for (int i = 0; i < (NMAX + 3) / 4; ++i)
                if (4 * i < n) reinterpret_cast<uint32_t*>(ad)[i] = apk[i];
            } else {
#pragma unroll
              for (int d = 0; d < NMAX; ++d)
                if (d < n) ad[d] = (int8_t)((apk[d >> 2] >> (8 * (d & 3))) & 0xFF);
            }
          }
          if (tk.logp) tk.logp[e * tk.aE + t * tk.aT] = (double)lpj;
          if (tk.logp32) tk.logp32[e * tk.aE + t * tk.aT] = lpj;
        }
      }
      ph ^= 1;
      TR(15)
      if constexpr (kStream) {
        if (t + 1 == seg_next && t + 1 < L.t_end) {
          __threadfence();  // this row's step-t outputs are visible GPU-wide (at L2) ...
          sync_slot(slot);  // ... for every row of the slot
          const uint32_t sg = (uint32_t)(t * L.nseg) / (uint32_t)T;  // the segment step t closes
          if (leader) {
            __threadfence_system();
            atomicAdd(L.progress + sg, 1u);
          }
          seg_next = (int)(((sg + 2) * (uint32_t)T + (uint32_t)L.nseg - 1) / (uint32_t)L.nseg);
        }
      }
    }
#undef TR
    if (tk.gnode && lr && L.t_end == T)  // row T
      tk.score[e * tk.sE + T * tk.sT] =
          kt::dadd(tk.gbase, kt::dmul(tk.glr, gbt_walk(0.0, s_node, s_leaf, mycol, 0, tk.ntrees, tk.depth)));
  }
  kt::tc::fence_before();
  __syncthreads();
  if (w == 0) kt::tc::tmem_dealloc(tbase_sh, 512);
}

// Power-of-two scale e with max|W| * 2^e < 2^14 (0 for an all-zero matrix).
int pow2_scale(double maxabs) {
  if (!(maxabs > 0.0)) return 0;
  int ex = 0;
  std::frexp(maxabs, &ex);  // maxabs < 2^ex
  return 14 - ex;
}

}  // namespace

namespace kt {

bool rollout_tc_eligible(const ktune_ac* ac, const ktune_space* sp) {
  if (!ac || !sp || ac->h != kH || ac->g != kG || ac->n < 1 || ac->n > kTcMaxN || sp->D != ac->n) return false;
  for (int c : sp->card)
    if (c > 2049) return false;  // fp16 holds the knob indices exactly up to 2048
  return true;
}

void resolve_counters(ktune_ctx* ctx) {
  if (!ctx->d_counters) return;
  unsigned long long c[4];
  KT_CUDA(cudaStreamSynchronize(ctx->stream));
  KT_CUDA(cudaMemcpy(c, ctx->d_counters, sizeof(c), cudaMemcpyDeviceToHost));
  KT_CUDA(cudaMemset(ctx->d_counters, 0, sizeof(c)));
  ctx->stats[KTUNE_STAT_ROLLOUT_FALLBACKS] += (int64_t)c[0];
  ctx->stats[KTUNE_STAT_ROLLOUT_CHECKED] += (int64_t)c[1];
  ctx->stats[KTUNE_STAT_ROLLOUT_MISMATCH] += (int64_t)c[2];
  float mx;
  const unsigned int bits = (unsigned int)c[3];
  std::memcpy(&mx, &bits, 4);
  ctx->stats[KTUNE_STAT_ROLLOUT_MAXERR] =
      std::max<int64_t>(ctx->stats[KTUNE_STAT_ROLLOUT_MAXERR], (int64_t)std::llround((double)mx * 1e12));
}

// Returns the number of episode slots launched (each adds 1 to progress[s] per segment s).
static int64_t rollout_tc_launch(ktune_ctx* ctx, std::vector<RolloutWork>& work, int T, int t_begin, int t_end,
                                 bool allow_fuse, unsigned int* progress, int nseg) {
  int64_t total = 0;
  if (!ctx->d_counters) {
    KT_CUDA(cudaMalloc(&ctx->d_counters, (4 + 8 * 16) * sizeof(unsigned long long)));
    KT_CUDA(cudaMemsetAsync(ctx->d_counters, 0, (4 + 8 * 16) * sizeof(unsigned long long), ctx->stream));
  }
  // Certification margin: fast-vs-exact probability error (calibrated with
  // KTUNE_OPT_ROLLOUT_CHECK) plus the 2^-24 draw truncation.
  const float delta = ctx->opt_rollout_delta > 0 ? (float)((double)ctx->opt_rollout_delta * 1e-12)
                                                  : (float)(0x1.0p-16 + 0x1.0p-24);
  const int S = sm_count(ctx);
  for (size_t t0 = 0; t0 < work.size(); t0 += kMaxTcTasks) {
    const size_t nt = std::min<size_t>(kMaxTcTasks, work.size() - t0);
    TcLaunch L{};
    L.check = (int)ctx->opt_rollout_check;  // 2: phase trace (debug)
    L.t_begin = t_begin;
    L.t_end = t_end;
    L.delta = delta;
    L.counters = ctx->d_counters;
    L.progress = progress;
    L.nseg = nseg;
    // warps per task, then the smallest per-CTA warp count m whose CTA total fits one wave
    std::vector<int64_t> W(nt);
    int64_t wsum = 0;
    int nmax = 1;
    for (size_t k = 0; k < nt; ++k) {
      W[k] = ceil_div(work[t0 + k].E, 32);
      wsum += W[k];
      nmax = std::max(nmax, work[t0 + k].ac->n);
    }
    int m = kMaxWarps;
    if (wsum <= (int64_t)kMaxWarps * S) {
      for (m = 1; m < kMaxWarps; ++m) {
        int64_t c = 0;
        for (size_t k = 0; k < nt; ++k) c += ceil_div(W[k], m);
        if (c <= S) break;
      }
    }
    int ctas = 0;
    int nl = 0;
    int64_t slots = 0;
    for (size_t k = 0; k < nt; ++k) {
      if (W[k] == 0) continue;
      const RolloutWork& rw = work[t0 + k];
      TcTask& tk = L.task[nl++];
      for (int d = 0; d < kMaxKnobs; ++d) {
        tk.card[d] = d < rw.space->D ? rw.space->card[d] : 1;
        tk.foff[d] = d < rw.space->D ? (int32_t)rw.space->val_off[d] : 0;
      }
      tk.flut = rw.space->d_lut;
      tk.params = rw.ac->d_params;
      tk.n = rw.ac->n;
      tk.T = T;
      tk.E = rw.E;
      tk.episode_offset = rw.episode_offset;
      tk.sE = rw.sE;
      tk.sT = rw.sT;
      tk.aE = rw.aE;
      tk.aT = rw.aT;
      tk.seed = rw.seed;
      tk.init_idx = rw.init_idx;
      tk.idx = rw.idx;
      tk.actions = rw.actions;
      tk.logp = rw.logp;
      tk.value = rw.value;
      tk.logp32 = rw.logp32;
      tk.value32 = rw.value32;
      tk.idx8 = rw.idx8;
      tk.ids = rw.ids;
      tk.act2 = rw.act2;
      if (!progress && (rw.idx8 || rw.ids || rw.act2))
        fail(KTUNE_ERR_LOGIC, "rollout: compact encodings are written by the streamed variant only");
      tk.warps = (int32_t)W[k];
      tk.ctas = (int32_t)ceil_div(W[k], m);
      tk.cta_base = ctas;
      ctas += tk.ctas;
      for (int jc = 0; jc < tk.ctas; ++jc)  // the kernel's split: wbase (+1 for the first wextra CTAs) warps
        slots += ceil_div((int64_t)(tk.warps / tk.ctas + (jc < tk.warps % tk.ctas ? 1 : 0)), 4);
      // weight scales from the host copy of the parameters (cached per parameter version and space)
      const int n = tk.n;
      if (rw.ac->scale_version != rw.ac->version || rw.ac->scale_space != rw.space) {
        const std::vector<double>& p = rw.ac->host_params;
        const int ob0 = kH * n, owp1 = ob0 + kH, obp1 = owp1 + kG * kH, owp2 = obp1 + kG,
                  obp2 = owp2 + 3 * n * kG, owv1 = obp2 + 3 * n, obv1 = owv1 + kG * kH;
        double m1 = 0, m2 = 0, m3 = 0;
        for (int i = 0; i < n; ++i)
          if (tk.card[i] > 1)
            for (int j = 0; j < kH; ++j) m1 = std::max(m1, std::fabs(p[i * kH + j]) / (double)(tk.card[i] - 1));
        for (int i = owp1; i < obp1; ++i) m2 = std::max(m2, std::fabs(p[i]));
        for (int i = owv1; i < obv1; ++i) m2 = std::max(m2, std::fabs(p[i]));
        for (int i = owp2; i < obp2; ++i) m3 = std::max(m3, std::fabs(p[i]));
        rw.ac->scale_e[0] = pow2_scale(m1);
        rw.ac->scale_e[1] = pow2_scale(m2);
        rw.ac->scale_e[2] = pow2_scale(m3);
        rw.ac->scale_space = rw.space;
        rw.ac->scale_version = rw.ac->version;
      }
      // optional fused scoring (complete-tree index layout that fits in shared memory)
      const ktune_gbt* g = rw.gbt;
      tk.gnode = nullptr;
      if (g && rw.score && g->has_space && g->complete && g->d_inode_idx && g->depth <= 8 && t_begin == 0 && t_end == T &&
          tc_smem_bytes(n, g->num_trees, g->depth) <= 227 * 1024 && ctx->opt_rollout_fuse_gbt && allow_fuse) {
        tk.gnode = g->d_inode_idx;
        tk.gleaf = g->d_leaf;
        tk.ntrees = g->num_trees;
        tk.depth = g->depth;
        tk.gbase = g->base;
        tk.glr = g->lr;
        tk.score = rw.score;
        work[t0 + k].scored = true;
      }
      tk.e1 = rw.ac->scale_e[0];
      tk.e2 = rw.ac->scale_e[1];
      tk.e3 = rw.ac->scale_e[2];
      if (tk.e1 > 100 || tk.e2 > 100 || tk.e3 > 100 || tk.e1 < -100 || tk.e2 < -100 || tk.e3 < -100)
        fail(KTUNE_ERR_CONFIG, "rollout: actor-critic weights out of the tensor-core path's range");
      ctx->stats[KTUNE_STAT_ROLLOUT_TC] += rw.E * (int64_t)(t_end - t_begin);
    }
    L.num_tasks = nl;
    if (ctas == 0 || (t_end <= t_begin && t_begin != 0)) continue;  // T = 0 still writes row 0
    size_t smem = 0;
    for (int k = 0; k < nl; ++k)
      smem = std::max<size_t>(smem, tc_smem_bytes(L.task[k].n, L.task[k].gnode ? L.task[k].ntrees : 0,
                                                   L.task[k].depth));
    auto kern = progress ? (nmax <= 8 ? rollout_tc_kernel<8, true>
                                      : (nmax <= 16 ? rollout_tc_kernel<16, true> : rollout_tc_kernel<24, true>))
                         : (nmax <= 8 ? rollout_tc_kernel<8, false>
                                      : (nmax <= 16 ? rollout_tc_kernel<16, false> : rollout_tc_kernel<24, false>));
    KT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)ctas, kThr, smem, ctx->stream>>>(L);
    check_launch(ctx, "rollout_tc");
    total += slots;
  }
  return total;
}

// Episodes [e, E) of a workload as a workload of its own (global ids, pointers advanced).
static RolloutWork episode_tail(const RolloutWork& w, int64_t e, int T) {
  RolloutWork t = w;
  const int64_t n = w.ac->n;
  t.E = w.E - e;
  t.episode_offset = w.episode_offset + e;
  t.init_idx = w.init_idx + e * n;
  t.idx = w.idx + e * w.sE * n;
  if (w.actions) t.actions = w.actions + e * w.aE * n;
  if (w.logp) t.logp = w.logp + e * w.aE;
  if (w.value) t.value = w.value + e * w.aE;
  if (w.logp32) t.logp32 = w.logp32 + e * w.aE;
  if (w.value32) t.value32 = w.value32 + e * w.aE;
  if (w.score) t.score = w.score + e * w.sE;
  if (w.idx8) t.idx8 = w.idx8 + e * w.sE * n;
  if (w.ids) t.ids = w.ids + e * w.sE;
  if (w.act2) t.act2 = w.act2 + e * w.aE * ((n + 3) / 4);
  t.scored = false;
  return t;
}

int64_t rollout_tc(ktune_ctx* ctx, std::vector<RolloutWork>& work, int T, int t_begin, int t_end,
                   unsigned int* progress, int nseg) {
  // A tile of episodes is bound to its slot for all T steps, so a workload larger than one
  // resident wave (kMaxWarps warps on every SM) would end with a part-filled wave running
  // at the full per-step latency. One workload: full waves, then the remainder spread thin
  // over every SM (e.g. 65,536 episodes = 1.15 waves).
  const int64_t cap = (int64_t)kMaxWarps * sm_count(ctx);
  if (work.size() != 1 || ceil_div(work[0].E, 32) <= cap) {
    return rollout_tc_launch(ctx, work, T, t_begin, t_end, true, progress, nseg);
  }
  int64_t total = 0;
  RolloutWork rest = work[0];
  while (ceil_div(rest.E, 32) > cap) {
    std::vector<RolloutWork> wave(1, rest);
    wave[0].E = cap * 32;
    total += rollout_tc_launch(ctx, wave, T, t_begin, t_end, false, progress, nseg);
    rest = episode_tail(rest, cap * 32, T);
  }
  std::vector<RolloutWork> last(1, rest);
  total += rollout_tc_launch(ctx, last, T, t_begin, t_end, false, progress, nseg);
  work[0].scored = false;
  return total;
}

}  // namespace kt

extern "C" int ktune_debug_trace(ktune_ctx* ctx, unsigned long long* out) {
  return kt_guard(ctx, [&] {
    if (!ctx->d_counters) kt::fail(KTUNE_ERR_CONFIG, "no tcgen05 rollout has run on this context");
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    KT_CUDA(cudaMemcpy(out, ctx->d_counters, (4 + 8 * 16) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}
