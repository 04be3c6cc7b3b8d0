// K2: persistent batched rollout (run_episodes) and the
// ActorCritic forward (actor_critic.hpp:43).
//
// Exact fp64 path: every dot product, tanh/exp/log and the sampling compare
// evaluates exactly as the oracle restatement does, so
// actions, configurations, log-probabilities and values are bit-identical.
//
// Layout: one CTA of 128 threads owns a tile of 32 episodes for all T steps;
// the configurations stay resident in shared memory for the whole episode
// and the actor-critic parameters (fp64, ~175 KB at n=16) are staged into
// shared memory once per CTA. Per step:
//   0: x[i][c] = idx/(card-1)
//   A: h0[j][c] = tanh(W0 x + b0)            thread = hidden unit j
//   B: hp/hv[u][c] = tanh(W h0 + b)           thread = head unit u, 8 configs per weight load
//   C: logits[a][c], value[c]                 thread = (config, logit) items
//   D: per (config, knob) log-softmax, counter-RNG draw, saturating move
//   E: joint log-probability, trajectory writes
#include <cuda.h>  // CUresult / CUstream for the cuStreamWaitValue32 entry point (no -lcuda)

#include <algorithm>
#include <cstdlib>
#include <array>

#include "device.cuh"
#include "internal.cuh"

namespace {

constexpr int kThreads = 512;  // 16 warps per CTA; every phase maps lane <-> episode
constexpr int kWarps = kThreads / 32;
constexpr int kUnits = 8;      // hidden units per thread per pass (independent fp64 chains)

struct AcOff {
  int w0, b0, wp1, bp1, wp2, bp2, wv1, bv1, wv2, bv2, total;
};

__host__ __device__ inline AcOff ac_layout(int n, int h, int g) {
  AcOff o;
  o.w0 = 0;
  o.b0 = o.w0 + h * n;
  o.wp1 = o.b0 + h;
  o.bp1 = o.wp1 + g * h;
  o.wp2 = o.bp1 + g;
  o.bp2 = o.wp2 + 3 * n * g;
  o.wv1 = o.bp2 + 3 * n;
  o.bv1 = o.wv1 + g * h;
  o.wv2 = o.bv1 + g;
  o.bv2 = o.wv2 + g;
  o.total = o.bv2 + 1;
  return o;
}

struct RolloutTask {
  int32_t card[kt::kMaxKnobs];
  const double* params;  // device, flat layout
  int n, h, g;
  int T;
  int64_t E;
  int64_t episode_offset;
  uint64_t seed;
  const uint16_t* init_idx;
  uint16_t* idx;
  int8_t* actions;
  double* logp;
  double* value;
  float* logp32;
  float* value32;
  // trajectory layout (rows): (e, t) of the (T+1)-row arrays at e*sE + t*sT, of the T-row
  // arrays at e*aE + t*aT: episode-major (T+1, 1, T, 1) or step-major (1, E, 1, E)
  int64_t sE, sT, aE, aT;
};

// Whole launch description passed BY VALUE (kernel parameter space), so a
// launch needs no host->device copy: CTA b serves task t with
// cta_base[t] <= b < cta_base[t+1].
constexpr int kMaxTasksPerLaunch = 12;
struct RolloutLaunch {
  int32_t num_tasks;
  int32_t cta_base[kMaxTasksPerLaunch + 1];
  RolloutTask task[kMaxTasksPerLaunch];
};

__host__ __device__ inline int act_rows(int n, int h, int g) {
  int r = h > 2 * g ? h : 2 * g;
  return r > 3 * n ? r : 3 * n;  // logits alias the activation rows after layer 2
}

// Shared-memory carve-up (doubles): params (even-padded) | act [rows][tile] |
// x [n][tile] | val [tile] | then uint16 cfg [n][tile] | int32 card [n].
__host__ __device__ inline size_t rollout_smem_bytes(int n, int h, int g, bool smem_params, int cpl) {
  const AcOff o = ac_layout(n, h, g);
  const int tile = 32 * cpl;
  size_t d = (smem_params ? (size_t)((o.total + 1) & ~1) : 0) + (size_t)act_rows(n, h, g) * tile +
             (size_t)n * tile + tile;
  return d * 8 + (size_t)tile * n * 2 + (size_t)n * 4 + 16;
}

__device__ __forceinline__ void load8(const double* p, double (&w)[kUnits]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int r = 0; r < kUnits / 2; ++r) {
    const double2 v = q[r];
    w[2 * r] = v.x;
    w[2 * r + 1] = v.y;
  }
}

// One exact forward pass over the tile's states held in x[i][e] (e = lane + 32q).
// Leaves logits in act[a][e] (aliasing the hidden activations), values in val[e].
// Weight reads are warp-uniform 16-byte broadcasts feeding 32*CPL FMAs each;
// activation reads are lane-contiguous (conflict-free).
template <int CPL>
__device__ void forward_tile(const double* __restrict__ P, const AcOff& o, int n, int h, int g,
                             double* act, const double* x, double* val) {
  constexpr int tile = 32 * CPL;
  const int c = threadIdx.x & 31, w = threadIdx.x >> 5;
  // ---- A: h0[j][e] = tanh(sum_i fma(W0(j,i), x[i][e]) + b0[j]);  W0 column-major (h x n)
  for (int ub = w * kUnits; ub < h; ub += kWarps * kUnits) {
    double acc[CPL][kUnits];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int r = 0; r < kUnits; ++r) acc[q][r] = 0.0;
    for (int i = 0; i < n; ++i) {
      double wr[kUnits];
      load8(P + o.w0 + i * h + ub, wr);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const double xv = x[i * tile + c + 32 * q];
#pragma unroll
        for (int r = 0; r < kUnits; ++r) acc[q][r] = __fma_rn(wr[r], xv, acc[q][r]);
      }
    }
    double b[kUnits];
    load8(P + o.b0 + ub, b);
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int r = 0; r < kUnits; ++r)
        act[(ub + r) * tile + c + 32 * q] = kt::kt_tanh_bf(kt::dadd(acc[q][r], b[r]));
  }
  __syncthreads();
  // ---- B: units u < g: hp = tanh(Wp1 h0 + bp1); g <= u < 2g: hv = tanh(Wv1 h0 + bv1)
  constexpr int kPasses = CPL == 1 ? 2 : 1;  // 2g <= 256 (CPL 1) or <= 128 (CPL 2)
  double res[kPasses][CPL][kUnits];
#pragma unroll
  for (int pass = 0; pass < kPasses; ++pass) {
    const int ub = w * kUnits + pass * kWarps * kUnits;
    if (ub >= 2 * g) break;
    const double* wb = ub < g ? P + o.wp1 + ub : P + o.wv1 + (ub - g);
    double acc[CPL][kUnits];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int r = 0; r < kUnits; ++r) acc[q][r] = 0.0;
#pragma unroll 2
    for (int i = 0; i < h; ++i) {
      double wr[kUnits];
      load8(wb + i * g, wr);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const double xv = act[i * tile + c + 32 * q];
#pragma unroll
        for (int r = 0; r < kUnits; ++r) acc[q][r] = __fma_rn(wr[r], xv, acc[q][r]);
      }
    }
    double b[kUnits];
    load8(ub < g ? P + o.bp1 + ub : P + o.bv1 + (ub - g), b);
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int r = 0; r < kUnits; ++r) res[pass][q][r] = kt::kt_tanh_bf(kt::dadd(acc[q][r], b[r]));
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < kPasses; ++pass) {
    const int ub = w * kUnits + pass * kWarps * kUnits;
    if (ub >= 2 * g) break;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int r = 0; r < kUnits; ++r) act[(ub + r) * tile + c + 32 * q] = res[pass][q][r];
  }
  __syncthreads();
  // ---- C: logits (Wp2 column-major 3n x g) and value; items a = w + 16j, up to
  // 8 per warp (n <= 32), held in registers until every hp/hv read is done,
  // then written over the activation rows.
  const int na = 3 * n + 1;
  double outv[2][4][CPL];
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int a0 = w + pass * 4 * kWarps;
    if (a0 >= na) break;
    const double* wp[4];
    int ws[4];
    const double* hrow[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = a0 + k * kWarps;
      const bool is_val = a == 3 * n;
      wp[k] = is_val ? P + o.wv2 : P + o.wp2 + (a < 3 * n ? a : 0);
      ws[k] = is_val ? 1 : 3 * n;
      hrow[k] = act + (is_val ? g : 0) * tile + c;
    }
    double acc[4][CPL];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[k][q] = 0.0;
    for (int j = 0; j < g; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double wv = wp[k][j * ws[k]];
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[k][q] = __fma_rn(wv, hrow[k][j * tile + 32 * q], acc[k][q]);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < CPL; ++q) outv[pass][k][q] = acc[k][q];
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int a0 = w + pass * 4 * kWarps;
    if (a0 >= na) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = a0 + k * kWarps;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        if (a < 3 * n) act[a * tile + c + 32 * q] = kt::dadd(outv[pass][k][q], P[o.bp2 + a]);
        else if (a == 3 * n) val[c + 32 * q] = kt::dadd(outv[pass][k][q], P[o.bv2]);
      }
    }
  }
  __syncthreads();
}

using kt::Knob3;
using kt::softmax3;

template <bool SP, int CPL>
__global__ void __launch_bounds__(kThreads, 1) rollout_kernel(const __grid_constant__ RolloutLaunch L) {
  constexpr int tile = 32 * CPL;
  extern __shared__ __align__(16) double sm[];
  int ti = 0;
  while (ti + 1 < L.num_tasks && L.cta_base[ti + 1] <= (int)blockIdx.x) ++ti;
  const int64_t first = (int64_t)((int)blockIdx.x - L.cta_base[ti]) * tile;
  const RolloutTask* tkp = &L.task[ti];
  const int n = tkp->n, h = tkp->h, g = tkp->g, T = tkp->T;
  const int64_t E = tkp->E, eoff = tkp->episode_offset;
  const uint64_t seed = tkp->seed;
  uint16_t* __restrict__ out_idx = tkp->idx;
  int8_t* __restrict__ out_act = tkp->actions;
  double* __restrict__ out_logp = tkp->logp;
  double* __restrict__ out_val = tkp->value;
  const AcOff o = ac_layout(n, h, g);
  const double* P = tkp->params;
  if (SP) {
    for (int i = threadIdx.x; i < o.total; i += kThreads) sm[i] = P[i];
    P = sm;
  }
  double* act = sm + (SP ? ((o.total + 1) & ~1) : 0);  // 16-byte aligned (double2 loads)
  double* xb = act + act_rows(n, h, g) * tile;
  double* val = xb + n * tile;
  uint16_t* cfg = reinterpret_cast<uint16_t*>(val + tile);  // [d][e]
  int* card = reinterpret_cast<int*>(cfg + n * tile);
  const int c = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < n) card[threadIdx.x] = tkp->card[threadIdx.x];
  // initial configurations (trajectory row 0)
  for (int d = w; d < n; d += kWarps)
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int64_t e = first + c + 32 * q;
      uint16_t v = 0;
      if (e < E) {
        v = tkp->init_idx[e * n + d];
        out_idx[(e * tkp->sE) * n + d] = v;
      }
      cfg[d * tile + c + 32 * q] = v;
    }
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    // ---- 0: features x = idx / (card - 1) (design_space.cpp:195-197)
    for (int d = w; d < n; d += kWarps) {
      const int cd = card[d];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int e = c + 32 * q;
        xb[d * tile + e] = cd > 1 ? kt::ddiv((double)cfg[d * tile + e], (double)(cd - 1)) : 0.0;
      }
    }
    __syncthreads();
    forward_tile<CPL>(P, o, n, h, g, act, xb, val);
    // ---- D: per knob: log-softmax, counter-RNG draw, inverse CDF, saturating move
    for (int d = w; d < n; d += kWarps) {
      const int cd = card[d];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int el = c + 32 * q;
        const int64_t e = first + el;
        const Knob3 k3 = softmax3(act[(3 * d) * tile + el], act[(3 * d + 1) * tile + el],
                                  act[(3 * d + 2) * tile + el]);
        const uint64_t ge = (uint64_t)(eoff + e);
        const double u = kt::hash01(seed, (ge * (uint64_t)T + (uint64_t)t) * (uint64_t)n + (uint64_t)d);
        const int a = u < k3.p[0] ? 0 : (u < kt::dadd(k3.p[0], k3.p[1]) ? 1 : 2);
        int v = (int)cfg[d * tile + el] + (a - 1);
        v = v < 0 ? 0 : (v > cd - 1 ? cd - 1 : v);
        cfg[d * tile + el] = (uint16_t)v;
        act[(3 * d) * tile + el] = a == 0 ? k3.lp[0] : (a == 1 ? k3.lp[1] : k3.lp[2]);
        if (e < E) {
          if (out_act) out_act[(e * tkp->aE + t * tkp->aT) * n + d] = (int8_t)(a - 1);
          out_idx[(e * tkp->sE + (t + 1) * tkp->sT) * n + d] = (uint16_t)v;
        }
      }
    }
    __syncthreads();
    // ---- E: joint log-probability in knob order, value
    if (w < CPL) {
      const int el = c + 32 * w;
      const int64_t e = first + el;
      if (e < E) {
        double lp = 0.0;
        for (int d = 0; d < n; ++d) lp = kt::dadd(lp, act[(3 * d) * tile + el]);
        const int64_t o = e * tkp->aE + t * tkp->aT;
        if (out_logp) out_logp[o] = lp;
        if (out_val) out_val[o] = val[el];
        if (tkp->logp32) tkp->logp32[o] = (float)lp;
        if (tkp->value32) tkp->value32[o] = (float)val[el];
      }
    }
    __syncthreads();
  }
}

// ActorCritic::forward over arbitrary fp64 states (32-state tiles).
__global__ void __launch_bounds__(kThreads, 1)
ac_forward_kernel(const double* __restrict__ params, int n, int h, int g,
                  const double* __restrict__ states, int64_t B, double* __restrict__ log_probs,
                  double* __restrict__ probs, double* __restrict__ values, int smem_params) {
  constexpr int tile = 32;
  extern __shared__ __align__(16) double sm[];
  const AcOff o = ac_layout(n, h, g);
  const double* P = params;
  if (smem_params) {
    for (int i = threadIdx.x; i < o.total; i += kThreads) sm[i] = params[i];
    P = sm;
  }
  double* act = sm + (smem_params ? ((o.total + 1) & ~1) : 0);
  double* xb = act + act_rows(n, h, g) * tile;
  double* val = xb + n * tile;
  const int tid = threadIdx.x;
  for (int64_t first = (int64_t)blockIdx.x * tile; first < B; first += (int64_t)gridDim.x * tile) {
    __syncthreads();
    for (int item = tid; item < tile * n; item += kThreads) {
      const int c = item / n, d = item % n;
      xb[d * tile + c] = first + c < B ? states[(first + c) * n + d] : 0.0;
    }
    __syncthreads();
    forward_tile<1>(P, o, n, h, g, act, xb, val);
    for (int item = tid; item < tile * n; item += kThreads) {
      const int c = item % tile, d = item / tile;
      const int64_t b = first + c;
      if (b >= B) continue;
      const Knob3 k3 = softmax3(act[(3 * d) * tile + c], act[(3 * d + 1) * tile + c], act[(3 * d + 2) * tile + c]);
      for (int a = 0; a < 3; ++a) {
        if (log_probs) log_probs[b * 3 * n + 3 * d + a] = k3.lp[a];
        if (probs) probs[b * 3 * n + 3 * d + a] = k3.p[a];
      }
    }
    if (values && tid < tile && first + tid < B) values[first + tid] = val[tid];
  }
}

__global__ void debug_math_kernel(int op, const double* __restrict__ x, int64_t n,
                                  double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = op == 0 ? kt::kt_exp(x[i]) : (op == 1 ? kt::kt_log(x[i]) : kt::kt_tanh(x[i]));
}

// uint16 -> uint8 copy of trajectory rows [r0, r0 + rows) of every episode (idx_u8 outputs).
// fp32 copies of trajectory score rows [r0, r0 + len) of every episode (row pitch P).
__global__ void score_f32_kernel(const double* __restrict__ src, float* __restrict__ dst, int64_t E, int64_t P,
                                 int64_t r0, int64_t len) {
  const int64_t n = E * len;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = j / len, i = e * P + r0 + (j - e * len);
    dst[i] = (float)src[i];
  }
}

__global__ void narrow_idx_kernel(const uint16_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t E,
                                  int64_t rows_per_ep, int n, int64_t r0, int64_t rows) {
  const int64_t per = (int64_t)rows * n, total = E * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / per, j = (e * rows_per_ep + r0) * n + (i % per);
    dst[j] = (uint8_t)src[j];
  }
}

// Configuration ids id_of(Θ) (design_space.cpp:158-167: mixed radix, last knob fastest) of
// trajectory rows [r0, r0 + rows) of every episode (ids_u32 outputs; |space| <= 2^32).
struct IdRadix {
  int n;
  uint32_t card[kt::kMaxKnobs];
};
__global__ void ids_rows_kernel(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst, IdRadix rx, int64_t E,
                                int64_t rows_per_ep, int64_t r0, int64_t rows) {
  const int64_t total = E * rows;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / rows, r = e * rows_per_ep + r0 + (i - e * rows);
    const uint16_t* row = src + r * rx.n;
    uint32_t id = 0;
    if (rx.n == 8) {  // one 16-byte load per row
      const uint4 v = *reinterpret_cast<const uint4*>(row);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int d = 0; d < 8; ++d) id = id * rx.card[d] + ((w[d >> 1] >> (16 * (d & 1))) & 0xffffu);
    } else {
      for (int d = 0; d < rx.n; ++d) id = id * rx.card[d] + row[d];
    }
    dst[r] = id;
  }
}

// int8 directions -> 2-bit codes (direction + 1), 4 knobs per byte, for steps [t0, t0 + steps).
__global__ void pack_actions_kernel(const int8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t E, int64_t T,
                                    int n, int64_t t0, int64_t steps) {
  const int nb = (n + 3) / 4;
  const int64_t per = (int64_t)steps * nb, total = E * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / per, rem = i % per;
    const int64_t step = t0 + rem / nb;
    const int b = (int)(rem % nb);
    const int8_t* a = src + (e * T + step) * n;
    uint32_t v = 0;
    for (int j = 0; j < 4; ++j) {
      const int d = 4 * b + j;
      if (d < n) v |= (uint32_t)(a[d] + 1) << (2 * j);
    }
    dst[(e * T + step) * nb + b] = (uint8_t)v;
  }
}

// cuStreamWaitValue32 through the runtime's driver entry point (resolved once per context):
// the copy stream of a streamed rollout waits until the kernel's progress counter reaches a
// segment's count. False when the driver does not offer stream memory operations.
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
bool wait_value_available(ktune_ctx* ctx) {
  if (ctx->wait_value_state == 0) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    int ok = 0;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      ok = 1;
    cudaGetLastError();
    ctx->fn_wait_value = fn;
    ctx->wait_value_state = ok ? 1 : -1;
  }
  return ctx->wait_value_state == 1;
}
void wait_value_geq(ktune_ctx* ctx, cudaStream_t st, const unsigned int* addr, unsigned int v) {
  const CUresult r = reinterpret_cast<WaitValueFn>(ctx->fn_wait_value)((CUstream)st, (CUdeviceptr)addr, v,
                                                                      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) kt::fail(KTUNE_ERR_BACKEND, "rollout: cuStreamWaitValue32 failed");
}

bool fits_smem(int n, int h, int g, int cpl = 1) { return rollout_smem_bytes(n, h, g, true, cpl) <= 227 * 1024; }


void check_dims(int n, int h, int g) {
  if (n < 1 || n > kt::kMaxKnobs) kt::fail(KTUNE_ERR_CONFIG, "actor-critic: 1 <= num_knobs <= 32 on the device path");
  if (h < 8 || g < 8 || h % 8 || g % 8 || 2 * g > 2 * kWarps * kUnits || h > 1024)
    kt::fail(KTUNE_ERR_CONFIG, "actor-critic: device path needs hidden_dim, head_hidden multiples of 8, "
                               "head_hidden <= 128, hidden_dim <= 1024");
}

}  // namespace


extern "C" {

int64_t ktune_ac_num_params(int n, int h, int g) { return ac_layout(n, h, g).total; }

int ktune_ac_init_params(int n, int h, int g, uint64_t seed, double* p) {
  // Pinned init: one Rng(seed) stream; weights in flat-layout
  // order as normal()/sqrt(fan_in) (Box-Muller, rng.hpp:78-83); biases 0.
  return kt_guard(nullptr, [&] {
    const AcOff o = ac_layout(n, h, g);
    std::fill(p, p + o.total, 0.0);
    uint64_t st = seed;
    auto normal = [&]() {
      double u1 = (double)(kt::rng_next(st) >> 11) * 0x1.0p-53;
      const double u2 = (double)(kt::rng_next(st) >> 11) * 0x1.0p-53;
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    };
    const double s0 = 1.0 / std::sqrt((double)n), s1 = 1.0 / std::sqrt((double)h),
                 s2 = 1.0 / std::sqrt((double)g);
    for (int i = o.w0; i < o.b0; ++i) p[i] = normal() * s0;
    for (int i = o.wp1; i < o.bp1; ++i) p[i] = normal() * s1;
    for (int i = o.wp2; i < o.bp2; ++i) p[i] = normal() * s2;
    for (int i = o.wv1; i < o.bv1; ++i) p[i] = normal() * s1;
    for (int i = o.wv2; i < o.bv2; ++i) p[i] = normal() * s2;
  });
}

int ktune_ac_create(ktune_ctx* ctx, int n, int h, int g, const double* flat, ktune_ac** out) {
  return kt_guard(ctx, [&] {
    check_dims(n, h, g);
    auto* a = new ktune_ac();
    a->ctx = ctx;
    a->n = n;
    a->h = h;
    a->g = g;
    a->num_params = ac_layout(n, h, g).total;
    a->host_params.assign(flat, flat + a->num_params);
    cudaSetDevice(ctx->device);
    KT_CUDA(cudaMalloc(&a->d_params, sizeof(double) * a->num_params));
    KT_CUDA(cudaMemcpy(a->d_params, flat, sizeof(double) * a->num_params, cudaMemcpyHostToDevice));
    *out = a;
  });
}

int ktune_ac_destroy(ktune_ac* a) {
  if (!a) return KTUNE_OK;
  cudaFree(a->d_params);
  delete a;
  return KTUNE_OK;
}

int ktune_ac_forward(ktune_ctx* ctx, const ktune_ac* ac, const double* states, int64_t B,
                     double* log_probs, double* probs, double* values, int flags) {
  return kt_guard(ctx, [&] {
    if (B < 0) kt::fail(KTUNE_ERR_CONFIG, "negative batch");
    if (B == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const int n = ac->n;
    const double* d_s = (const double*)kt::stage_in(ctx, kt::WS_IN0, states, sizeof(double) * B * n, dev);
    double* d_lp = log_probs ? (double*)kt::out_buf(ctx, kt::WS_OUT0, log_probs, sizeof(double) * B * 3 * n, dev) : nullptr;
    double* d_p = probs ? (double*)kt::out_buf(ctx, kt::WS_OUT1, probs, sizeof(double) * B * 3 * n, dev) : nullptr;
    double* d_v = values ? (double*)kt::out_buf(ctx, kt::WS_OUT2, values, sizeof(double) * B, dev) : nullptr;
    const bool sp = fits_smem(n, ac->h, ac->g);
    const size_t smem = rollout_smem_bytes(n, ac->h, ac->g, sp, 1);
    KT_CUDA(cudaFuncSetAttribute(ac_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>(kt::ceil_div(B, 32), kt::sm_count(ctx));
    ac_forward_kernel<<<grid, kThreads, smem, ctx->stream>>>(ac->d_params, n, ac->h, ac->g, d_s, B, d_lp,
                                                             d_p, d_v, sp ? 1 : 0);
    kt::check_launch(ctx, "ac_forward");
    if (d_lp) kt::stage_out(ctx, log_probs, d_lp, sizeof(double) * B * 3 * n, dev);
    if (d_p) kt::stage_out(ctx, probs, d_p, sizeof(double) * B * 3 * n, dev);
    if (d_v) kt::stage_out(ctx, values, d_v, sizeof(double) * B, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_debug_math(ktune_ctx* ctx, int op, const double* x, int64_t n, double* out) {
  return kt_guard(ctx, [&] {
    if (n <= 0) return;
    const double* d_x = (const double*)kt::stage_in(ctx, kt::WS_IN0, x, sizeof(double) * n, false);
    double* d_o = (double*)kt::out_buf(ctx, kt::WS_OUT0, out, sizeof(double) * n, false);
    debug_math_kernel<<<(int)std::min<int64_t>(kt::ceil_div(n, 256), 4096), 256, 0, ctx->stream>>>(op, d_x, n, d_o);
    kt::check_launch(ctx, "debug_math");
    kt::stage_out(ctx, out, d_o, sizeof(double) * n, false);
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_rollout(ktune_ctx* ctx, int num_tasks, const ktune_rollout_task* tasks, int32_t T,
                  int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_rollout");
    if (num_tasks < 0 || T < 0) kt::fail(KTUNE_ERR_CONFIG, "rollout: bad task count or steps");
    if (num_tasks == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const bool grouped = flags & KTUNE_F_STEP_MAJOR_GROUPED;  // one step-major array over all tasks' episodes
    const bool stepm = grouped || (flags & KTUNE_F_STEP_MAJOR);  // [T+1][E] / [T][E] instead of [E][T+1] / [E][T]
    std::vector<RolloutTask> dt(num_tasks);
    // grouped: task k's episodes are columns [goff[k], goff[k] + E_k) of ONE step-major array of
    // Etot columns per output, so every step (and every segment) of all tasks is contiguous
    std::vector<int64_t> goff(num_tasks + 1, 0);
    for (int k = 0; k < num_tasks; ++k) goff[k + 1] = goff[k] + std::max<int64_t>(0, tasks[k].num_episodes);
    const int64_t Etot = goff[num_tasks];
    // per output kind (idx, score, actions, logp, value, logp32, value32, idx8, actions2, score32, ids32):
    // the tasks that request it form one contiguous run [lo, hi] whose columns are a W-wide
    // step-major array at the host pointer of task lo (task k at column goff[k] - goff[lo])
    struct GKind {
      int lo = -1, hi = -1;
      int64_t W = 0;
      void* host = nullptr;
      size_t rb = 0;  // bytes per row element (per episode column)
    };
    constexpr int kKinds = 11;
    std::array<GKind, kKinds> gk{};
    auto kind_ptr = [&](const ktune_rollout_task& t, int q) -> void* {
      void* const v[kKinds] = {t.idx,  t.score,    t.actions,    t.logp,      t.value,  t.logp_f32,
                               t.value_f32, t.idx_u8, t.actions_u2, t.score_f32, t.ids_u32};
      return v[q];
    };
    if (grouped) {
      for (int k = 1; k < num_tasks; ++k)
        if (!tasks[k].ac || !tasks[0].ac || tasks[k].ac->n != tasks[0].ac->n)
          kt::fail(KTUNE_ERR_CONFIG, "rollout: grouped layout needs the same knob count in every task");
      const int64_t n = tasks[0].ac ? tasks[0].ac->n : 0;
      const size_t rbs[kKinds] = {(size_t)(2 * n), 8, (size_t)n, 8, 8, 4, 4, (size_t)n, (size_t)((n + 3) / 4), 4, 4};
      for (int q = 0; q < kKinds; ++q) {
        GKind& g = gk[q];
        g.rb = rbs[q];
        for (int k = 0; k < num_tasks; ++k) {
          void* pk = kind_ptr(tasks[k], q);
          if (!pk) continue;
          if (g.lo < 0) {
            g.lo = k;
            g.host = pk;
          } else if (g.hi != k - 1 || (char*)pk != (char*)g.host + (goff[k] - goff[g.lo]) * (int64_t)g.rb) {
            kt::fail(KTUNE_ERR_CONFIG, "rollout: grouped layout needs each output's tasks contiguous, every task "
                                       "at its episode offset of the first one's array");
          }
          g.hi = k;
        }
        if (g.lo >= 0) g.W = goff[g.hi + 1] - goff[g.lo];
        if (dev && g.lo >= 0 && g.W != Etot)  // device pointers: the kernel writes Etot-wide rows
          kt::fail(KTUNE_ERR_CONFIG, "rollout: grouped device outputs must be requested by every task");
      }
    }
    struct HostIo {
      const uint16_t* d_init;
      uint16_t* d_idx;
      int8_t* d_act;
      double* d_logp;
      double* d_val;
      double* d_score;
      float* d_logp32;
      float* d_val32;
      uint8_t* d_u8;
      uint8_t* d_a2;
      float* d_s32;
      uint32_t* d_ids;
    };
    std::vector<HostIo> io(num_tasks);
    bool smem_params = true;
    size_t arena = 0;
    auto slice = [&](size_t bytes) {
      const size_t o = arena;
      arena += (std::max<size_t>(bytes, 8) + 255) & ~(size_t)255;
      return o;
    };
    std::vector<std::array<size_t, 12>> offs(num_tasks);
    for (int k = 0; k < num_tasks; ++k) {
      const ktune_rollout_task& t = tasks[k];
      if (!t.space || !t.ac) kt::fail(KTUNE_ERR_CONFIG, "rollout: task needs a space and an agent");
      if (t.ac->n != t.space->D) kt::fail(KTUNE_ERR_CONFIG, "rollout: agent/space knob count mismatch");
      if (t.gbt && t.gbt->num_features != t.space->D) kt::fail(KTUNE_ERR_CONFIG, "rollout: cost model/space mismatch");
      if (t.num_episodes < 0 || (!t.idx && (dev || (!t.idx_u8 && !t.ids_u32))))
        kt::fail(KTUNE_ERR_CONFIG, "rollout: bad episode count or missing idx output");
      if (t.actions_u2 && dev && !t.actions)
        kt::fail(KTUNE_ERR_CONFIG, "rollout: device-pointer calls need actions alongside actions_u2");
      if (t.score_f32 && dev && !t.score)
        kt::fail(KTUNE_ERR_CONFIG, "rollout: device-pointer calls need score alongside score_f32");
      if (t.idx_u8)
        for (int c : t.space->card)
          if (c > 256) kt::fail(KTUNE_ERR_CONFIG, "rollout: idx_u8 needs every knob cardinality <= 256");
      if (t.ids_u32) {
        double sz = 1;
        for (int c : t.space->card) sz *= c;
        if (sz > 4294967296.0) kt::fail(KTUNE_ERR_CONFIG, "rollout: ids_u32 needs a design space of at most 2^32 configurations");
      }
      smem_params = smem_params && fits_smem(t.ac->n, t.ac->h, t.ac->g);
      if (!dev && !grouped) {
        const size_t E = (size_t)t.num_episodes, n = (size_t)t.ac->n;
        offs[k] = {slice(E * n * 2), slice(E * (T + 1) * n * 2), (t.actions || t.actions_u2) ? slice(E * T * n) : SIZE_MAX,
                   t.logp ? slice(E * T * 8) : SIZE_MAX, t.value ? slice(E * T * 8) : SIZE_MAX,
                   (t.score || t.score_f32) ? slice(E * (T + 1) * 8) : SIZE_MAX, t.logp_f32 ? slice(E * T * 4) : SIZE_MAX,
                   t.value_f32 ? slice(E * T * 4) : SIZE_MAX, t.idx_u8 ? slice(E * (T + 1) * n) : SIZE_MAX,
                   t.actions_u2 ? slice(E * T * ((n + 3) / 4)) : SIZE_MAX,
                   t.score_f32 ? slice(E * (T + 1) * 4) : SIZE_MAX, t.ids_u32 ? slice(E * (T + 1) * 4) : SIZE_MAX};
      }
    }
    if (!dev && grouped && num_tasks > 0) {  // one Etot-wide slice per output any task requests
      const size_t E = (size_t)Etot, n = (size_t)tasks[0].ac->n;
      auto any = [&](int q) { return gk[q].lo >= 0; };
      offs[0] = {slice(E * n * 2), slice(E * (T + 1) * n * 2), (any(2) || any(8)) ? slice(E * T * n) : SIZE_MAX,
                 any(3) ? slice(E * T * 8) : SIZE_MAX, any(4) ? slice(E * T * 8) : SIZE_MAX,
                 (any(1) || any(9)) ? slice(E * (T + 1) * 8) : SIZE_MAX, any(5) ? slice(E * T * 4) : SIZE_MAX,
                 any(6) ? slice(E * T * 4) : SIZE_MAX, any(7) ? slice(E * (T + 1) * n) : SIZE_MAX,
                 any(8) ? slice(E * T * ((n + 3) / 4)) : SIZE_MAX, any(9) ? slice(E * (T + 1) * 4) : SIZE_MAX,
                 any(10) ? slice(E * (T + 1) * 4) : SIZE_MAX};
    }
    unsigned char* base = dev ? nullptr : (unsigned char*)ctx->dev(kt::WS_ROLLOUT, std::max<size_t>(arena, 256));
    auto at = [&](size_t o) { return o == SIZE_MAX ? nullptr : (void*)(base + o); };
    for (int k = 0; k < num_tasks; ++k) {
      const ktune_rollout_task& t = tasks[k];
      const int n = t.ac->n;
      const int64_t E = t.num_episodes;
      HostIo& h = io[k];
      if (dev) {
        h = {t.init_idx, t.idx,    t.actions,    t.logp,      t.value,  t.score,
             t.logp_f32, t.value_f32, t.idx_u8, t.actions_u2, t.score_f32, t.ids_u32};
      } else if (grouped) {  // task 0's slices, shifted to this task's episode columns
        const int64_t o = goff[k];
        auto sh = [&](size_t off, int64_t per_row) -> unsigned char* {
          return off == SIZE_MAX ? nullptr : (unsigned char*)at(off) + o * per_row;
        };
        h = {(const uint16_t*)sh(offs[0][0], 2 * n), (uint16_t*)sh(offs[0][1], 2 * n), (int8_t*)sh(offs[0][2], n),
             (double*)sh(offs[0][3], 8),             (double*)sh(offs[0][4], 8),       (double*)sh(offs[0][5], 8),
             (float*)sh(offs[0][6], 4),              (float*)sh(offs[0][7], 4),        (uint8_t*)sh(offs[0][8], n),
             (uint8_t*)sh(offs[0][9], (n + 3) / 4),  (float*)sh(offs[0][10], 4),       (uint32_t*)sh(offs[0][11], 4)};
        if (E > 0)
          KT_CUDA(cudaMemcpyAsync((void*)h.d_init, t.init_idx, (size_t)E * n * 2, cudaMemcpyHostToDevice, ctx->stream));
      } else {
        h = {(const uint16_t*)at(offs[k][0]), (uint16_t*)at(offs[k][1]), (int8_t*)at(offs[k][2]),
             (double*)at(offs[k][3]),         (double*)at(offs[k][4]),   (double*)at(offs[k][5]),
             (float*)at(offs[k][6]),          (float*)at(offs[k][7]),    (uint8_t*)at(offs[k][8]),
             (uint8_t*)at(offs[k][9]),        (float*)at(offs[k][10]),   (uint32_t*)at(offs[k][11])};
        if (E > 0)
          KT_CUDA(cudaMemcpyAsync((void*)h.d_init, t.init_idx, (size_t)E * n * 2, cudaMemcpyHostToDevice, ctx->stream));
      }
      RolloutTask& r = dt[k];
      for (int d = 0; d < kt::kMaxKnobs; ++d) r.card[d] = d < n ? t.space->card[d] : 1;
      r.params = t.ac->d_params;
      r.n = n;
      r.h = t.ac->h;
      r.g = t.ac->g;
      r.T = T;
      r.E = E;
      r.episode_offset = t.episode_offset;
      r.seed = t.explore_seed;
      r.init_idx = h.d_init;
      r.idx = h.d_idx;
      r.actions = h.d_act;
      r.logp = h.d_logp;
      r.value = h.d_val;
      r.logp32 = h.d_logp32;
      r.value32 = h.d_val32;
      r.sE = stepm ? 1 : (int64_t)T + 1;
      r.sT = stepm ? (grouped ? Etot : E) : 1;
      r.aE = stepm ? 1 : (int64_t)T;
      r.aT = stepm ? (grouped ? Etot : E) : 1;
    }
    // tcgen05 path with certified sampling unless the exact fp64 forward is
    // requested (or a task is outside the tensor-core path's shapes)
    bool use_tc = !(flags & KTUNE_F_EXACT_ROLLOUT);
    for (int k = 0; k < num_tasks && use_tc; ++k) use_tc = kt::rollout_tc_eligible(tasks[k].ac, tasks[k].space);
    // Host outputs on the tcgen05 path: the episode runs in S segments of
    // steps; each segment's scoring and device->host copies (copy stream)
    // overlap the next segment's compute, so the end-to-end call approaches
    // max(compute, PCIe) instead of their sum.
    bool segmented = use_tc && !dev && T >= 128;
    for (int k = 0; k < num_tasks && segmented; ++k)
      if (tasks[k].gbt && (tasks[k].score || tasks[k].score_f32) && !tasks[k].gbt->d_inode_pk) segmented = false;
    if (ctx->opt_rollout_segments == 1) segmented = false;
    const int S = !segmented ? 1
                  : ctx->opt_rollout_segments > 1 ? (int)std::min<int64_t>(ctx->opt_rollout_segments, T)
                                                  : (int)std::min<int64_t>(16, std::max<int64_t>(2, T / 40));
    if (segmented && !ctx->copy_stream) KT_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> events;
    std::vector<kt::GbtJob> jobs;
    auto score_rows = [&](int k, int r0, int r1) {  // queue trajectory rows [r0, r1] of every episode
      const ktune_rollout_task& t = tasks[k];
      if (!t.gbt || !io[k].d_score || t.num_episodes == 0) return;
      const int64_t len = r1 - r0 + 1, E = t.num_episodes;
      if (grouped) {  // this task's columns of rows r0..r1: blocks of E every Etot
        jobs.push_back({t.gbt, io[0].d_idx, E * len, io[0].d_score, kt::RowMap{E, Etot, r0 * Etot + goff[k]}});
      } else if (stepm) {  // rows r0..r1 of every episode are one contiguous block
        jobs.push_back({t.gbt, io[k].d_idx + r0 * E * t.ac->n, E * len, io[k].d_score + r0 * E, kt::RowMap()});
      } else {
        kt::RowMap m;
        if (len != T + 1) m = kt::RowMap{len, (int64_t)T + 1, r0};
        jobs.push_back({t.gbt, io[k].d_idx, E * len, io[k].d_score, m});
      }
    };
    auto flush_scores = [&]() {  // every queued task in one K1 launch
      kt::gbt_predict_idx_device_multi(ctx, jobs, 2);
      jobs.clear();
    };
    auto score32_rows = [&](int k, int r0, int r1) {  // fp32 copies of the scores of rows [r0, r1]
      const ktune_rollout_task& t = tasks[k];
      if (grouped) {  // one flat pass over every task's columns (task 0's pointers are the slice starts)
        if (k > 0 || gk[9].lo < 0 || Etot == 0) return;
      } else if (!t.gbt || !io[k].d_s32 || t.num_episodes == 0) {
        return;
      }
      const int64_t len = r1 - r0 + 1, E = grouped ? Etot : t.num_episodes, work = E * len;
      // step-major: one flat range [r0*E, (r1+1)*E) of a single "episode"
      score_f32_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(work, 256), (int64_t)kt::sm_count(ctx) * 16), 256, 0,
                         ctx->stream>>>(io[k].d_score, io[k].d_s32, stepm ? 1 : E, T + 1, stepm ? r0 * E : r0,
                                        stepm ? len * E : len);
      kt::check_launch(ctx, "score_f32");
    };
    auto narrow_rows = [&](int k, int r0, int r1) {  // uint16 -> uint8 trajectory rows [r0, r1]
      const ktune_rollout_task& t = tasks[k];
      if (grouped ? (k > 0 || gk[7].lo < 0 || Etot == 0) : (!t.idx_u8 || t.num_episodes == 0)) return;
      const int64_t E = grouped ? Etot : t.num_episodes;
      narrow_idx_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(E * (int64_t)(r1 - r0 + 1) * t.ac->n, 256),
                                                     (int64_t)kt::sm_count(ctx) * 16),
                          256, 0, ctx->stream>>>(io[k].d_idx, io[k].d_u8, stepm ? 1 : E, T + 1,
                                                 t.ac->n, stepm ? r0 * E : r0,
                                                 stepm ? (r1 - r0 + 1) * E : r1 - r0 + 1);
      kt::check_launch(ctx, "narrow_idx");
    };
    auto ids_rows = [&](int k, int r0, int r1) {  // configuration ids of trajectory rows [r0, r1]
      const ktune_rollout_task& t = tasks[k];
      if (t.num_episodes == 0 || (grouped ? (k < gk[10].lo || k > gk[10].hi) : !t.ids_u32)) return;
      const int64_t E = t.num_episodes, len = r1 - r0 + 1;
      IdRadix rx{};  // per task: the radix is the task's own space
      rx.n = t.ac->n;
      for (int d = 0; d < rx.n; ++d) rx.card[d] = (uint32_t)t.space->card[d];
      // (outer, inner, outer pitch, first): grouped = rows of this task's E columns every Etot;
      // step-major = one flat block; episode-major = rows [r0, r1] of every episode
      const int64_t outer = grouped ? len : stepm ? 1 : E, inner = grouped ? E : stepm ? len * E : len;
      const int64_t pitch = grouped ? Etot : T + 1, first = grouped ? r0 * Etot : stepm ? r0 * E : r0;
      ids_rows_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(E * len, 256), (int64_t)kt::sm_count(ctx) * 16), 256,
                        0, ctx->stream>>>(io[k].d_idx, io[k].d_ids, rx, outer, pitch, first, inner);
      kt::check_launch(ctx, "ids_rows");
    };
    auto pack_steps = [&](int k, int t0, int t1) {  // int8 -> 2-bit actions of steps [t0, t1)
      const ktune_rollout_task& t = tasks[k];
      if (t1 <= t0 || (grouped ? (k > 0 || gk[8].lo < 0 || Etot == 0) : (!t.actions_u2 || t.num_episodes == 0)))
        return;
      const int64_t E = grouped ? Etot : t.num_episodes;
      const int64_t work = E * (int64_t)(t1 - t0) * ((t.ac->n + 3) / 4);
      pack_actions_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(work, 256), (int64_t)kt::sm_count(ctx) * 16), 256,
                            0, ctx->stream>>>(io[k].d_act, io[k].d_a2, stepm ? 1 : E, T, t.ac->n,
                                              stepm ? (int64_t)t0 * E : t0, stepm ? (int64_t)(t1 - t0) * E : t1 - t0);
      kt::check_launch(ctx, "pack_actions");
    };
    // steps [t0, t1): rows (t0, t1] (+ row 0); what: 1 the trajectory, 2 the scores, 3 both
    auto copy_out = [&](int k, int t0, int t1, cudaStream_t st, int what) {
      const ktune_rollout_task& t = tasks[k];
      const bool traj = what & 1, scores = what & 2;
      if (grouped) {  // once for every task: per output, the W columns of its task run in one copy
        if (k > 0) return;
        const int r0 = t0 == 0 ? 0 : t0 + 1;
        const int64_t nr[kKinds] = {t1 - r0 + 1, t1 - r0 + 1, t1 - t0,     t1 - t0, t1 - t0,     t1 - t0,
                                    t1 - t0,     t1 - r0 + 1, t1 - t0,     t1 - r0 + 1, t1 - r0 + 1};
        const int64_t first[kKinds] = {r0, r0, t0, t0, t0, t0, t0, r0, t0, r0, r0};
        const void* dsrc[kKinds] = {io[0].d_idx,   io[0].d_score, io[0].d_act, io[0].d_logp, io[0].d_val, io[0].d_logp32,
                                    io[0].d_val32, io[0].d_u8,    io[0].d_a2,  io[0].d_s32,  io[0].d_ids};
        for (int q = 0; q < kKinds; ++q) {
          const GKind& g = gk[q];
          if (g.lo < 0 || g.W == 0 || nr[q] <= 0 || !dsrc[q]) continue;
          if ((q == 1 || q == 9) && (!tasks[g.lo].gbt || !scores)) continue;
          if (q != 1 && q != 9 && !traj) continue;
          const size_t spitch = (size_t)Etot * g.rb, dpitch = (size_t)g.W * g.rb, width = dpitch;
          const char* src = (const char*)dsrc[q] + (size_t)first[q] * spitch + (size_t)goff[g.lo] * g.rb;
          char* dst = (char*)g.host + (size_t)first[q] * dpitch;
          if (spitch == dpitch)
            KT_CUDA(cudaMemcpyAsync(dst, src, width * (size_t)nr[q], cudaMemcpyDeviceToHost, st));
          else
            KT_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, (size_t)nr[q], cudaMemcpyDeviceToHost, st));
        }
        return;
      }
      const size_t E = (size_t)t.num_episodes, n = (size_t)t.ac->n;
      if (E == 0) return;
      const HostIo& h = io[k];
      const int r0 = t0 == 0 ? 0 : t0 + 1;
      const size_t rows = (size_t)(t1 - r0 + 1), steps = (size_t)(t1 - t0);
      if (stepm) {  // every output's segment is one contiguous block: 1-D copies
        auto cp = [&](void* dst, const void* src, size_t off, size_t bytes, bool is_score = false) {
          if (dst && bytes && (is_score ? scores : traj))
            KT_CUDA(cudaMemcpyAsync((char*)dst + off, (const char*)src + off, bytes, cudaMemcpyDeviceToHost, st));
        };
        const size_t nb = (n + 3) / 4;
        cp(t.idx, h.d_idx, r0 * E * n * 2, rows * E * n * 2);
        cp(t.idx_u8, h.d_u8, r0 * E * n, rows * E * n);
        cp(t.ids_u32, h.d_ids, r0 * E * 4, rows * E * 4);
        cp(t.actions, h.d_act, t0 * E * n, steps * E * n);
        cp(t.actions_u2, h.d_a2, t0 * E * nb, steps * E * nb);
        cp(t.logp, h.d_logp, t0 * E * 8, steps * E * 8);
        cp(t.value, h.d_val, t0 * E * 8, steps * E * 8);
        cp(t.logp_f32, h.d_logp32, t0 * E * 4, steps * E * 4);
        cp(t.value_f32, h.d_val32, t0 * E * 4, steps * E * 4);
        if (t.gbt) {
          cp(t.score, h.d_score, r0 * E * 8, rows * E * 8, true);
          cp(t.score_f32, h.d_s32, r0 * E * 4, rows * E * 4, true);
        }
        return;
      }
      if (traj && t.idx)
        KT_CUDA(cudaMemcpy2DAsync(t.idx + r0 * n, (T + 1) * n * 2, h.d_idx + r0 * n, (T + 1) * n * 2, rows * n * 2,
                                  E, cudaMemcpyDeviceToHost, st));
      if (traj && t.idx_u8)
        KT_CUDA(cudaMemcpy2DAsync(t.idx_u8 + r0 * n, (T + 1) * n, h.d_u8 + r0 * n, (T + 1) * n, rows * n, E,
                                  cudaMemcpyDeviceToHost, st));
      if (traj && t.ids_u32)
        KT_CUDA(cudaMemcpy2DAsync(t.ids_u32 + r0, (T + 1) * 4, h.d_ids + r0, (T + 1) * 4, rows * 4, E,
                                  cudaMemcpyDeviceToHost, st));
      if (traj && t.actions && steps)
        KT_CUDA(cudaMemcpy2DAsync(t.actions + t0 * n, T * n, h.d_act + t0 * n, T * n, steps * n, E,
                                  cudaMemcpyDeviceToHost, st));
      if (traj && t.actions_u2 && steps) {
        const size_t nb = (n + 3) / 4;
        KT_CUDA(cudaMemcpy2DAsync(t.actions_u2 + t0 * nb, T * nb, h.d_a2 + t0 * nb, T * nb, steps * nb, E,
                                  cudaMemcpyDeviceToHost, st));
      }
      if (traj && t.logp && steps)
        KT_CUDA(cudaMemcpy2DAsync(t.logp + t0, T * 8, h.d_logp + t0, T * 8, steps * 8, E, cudaMemcpyDeviceToHost, st));
      if (traj && t.value && steps)
        KT_CUDA(cudaMemcpy2DAsync(t.value + t0, T * 8, h.d_val + t0, T * 8, steps * 8, E, cudaMemcpyDeviceToHost, st));
      if (traj && t.logp_f32 && steps)
        KT_CUDA(cudaMemcpy2DAsync(t.logp_f32 + t0, T * 4, h.d_logp32 + t0, T * 4, steps * 4, E,
                                  cudaMemcpyDeviceToHost, st));
      if (traj && t.value_f32 && steps)
        KT_CUDA(cudaMemcpy2DAsync(t.value_f32 + t0, T * 4, h.d_val32 + t0, T * 4, steps * 4, E,
                                  cudaMemcpyDeviceToHost, st));
      if (scores && t.score && t.gbt)
        KT_CUDA(cudaMemcpy2DAsync(t.score + r0, (T + 1) * 8, h.d_score + r0, (T + 1) * 8, rows * 8, E,
                                  cudaMemcpyDeviceToHost, st));
      if (scores && t.score_f32 && t.gbt)
        KT_CUDA(cudaMemcpy2DAsync(t.score_f32 + r0, (T + 1) * 4, h.d_s32 + r0, (T + 1) * 4, rows * 4, E,
                                  cudaMemcpyDeviceToHost, st));
    };
    std::vector<char> scored(num_tasks, 0);
    if (use_tc) {
      std::vector<kt::RolloutWork> work(num_tasks);
      for (int k = 0; k < num_tasks; ++k)
        work[k] = {tasks[k].space, tasks[k].ac, dt[k].E,     dt[k].episode_offset, dt[k].seed, dt[k].init_idx,
                   dt[k].idx,      dt[k].actions, dt[k].logp, dt[k].value,         tasks[k].gbt, io[k].d_score,
                   io[k].d_logp32, io[k].d_val32};
      for (int k = 0; k < num_tasks; ++k) {
        work[k].sE = dt[k].sE;
        work[k].sT = dt[k].sT;
        work[k].aE = dt[k].aE;
        work[k].aT = dt[k].aT;
      }
      // Streamed (default for host buffers): ONE rollout launch; each slot publishes the segments
      // it has finished in device memory and the copy stream waits on that counter
      // (cuStreamWaitValue32), copying every finished segment of the trajectory (ids / idx, actions,
      // logp, value, in the compact encodings the kernel writes itself) while the kernel runs on.
      // The cost model then scores the whole trajectory in a few row chunks whose score copies
      // overlap the next chunk's scoring.
      const bool streamed = segmented && ctx->opt_rollout_streamed != 1 && !ctx->opt_rollout_fuse_gbt &&
                            wait_value_available(ctx);
      if (streamed) {
        const int SS = ctx->opt_rollout_segments > 1 ? (int)std::min<int64_t>(ctx->opt_rollout_segments, T)
                                                     : (int)std::min<int64_t>(32, std::max<int64_t>(2, T / 25));
        auto in_run = [&](int q, int k, bool own) { return grouped ? (k >= gk[q].lo && k <= gk[q].hi) : own; };
        for (int k = 0; k < num_tasks; ++k) {  // the kernel writes the compact encodings directly
          const ktune_rollout_task& t = tasks[k];
          work[k].idx8 = in_run(7, k, t.idx_u8 != nullptr) ? io[k].d_u8 : nullptr;
          work[k].act2 = in_run(8, k, t.actions_u2 != nullptr) ? io[k].d_a2 : nullptr;
          work[k].ids = in_run(10, k, t.ids_u32 != nullptr) ? io[k].d_ids : nullptr;
          if (!in_run(2, k, t.actions != nullptr)) work[k].actions = nullptr;  // int8 directions not requested
        }
        constexpr int kMaxSegs = 64;
        if (!ctx->d_progress) KT_CUDA(cudaMalloc(&ctx->d_progress, kMaxSegs * sizeof(unsigned int)));
        if (SS > kMaxSegs || (int64_t)T * SS >= (1ll << 31))
          kt::fail(KTUNE_ERR_CONFIG, "rollout: at most 64 streamed segments and T x segments < 2^31");
        KT_CUDA(cudaMemsetAsync(ctx->d_progress, 0, SS * sizeof(unsigned int), ctx->stream));
        auto fence = [&](cudaStream_t from, cudaStream_t to) {
          cudaEvent_t ev;
          KT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          events.push_back(ev);
          KT_CUDA(cudaEventRecord(ev, from));
          KT_CUDA(cudaStreamWaitEvent(to, ev, 0));
        };
        fence(ctx->stream, ctx->copy_stream);  // the counter is reset before any wait reads it
        int64_t slots = 0;
        {
          kt::ProfScope prof(ctx, KTUNE_STAT_ROLLOUT_NS);
          slots = kt::rollout_tc(ctx, work, T, 0, T, ctx->d_progress, SS);
        }
        // Once the rollout is done every wait is satisfied, whatever the count, so no wait can hang.
        // The driver's GEQ test is cyclic ((int32_t)(*addr - v) >= 0): the release value 0x7F7F7F7F
        // passes every wait value v <= 0x7F7F7F7F and no count reached before it does.
        constexpr unsigned int kRelease = 0x7F7F7F7Fu;
        KT_CUDA(cudaMemsetAsync(ctx->d_progress, 0x7F, SS * sizeof(unsigned int), ctx->stream));
        if (slots >= (int64_t)kRelease) kt::fail(KTUNE_ERR_CONFIG, "rollout: too many slots");
        for (int sg = 0; sg < SS; ++sg) {
          const int t0 = (int)(((int64_t)sg * T + SS - 1) / SS), t1 = (int)(((int64_t)(sg + 1) * T + SS - 1) / SS);
          if (t1 <= t0) continue;
          // the last segment is never counted by the kernel: its copies follow the release
          wait_value_geq(ctx, ctx->copy_stream, ctx->d_progress + sg, sg + 1 < SS ? (unsigned int)slots : kRelease);
          for (int k = 0; k < num_tasks; ++k) copy_out(k, t0, t1, ctx->copy_stream, 1);
        }
        const int C = (int)std::min<int64_t>(4, T);  // score chunks (2..8 and 10..32 segments measured within noise)
        for (int c = 0; c < C; ++c) {
          const int t0 = (int)((int64_t)c * T / C), t1 = (int)((int64_t)(c + 1) * T / C);
          const int r0 = t0 == 0 ? 0 : t0 + 1;
          for (int k = 0; k < num_tasks; ++k) score_rows(k, r0, t1);
          flush_scores();
          for (int k = 0; k < num_tasks; ++k) score32_rows(k, r0, t1);
          fence(ctx->stream, ctx->copy_stream);
          for (int k = 0; k < num_tasks; ++k) copy_out(k, t0, t1, ctx->copy_stream, 2);
        }
        KT_CUDA(cudaStreamSynchronize(ctx->copy_stream));
        for (cudaEvent_t ev : events) cudaEventDestroy(ev);
        KT_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
      }
      if (segmented) {
        for (int sg = 0; sg < S; ++sg) {
          const int t0 = (int)((int64_t)sg * T / S), t1 = (int)((int64_t)(sg + 1) * T / S);
          {
            kt::ProfScope prof(ctx, KTUNE_STAT_ROLLOUT_NS);
            kt::rollout_tc(ctx, work, T, t0, t1);
          }
          for (int k = 0; k < num_tasks; ++k) score_rows(k, t0 == 0 ? 0 : t0 + 1, t1);
          flush_scores();
          for (int k = 0; k < num_tasks; ++k) {  // after every task's scores (grouped: one pass for all)
            score32_rows(k, t0 == 0 ? 0 : t0 + 1, t1);
            narrow_rows(k, t0 == 0 ? 0 : t0 + 1, t1);
            ids_rows(k, t0 == 0 ? 0 : t0 + 1, t1);
            pack_steps(k, t0, t1);
          }
          cudaEvent_t ev;
          KT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          events.push_back(ev);
          KT_CUDA(cudaEventRecord(ev, ctx->stream));
          KT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev, 0));
          for (int k = 0; k < num_tasks; ++k) copy_out(k, t0, t1, ctx->copy_stream, 3);
        }
        KT_CUDA(cudaStreamSynchronize(ctx->copy_stream));
        for (cudaEvent_t ev : events) cudaEventDestroy(ev);
        KT_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
      }
      kt::ProfScope prof(ctx, KTUNE_STAT_ROLLOUT_NS);
      kt::rollout_tc(ctx, work, T, 0, T);
      for (int k = 0; k < num_tasks; ++k) scored[k] = work[k].scored;
    } else {
      // exact path: one launch config for all tasks: smem sized for the largest task;
      // 64-episode tiles (2 per lane) when they fit, else 32
      int cpl = 2;
      for (int k = 0; k < num_tasks; ++k)
        if (!smem_params || rollout_smem_bytes(dt[k].n, dt[k].h, dt[k].g, true, 2) > 227 * 1024 || 2 * dt[k].g > 128)
          cpl = 1;
      size_t smem = 0;
      for (int k = 0; k < num_tasks; ++k)
        smem = std::max(smem, rollout_smem_bytes(dt[k].n, dt[k].h, dt[k].g, smem_params, cpl));
      if (smem > 227 * 1024) kt::fail(KTUNE_ERR_CONFIG, "rollout: agent too large for shared memory");
      auto kern = smem_params ? (cpl == 2 ? rollout_kernel<true, 2> : rollout_kernel<true, 1>)
                              : rollout_kernel<false, 1>;
      KT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kt::ProfScope prof(ctx, KTUNE_STAT_ROLLOUT_NS);
      for (int t0 = 0; t0 < num_tasks; t0 += kMaxTasksPerLaunch) {  // grouped launches
        RolloutLaunch L{};
        L.num_tasks = std::min(kMaxTasksPerLaunch, num_tasks - t0);
        int ctas = 0;
        for (int q = 0; q < L.num_tasks; ++q) {
          L.task[q] = dt[t0 + q];
          L.cta_base[q] = ctas;
          ctas += (int)kt::ceil_div(dt[t0 + q].E, 32 * cpl);
        }
        L.cta_base[L.num_tasks] = ctas;
        if (ctas > 0) kern<<<(unsigned)ctas, kThreads, smem, ctx->stream>>>(L);
      }
      kt::check_launch(ctx, "rollout");
    }
    // cost-model scores of every visited configuration (K1 over the trajectory)
    for (int k = 0; k < num_tasks; ++k)
      if (!scored[k]) score_rows(k, 0, T);
    flush_scores();
    for (int k = 0; k < num_tasks; ++k) {  // after every task's scores (grouped: one pass for all)
      score32_rows(k, 0, T);
      narrow_rows(k, 0, T);
      ids_rows(k, 0, T);
      pack_steps(k, 0, T);
    }
    if (!dev) {
      for (int k = 0; k < num_tasks; ++k) copy_out(k, 0, T, ctx->stream, 3);
      KT_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

}  // extern "C"
