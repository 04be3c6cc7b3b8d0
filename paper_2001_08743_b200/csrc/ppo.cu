// PPO training step on the device: the actor-critic's forward
// with its caches (ActorCritic::Forward, actor_critic.hpp:31-43), backward
// (actor_critic.hpp:45-49), AdamOptimizer::step (:66-79), compute_gae
// and ppo_update. The reference declares these and defines none; the
// arithmetic is builder-pinned and restated in oracle/ktune_oracle.c
// (ko_ac_backward, ko_adam_step, ko_compute_gae, ko_ppo_update): every batch reduction is
// a sequential chain in ascending sample order (products fused with __fma_rn, everything
// else separately rounded), so the device results are bit-identical to the restatement.
//
// Work split per PPO minibatch step (B <= a few hundred samples, ~22k parameters):
//  (1) ppo_row_kernel: one warp per sample — the exact fp64 forward (units spread over
//      lanes), the clipped-surrogate / value / entropy loss gradients w.r.t. the logits
//      and the value, and the per-sample backward through the three tanh layers;
//  (2) param_grad_kernel: one thread per parameter — the batch reduction of its
//      gradient (a B-long fma chain over coalesced rows) fused with its Adam update.
// The host loop only draws the epoch permutations (the reference Rng) and computes the
// Adam bias corrections; everything else stays on the device.
#include <algorithm>
#include <vector>

#include "device.cuh"
#include "internal.cuh"

struct ktune_adam {
  ktune_ctx* ctx = nullptr;
  int64_t dim = 0;
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  int64_t t = 0;
  double* d_m = nullptr;  // first moments
  double* d_v = nullptr;  // second moments
};

namespace {

using kt::dadd;
using kt::ddiv;
using kt::dmul;
using kt::dsub;

struct AcOff {
  int64_t w0, b0, wp1, bp1, wp2, bp2, wv1, bv1, wv2, bv2, total;
};
__host__ __device__ inline AcOff ac_off(int n, int h, int g) {  // actor_critic.hpp:52-53
  AcOff o;
  o.w0 = 0;
  o.b0 = (int64_t)h * n;
  o.wp1 = o.b0 + h;
  o.bp1 = o.wp1 + (int64_t)g * h;
  o.wp2 = o.bp1 + g;
  o.bp2 = o.wp2 + (int64_t)3 * n * g;
  o.wv1 = o.bp2 + 3 * n;
  o.bv1 = o.wv1 + (int64_t)g * h;
  o.wv2 = o.bv1 + g;
  o.bv2 = o.wv2 + g;
  o.total = o.bv2 + 1;
  return o;
}

constexpr int kRowWarps = 8;

// Per-sample inputs/outputs of the row kernel (all device pointers; NULL = unused).
struct RowIo {
  int n, h, g;
  int64_t B;
  const double* params;
  // states: x = states + src_row * n, src_row = perm ? perm[s0 + b] : b
  const double* states;
  const int64_t* perm;
  int64_t s0;
  // PPO sample data (indexed by src_row)
  const int8_t* actions;
  const double* old_logp;
  const double* adv;
  const double* ret;
  double clip_eps, c_v, c_e;
  // given caches / upstream gradients (backward-only mode, indexed by b)
  const double* in_h0;
  const double* in_hp;
  const double* in_hv;
  const double* in_dl;
  const double* in_dv;
  // outputs (indexed by b)
  double *x, *h0, *hp, *hv, *logits, *logp, *probs, *value;
  double *dl, *dv, *dz0, *dzp, *dzv;
  double* row_stats;  // B x 3: surrogate, squared value error, entropy
};

// mode bit 0: forward, bit 1: PPO loss gradients, bit 2: per-sample backward
template <int MODE>
__global__ void __launch_bounds__(32 * kRowWarps) ppo_row_kernel(const RowIo io) {
  extern __shared__ __align__(16) double sm[];
  const int n = io.n, h = io.h, g = io.g, n3 = 3 * io.n;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * kRowWarps + w;
  if (b >= io.B) return;
  const int per = n + 2 * h + 4 * g + 4 * n3 + n;
  double* x = sm + (size_t)w * per;
  double* h0 = x + n;
  double* hp = h0 + h;
  double* hv = hp + g;
  double* lg = hv + g;
  double* lp = lg + n3;
  double* pr = lp + n3;
  double* dl = pr + n3;
  double* dzv = dl + n3;
  double* dzp = dzv + g;
  double* dz0 = dzp + g;
  double* Hd = dz0 + h;
  const double* P = io.params;
  const AcOff o = ac_off(n, h, g);
  const int64_t src = io.perm ? io.perm[io.s0 + b] : b;
  double v = 0.0;
  if (MODE & 1) {
    for (int i = lane; i < n; i += 32) x[i] = io.states[src * n + i];
    __syncwarp();
    for (int j = lane; j < h; j += 32) {  // h0 = tanh(W0 x + b0)
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc = __fma_rn(P[o.w0 + (int64_t)i * h + j], x[i], acc);
      h0[j] = kt::kt_tanh(dadd(acc, P[o.b0 + j]));
    }
    __syncwarp();
    for (int j = lane; j < g; j += 32) {  // hp, hv
      double ap = 0.0, av = 0.0;
      for (int i = 0; i < h; ++i) {
        ap = __fma_rn(P[o.wp1 + (int64_t)i * g + j], h0[i], ap);
        av = __fma_rn(P[o.wv1 + (int64_t)i * g + j], h0[i], av);
      }
      hp[j] = kt::kt_tanh(dadd(ap, P[o.bp1 + j]));
      hv[j] = kt::kt_tanh(dadd(av, P[o.bv1 + j]));
    }
    __syncwarp();
    for (int a = lane; a < n3; a += 32) {  // logits = Wp2 hp + bp2
      double acc = 0.0;
      for (int j = 0; j < g; ++j) acc = __fma_rn(P[o.wp2 + (int64_t)j * n3 + a], hp[j], acc);
      lg[a] = dadd(acc, P[o.bp2 + a]);
    }
    __syncwarp();
    for (int d = lane; d < n; d += 32) {  // per-knob log-softmax (actor_critic.hpp:13-14)
      const kt::Knob3 k3 = kt::softmax3(lg[3 * d], lg[3 * d + 1], lg[3 * d + 2]);
      for (int k = 0; k < 3; ++k) {
        lp[3 * d + k] = k3.lp[k];
        pr[3 * d + k] = k3.p[k];
      }
    }
    for (int j = 0; j < g; ++j) v = __fma_rn(P[o.wv2 + j], hv[j], v);  // every lane: the same chain
    v = dadd(v, P[o.bv2]);
    __syncwarp();
    if (io.x)
      for (int i = lane; i < n; i += 32) io.x[b * n + i] = x[i];
    if (io.h0)
      for (int j = lane; j < h; j += 32) io.h0[b * h + j] = h0[j];
    if (io.hp)
      for (int j = lane; j < g; j += 32) io.hp[b * g + j] = hp[j];
    if (io.hv)
      for (int j = lane; j < g; j += 32) io.hv[b * g + j] = hv[j];
    for (int a = lane; a < n3; a += 32) {
      if (io.logits) io.logits[b * n3 + a] = lg[a];
      if (io.logp) io.logp[b * n3 + a] = lp[a];
      if (io.probs) io.probs[b * n3 + a] = pr[a];
    }
    if (io.value && lane == 0) io.value[b] = v;
  } else {  // backward only: the caller's caches and upstream gradients
    for (int j = lane; j < h; j += 32) h0[j] = io.in_h0[b * h + j];
    for (int j = lane; j < g; j += 32) {
      hp[j] = io.in_hp[b * g + j];
      hv[j] = io.in_hv[b * g + j];
    }
    for (int a = lane; a < n3; a += 32) dl[a] = io.in_dl[b * n3 + a];
  }
  double dvb = (MODE & 1) ? 0.0 : io.in_dv[b];
  if (MODE & 2) {  // clipped surrogate + value + entropy gradients (ko_ppo_loss_grad)
    const double invB = ddiv(1.0, (double)io.B);
    // sequential per-sample sums over knobs (every lane computes the same chain)
    double lpj = 0.0, H = 0.0;
    for (int d = 0; d < n; ++d) {
      lpj = dadd(lpj, lp[3 * d + (io.actions[src * n + d] + 1)]);
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc = dadd(acc, dmul(pr[3 * d + k], lp[3 * d + k]));
      H = dadd(H, -acc);
      if ((d & 31) == lane) Hd[d] = -acc;
    }
    const double rho = kt::kt_exp(dsub(lpj, io.old_logp[src]));
    const double A = io.adv[src];
    const double un = dmul(rho, A);
    const double lo = dsub(1.0, io.clip_eps), hi = dadd(1.0, io.clip_eps);
    const double rc = rho < lo ? lo : (rho > hi ? hi : rho);
    const double cl = dmul(rc, A);
    const double s = un <= cl ? un : cl;
    const double gs = un <= cl ? dmul(A, rho) : 0.0;
    __syncwarp();
    for (int d = lane; d < n; d += 32) {
      const int act = io.actions[src * n + d] + 1;
      for (int k = 0; k < 3; ++k) {
        const double pk = pr[3 * d + k];
        const double t2 = dmul(gs, dsub(k == act ? 1.0 : 0.0, pk));
        const double t5 = dmul(io.c_e, dmul(pk, dadd(lp[3 * d + k], Hd[d])));
        dl[3 * d + k] = dmul(invB, dsub(t5, t2));
      }
    }
    const double diff = dsub(v, io.ret[src]);
    dvb = dmul(invB, dmul(dmul(2.0, io.c_v), diff));
    if (lane == 0) {
      if (io.dv) io.dv[b] = dvb;
      if (io.row_stats) {
        io.row_stats[b * 3] = s;
        io.row_stats[b * 3 + 1] = dmul(diff, diff);
        io.row_stats[b * 3 + 2] = H;
      }
    }
    __syncwarp();
    if (io.dl)
      for (int a = lane; a < n3; a += 32) io.dl[b * n3 + a] = dl[a];
  }
  if (MODE & 4) {  // per-sample backward (ko_ac_backward, first half)
    __syncwarp();
    for (int j = lane; j < g; j += 32) {
      dzv[j] = dmul(dmul(dvb, P[o.wv2 + j]), dsub(1.0, dmul(hv[j], hv[j])));
      double acc = 0.0;
      for (int a = 0; a < n3; ++a) acc = __fma_rn(P[o.wp2 + (int64_t)j * n3 + a], dl[a], acc);
      dzp[j] = dmul(acc, dsub(1.0, dmul(hp[j], hp[j])));
    }
    __syncwarp();
    for (int i = lane; i < h; i += 32) {
      double acc = 0.0;
      for (int j = 0; j < g; ++j) acc = __fma_rn(P[o.wp1 + (int64_t)i * g + j], dzp[j], acc);
      for (int j = 0; j < g; ++j) acc = __fma_rn(P[o.wv1 + (int64_t)i * g + j], dzv[j], acc);
      dz0[i] = dmul(acc, dsub(1.0, dmul(h0[i], h0[i])));
    }
    __syncwarp();
    for (int j = lane; j < g; j += 32) {
      io.dzv[b * g + j] = dzv[j];
      io.dzp[b * g + j] = dzp[j];
    }
    for (int i = lane; i < h; i += 32) io.dz0[b * h + i] = dz0[i];
  }
}

size_t row_smem(int n, int h, int g) { return sizeof(double) * kRowWarps * (size_t)(n + 2 * h + 4 * g + 13 * n); }

// Parameter gradients (ko_ac_backward, second half): thread p reduces over the batch in
// ascending sample order; optional fused Adam update (AdamOptimizer::step). Thread P
// (one extra) folds the minibatch loss sums into the running statistics.
struct GradIo {
  int n, h, g;
  int64_t B, P;
  const double *x, *h0, *hp, *hv, *dl, *dv, *dz0, *dzp, *dzv;
  double* grad;    // may be NULL when adam is set
  double* params;  // Adam target
  double *m, *v;
  double lr, beta1, beta2, eps, bc1, bc2;
  int adam;
  const double* row_stats;
  double* tot;  // [policy, value, entropy] running sums over minibatch steps
};

__global__ void __launch_bounds__(128) param_grad_kernel(const GradIo io) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = io.n, h = io.h, g = io.g, n3 = 3 * io.n;
  const int64_t B = io.B;
  if (p == io.P) {  // minibatch statistics (ko_ppo_update)
    if (io.row_stats && io.tot) {
      double ss = 0.0, sv = 0.0, se = 0.0;
      for (int64_t b = 0; b < B; ++b) {
        ss = dadd(ss, io.row_stats[b * 3]);
        sv = dadd(sv, io.row_stats[b * 3 + 1]);
        se = dadd(se, io.row_stats[b * 3 + 2]);
      }
      const double invB = ddiv(1.0, (double)B);
      io.tot[0] = dadd(io.tot[0], dmul(-ss, invB));
      io.tot[1] = dadd(io.tot[1], dmul(sv, invB));
      io.tot[2] = dadd(io.tot[2], dmul(se, invB));
    }
    return;
  }
  if (p > io.P) return;
  const AcOff o = ac_off(n, h, g);
  double acc = 0.0;
  if (p < o.b0) {  // W0(j, i), column-major h x n
    const int i = (int)(p / h), j = (int)(p % h);
    for (int64_t b = 0; b < B; ++b) acc = __fma_rn(io.dz0[b * h + j], io.x[b * n + i], acc);
  } else if (p < o.wp1) {
    const int j = (int)(p - o.b0);
    for (int64_t b = 0; b < B; ++b) acc = dadd(acc, io.dz0[b * h + j]);
  } else if (p < o.bp1) {  // Wp1(j, i), g x h
    const int64_t q = p - o.wp1;
    const int i = (int)(q / g), j = (int)(q % g);
    for (int64_t b = 0; b < B; ++b) acc = __fma_rn(io.dzp[b * g + j], io.h0[b * h + i], acc);
  } else if (p < o.wp2) {
    const int j = (int)(p - o.bp1);
    for (int64_t b = 0; b < B; ++b) acc = dadd(acc, io.dzp[b * g + j]);
  } else if (p < o.bp2) {  // Wp2(a, j), 3n x g
    const int64_t q = p - o.wp2;
    const int j = (int)(q / n3), a = (int)(q % n3);
    for (int64_t b = 0; b < B; ++b) acc = __fma_rn(io.dl[b * n3 + a], io.hp[b * g + j], acc);
  } else if (p < o.wv1) {
    const int a = (int)(p - o.bp2);
    for (int64_t b = 0; b < B; ++b) acc = dadd(acc, io.dl[b * n3 + a]);
  } else if (p < o.bv1) {  // Wv1(j, i), g x h
    const int64_t q = p - o.wv1;
    const int i = (int)(q / g), j = (int)(q % g);
    for (int64_t b = 0; b < B; ++b) acc = __fma_rn(io.dzv[b * g + j], io.h0[b * h + i], acc);
  } else if (p < o.wv2) {
    const int j = (int)(p - o.bv1);
    for (int64_t b = 0; b < B; ++b) acc = dadd(acc, io.dzv[b * g + j]);
  } else if (p < o.bv2) {
    const int j = (int)(p - o.wv2);
    for (int64_t b = 0; b < B; ++b) acc = __fma_rn(io.dv[b], io.hv[b * g + j], acc);
  } else {
    for (int64_t b = 0; b < B; ++b) acc = dadd(acc, io.dv[b]);
  }
  if (io.grad) io.grad[p] = acc;
  if (io.adam) {  // ko_adam_step
    const double m = dadd(dmul(io.beta1, io.m[p]), dmul(dsub(1.0, io.beta1), acc));
    const double v = dadd(dmul(io.beta2, io.v[p]), dmul(dsub(1.0, io.beta2), dmul(acc, acc)));
    io.m[p] = m;
    io.v[p] = v;
    const double mh = ddiv(m, io.bc1), vh = ddiv(v, io.bc2);
    io.params[p] = dsub(io.params[p], ddiv(dmul(io.lr, mh), dadd(__dsqrt_rn(vh), io.eps)));
  }
}

__global__ void adam_kernel(int64_t P, double* params, const double* grad, double* mm, double* vv, double lr,
                            double b1, double b2, double eps, double bc1, double bc2) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const double gi = grad[p];
    const double m = dadd(dmul(b1, mm[p]), dmul(dsub(1.0, b1), gi));
    const double v = dadd(dmul(b2, vv[p]), dmul(dsub(1.0, b2), dmul(gi, gi)));
    mm[p] = m;
    vv[p] = v;
    params[p] = dsub(params[p], ddiv(dmul(lr, ddiv(m, bc1)), dadd(__dsqrt_rn(ddiv(v, bc2)), eps)));
  }
}

// compute_gae: one thread per episode, backwards over its T steps.
__global__ void gae_kernel(int64_t E, int32_t T, const double* rw, const double* val, const double* term,
                           double gamma, double gl, double* adv, double* ret) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int32_t t = T - 1; t >= 0; --t) {
      const int64_t k = e * T + t;
      const double vn = t == T - 1 ? term[e] : val[k + 1];
      a = dadd(dsub(dadd(rw[k], dmul(gamma, vn)), val[k]), dmul(gl, a));
      adv[k] = a;
      ret[k] = dadd(a, val[k]);
    }
  }
}

// Advantage normalisation (ko_normalize_advantages): the two sequential sums run in one
// thread (N ~ 64k per PPO update), the division in parallel.
__global__ void adv_moments_kernel(int64_t N, const double* a, double* mom) {
  double s = 0.0;
  for (int64_t i = 0; i < N; ++i) s = dadd(s, a[i]);
  const double mean = ddiv(s, (double)N);
  double q = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double d = dsub(a[i], mean);
    q = dadd(q, dmul(d, d));
  }
  mom[0] = mean;
  mom[1] = dadd(__dsqrt_rn(ddiv(q, (double)N)), 1e-8);
}
__global__ void adv_norm_kernel(int64_t N, const double* a, const double* mom, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ddiv(dsub(a[i], mom[0]), mom[1]);
}

void adam_bias(double b1, double b2, int64_t t, double* bc1, double* bc2) {  // ko_adam_bias
  double p1 = 1.0, p2 = 1.0;
  for (int64_t i = 0; i < t; ++i) {
    p1 = p1 * b1;
    p2 = p2 * b2;
  }
  *bc1 = 1.0 - p1;
  *bc2 = 1.0 - p2;
}

uint64_t mix64(uint64_t z) {  // rng.hpp:16-23
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

template <int MODE>
void launch_rows(ktune_ctx* ctx, const RowIo& io) {
  const size_t smem = row_smem(io.n, io.h, io.g);
  KT_CUDA(cudaFuncSetAttribute(ppo_row_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ppo_row_kernel<MODE><<<(unsigned)kt::ceil_div(io.B, kRowWarps), 32 * kRowWarps, smem, ctx->stream>>>(io);
  kt::check_launch(ctx, "ppo_rows");
}

void check_ac(const ktune_ac* ac) {
  if (!ac || ac->n < 1 || ac->n > 32 || ac->h < 1 || ac->h > 1024 || ac->g < 1 || ac->g > 512)
    kt::fail(KTUNE_ERR_CONFIG, "actor-critic: unsupported dimensions for the training path");
}

}  // namespace

extern "C" {

int ktune_ac_get_params(ktune_ctx* ctx, const ktune_ac* ac, double* out) {
  return kt_guard(ctx, [&] {
    KT_CUDA(cudaMemcpyAsync(out, ac->d_params, sizeof(double) * ac->num_params, cudaMemcpyDeviceToHost, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_ac_forward_cache(ktune_ctx* ctx, const ktune_ac* ac, const double* states, int64_t B, double* h0,
                           double* hp, double* hv, double* logits, double* log_probs, double* probs, double* values,
                           int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_ac_forward_cache");
    check_ac(ac);
    if (B < 0) kt::fail(KTUNE_ERR_CONFIG, "negative batch");
    if (B == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const int n = ac->n, h = ac->h, g = ac->g;
    RowIo io{};
    io.n = n;
    io.h = h;
    io.g = g;
    io.B = B;
    io.params = ac->d_params;
    io.states = (const double*)kt::stage_in(ctx, kt::WS_IN0, states, sizeof(double) * B * n, dev);
    struct O {
      double* host;
      double** dst;
      size_t bytes;
      int slot;
    } outs[7] = {{h0, &io.h0, sizeof(double) * B * h, kt::WS_OUT0},
                 {hp, &io.hp, sizeof(double) * B * g, kt::WS_OUT1},
                 {hv, &io.hv, sizeof(double) * B * g, kt::WS_OUT2},
                 {logits, &io.logits, sizeof(double) * B * 3 * n, kt::WS_OUT3},
                 {log_probs, &io.logp, sizeof(double) * B * 3 * n, kt::WS_OUT4},
                 {probs, &io.probs, sizeof(double) * B * 3 * n, kt::WS_SCRATCH},
                 {values, &io.value, sizeof(double) * B, kt::WS_SCRATCH2}};
    for (auto& x : outs)
      if (x.host) *x.dst = (double*)kt::out_buf(ctx, x.slot, x.host, x.bytes, dev);
    launch_rows<1>(ctx, io);
    for (auto& x : outs)
      if (x.host) kt::stage_out(ctx, x.host, *x.dst, x.bytes, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_ac_backward(ktune_ctx* ctx, const ktune_ac* ac, const double* states, const double* h0,
                      const double* hp, const double* hv, int64_t B, const double* d_logits,
                      const double* d_values, double* grad, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_ac_backward");
    check_ac(ac);
    if (B < 0) kt::fail(KTUNE_ERR_CONFIG, "negative batch");
    const bool dev = flags & KTUNE_F_DEVICE;
    const int n = ac->n, h = ac->h, g = ac->g;
    const int64_t P = ac->num_params;
    double* d_grad = (double*)kt::out_buf(ctx, kt::WS_OUT0, grad, sizeof(double) * P, dev);
    if (B == 0) {
      KT_CUDA(cudaMemsetAsync(d_grad, 0, sizeof(double) * P, ctx->stream));
    } else {
      RowIo io{};
      io.n = n;
      io.h = h;
      io.g = g;
      io.B = B;
      io.params = ac->d_params;
      io.in_h0 = (const double*)kt::stage_in(ctx, kt::WS_IN0, h0, sizeof(double) * B * h, dev);
      io.in_hp = (const double*)kt::stage_in(ctx, kt::WS_IN1, hp, sizeof(double) * B * g, dev);
      io.in_hv = (const double*)kt::stage_in(ctx, kt::WS_IN2, hv, sizeof(double) * B * g, dev);
      io.in_dl = (const double*)kt::stage_in(ctx, kt::WS_OUT1, d_logits, sizeof(double) * B * 3 * n, dev);
      io.in_dv = (const double*)kt::stage_in(ctx, kt::WS_OUT2, d_values, sizeof(double) * B, dev);
      const double* d_x = (const double*)kt::stage_in(ctx, kt::WS_OUT3, states, sizeof(double) * B * n, dev);
      double* scr = (double*)ctx->dev(kt::WS_SCRATCH, sizeof(double) * B * (h + 2 * g));
      io.dz0 = scr;
      io.dzp = scr + B * h;
      io.dzv = io.dzp + B * g;
      launch_rows<4>(ctx, io);
      GradIo gi{};
      gi.n = n;
      gi.h = h;
      gi.g = g;
      gi.B = B;
      gi.P = P;
      gi.x = d_x;
      gi.h0 = io.in_h0;
      gi.hp = io.in_hp;
      gi.hv = io.in_hv;
      gi.dl = io.in_dl;
      gi.dv = io.in_dv;
      gi.dz0 = io.dz0;
      gi.dzp = io.dzp;
      gi.dzv = io.dzv;
      gi.grad = d_grad;
      param_grad_kernel<<<(unsigned)kt::ceil_div(P + 1, 128), 128, 0, ctx->stream>>>(gi);
      kt::check_launch(ctx, "param_grad");
    }
    kt::stage_out(ctx, grad, d_grad, sizeof(double) * P, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_adam_create(ktune_ctx* ctx, int64_t dim, double step_size, double beta1, double beta2, double epsilon,
                      ktune_adam** out) {
  return kt_guard(ctx, [&] {
    if (dim <= 0 || !(step_size > 0.0) || !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0) ||
        !(epsilon > 0.0))
      kt::fail(KTUNE_ERR_CONFIG, "adam: bad dimension or hyper-parameters");
    auto* a = new ktune_adam();
    a->ctx = ctx;
    a->dim = dim;
    a->lr = step_size;
    a->beta1 = beta1;
    a->beta2 = beta2;
    a->eps = epsilon;
    KT_CUDA(cudaMalloc(&a->d_m, sizeof(double) * dim * 2));
    a->d_v = a->d_m + dim;
    KT_CUDA(cudaMemsetAsync(a->d_m, 0, sizeof(double) * dim * 2, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = a;
  });
}

int ktune_adam_destroy(ktune_adam* a) {
  if (!a) return KTUNE_OK;
  cudaFree(a->d_m);
  delete a;
  return KTUNE_OK;
}

int ktune_adam_state(ktune_ctx* ctx, const ktune_adam* a, double* m, double* v, int64_t* t) {
  return kt_guard(ctx, [&] {
    if (m) KT_CUDA(cudaMemcpyAsync(m, a->d_m, sizeof(double) * a->dim, cudaMemcpyDeviceToHost, ctx->stream));
    if (v) KT_CUDA(cudaMemcpyAsync(v, a->d_v, sizeof(double) * a->dim, cudaMemcpyDeviceToHost, ctx->stream));
    KT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (t) *t = a->t;
  });
}

int ktune_adam_step(ktune_ctx* ctx, ktune_adam* a, double* params, const double* grad, int flags) {
  return kt_guard(ctx, [&] {
    const bool dev = flags & KTUNE_F_DEVICE;
    const int64_t P = a->dim;
    double* d_p = (double*)kt::stage_in(ctx, kt::WS_IN0, params, sizeof(double) * P, dev);
    const double* d_g = (const double*)kt::stage_in(ctx, kt::WS_IN1, grad, sizeof(double) * P, dev);
    a->t += 1;
    double bc1, bc2;
    adam_bias(a->beta1, a->beta2, a->t, &bc1, &bc2);
    adam_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(P, 256), 4096), 256, 0, ctx->stream>>>(
        P, d_p, d_g, a->d_m, a->d_v, a->lr, a->beta1, a->beta2, a->eps, bc1, bc2);
    kt::check_launch(ctx, "adam");
    kt::stage_out(ctx, params, d_p, sizeof(double) * P, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_compute_gae(ktune_ctx* ctx, int64_t E, int32_t T, const double* rewards, const double* values,
                      const double* terminal_values, double gamma, double lambda, double* advantages,
                      double* returns, int flags) {
  return kt_guard(ctx, [&] {
    if (E < 0 || T < 0) kt::fail(KTUNE_ERR_CONFIG, "compute_gae: length mismatch");
    if (E == 0 || T == 0) return;
    const bool dev = flags & KTUNE_F_DEVICE;
    const size_t nb = sizeof(double) * E * T;
    const double* d_r = (const double*)kt::stage_in(ctx, kt::WS_IN0, rewards, nb, dev);
    const double* d_v = (const double*)kt::stage_in(ctx, kt::WS_IN1, values, nb, dev);
    const double* d_t = (const double*)kt::stage_in(ctx, kt::WS_IN2, terminal_values, sizeof(double) * E, dev);
    double* d_a = (double*)kt::out_buf(ctx, kt::WS_OUT0, advantages, nb, dev);
    double* d_ret = (double*)kt::out_buf(ctx, kt::WS_OUT1, returns, nb, dev);
    gae_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(E, 128), 4096), 128, 0, ctx->stream>>>(
        E, T, d_r, d_v, d_t, gamma, gamma * lambda, d_a, d_ret);
    kt::check_launch(ctx, "gae");
    kt::stage_out(ctx, advantages, d_a, nb, dev);
    kt::stage_out(ctx, returns, d_ret, nb, dev);
    if (!dev) KT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ktune_ppo_update(ktune_ctx* ctx, ktune_ac* ac, ktune_adam* adam, const ktune_ppo_params* pp, int64_t N,
                     const double* states, const int8_t* actions, const double* old_logp, const double* advantages,
                     const double* returns, uint64_t seed, double* stats, int flags) {
  return kt_guard(ctx, [&] {
    KT_RANGE("ktune_ppo_update");
    check_ac(ac);
    if (!adam || !pp || adam->dim != ac->num_params) kt::fail(KTUNE_ERR_CONFIG, "ppo_update: optimizer/agent mismatch");
    if (N <= 0) kt::fail(KTUNE_ERR_CONFIG, "ppo_update: empty trajectory batch");
    if (pp->num_epochs <= 0 || pp->minibatch_size <= 0 || !(pp->clip_epsilon > 0.0))
      kt::fail(KTUNE_ERR_CONFIG, "ppo_update: bad parameters");
    const bool dev = flags & KTUNE_F_DEVICE;
    const int n = ac->n, h = ac->h, g = ac->g;
    const int64_t P = ac->num_params, mb = pp->minibatch_size, S = std::min(mb, N);
    cudaStream_t s = ctx->stream;
    const double* d_x = (const double*)kt::stage_in(ctx, kt::WS_IN0, states, sizeof(double) * N * n, dev);
    const int8_t* d_a = (const int8_t*)kt::stage_in(ctx, kt::WS_IN1, actions, (size_t)N * n, dev);
    const double* d_ol = (const double*)kt::stage_in(ctx, kt::WS_IN2, old_logp, sizeof(double) * N, dev);
    const double* d_adv = (const double*)kt::stage_in(ctx, kt::WS_OUT3, advantages, sizeof(double) * N, dev);
    const double* d_ret = (const double*)kt::stage_in(ctx, kt::WS_OUT4, returns, sizeof(double) * N, dev);
    // scratch: normalised advantages, moments, permutation, per-minibatch activations
    const size_t per_row = (size_t)(n + h + 2 * g + 3 * n + 1 + h + 2 * g + 3);
    double* scr = (double*)ctx->dev(kt::WS_SCRATCH, sizeof(double) * (N + 8 + 3 + (size_t)S * per_row));
    double* an = scr;
    double* mom = an + N;
    double* tot = mom + 4;
    double* xs = tot + 7;
    double* h0 = xs + S * n;
    double* hp = h0 + S * h;
    double* hv = hp + S * g;
    double* dl = hv + S * g;
    double* dv = dl + S * 3 * n;
    double* dz0 = dv + S;
    double* dzp = dz0 + S * h;
    double* dzv = dzp + S * g;
    double* rs = dzv + S * g;
    int64_t* perm = (int64_t*)ctx->dev(kt::WS_SCRATCH2, sizeof(int64_t) * N * pp->num_epochs);
    adv_moments_kernel<<<1, 1, 0, s>>>(N, d_adv, mom);
    adv_norm_kernel<<<(unsigned)std::min<int64_t>(kt::ceil_div(N, 256), 4096), 256, 0, s>>>(N, d_adv, mom, an);
    KT_CUDA(cudaMemsetAsync(tot, 0, sizeof(double) * 3, s));
    // epoch permutations: Fisher-Yates (rng.hpp:88-92) from Rng(seed_combine(seed, epoch))
    int64_t* hperm = (int64_t*)ctx->host(0, sizeof(int64_t) * N * pp->num_epochs);
    for (int ep = 0; ep < pp->num_epochs; ++ep) {
      int64_t* pe = hperm + (size_t)ep * N;
      for (int64_t i = 0; i < N; ++i) pe[i] = i;
      uint64_t st = mix64(seed + 0x9E3779B97F4A7C15ULL + mix64((uint64_t)ep));  // seed_combine (rng.hpp:26-28)
      auto below = [&](uint64_t m) {  // Rng::below (rng.hpp:63-69)
        const uint64_t thr = (0 - m) % m;
        for (;;) {
          st += 0x9E3779B97F4A7C15ULL;
          const uint64_t r = mix64(st);
          if (r >= thr) return r % m;
        }
      };
      for (int64_t i = N; i > 1; --i) std::swap(pe[i - 1], pe[below((uint64_t)i)]);
    }
    KT_CUDA(cudaMemcpyAsync(perm, hperm, sizeof(int64_t) * N * pp->num_epochs, cudaMemcpyHostToDevice, s));
    RowIo io{};
    io.n = n;
    io.h = h;
    io.g = g;
    io.params = ac->d_params;
    io.states = d_x;
    io.perm = perm;
    io.actions = d_a;
    io.old_logp = d_ol;
    io.adv = an;
    io.ret = d_ret;
    io.clip_eps = pp->clip_epsilon;
    io.c_v = pp->value_coef;
    io.c_e = pp->entropy_coef;
    io.x = xs;
    io.h0 = h0;
    io.hp = hp;
    io.hv = hv;
    io.dl = dl;
    io.dv = dv;
    io.dz0 = dz0;
    io.dzp = dzp;
    io.dzv = dzv;
    io.row_stats = rs;
    GradIo gi{};
    gi.n = n;
    gi.h = h;
    gi.g = g;
    gi.P = P;
    gi.x = xs;
    gi.h0 = h0;
    gi.hp = hp;
    gi.hv = hv;
    gi.dl = dl;
    gi.dv = dv;
    gi.dz0 = dz0;
    gi.dzp = dzp;
    gi.dzv = dzv;
    gi.params = ac->d_params;
    gi.m = adam->d_m;
    gi.v = adam->d_v;
    gi.lr = adam->lr;
    gi.beta1 = adam->beta1;
    gi.beta2 = adam->beta2;
    gi.eps = adam->eps;
    gi.adam = 1;
    gi.row_stats = rs;
    gi.tot = tot;
    const size_t smem = row_smem(n, h, g);
    KT_CUDA(cudaFuncSetAttribute(ppo_row_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t steps = 0;
    for (int ep = 0; ep < pp->num_epochs; ++ep) {
      for (int64_t s0 = 0; s0 < N; s0 += mb) {
        const int64_t B = std::min(mb, N - s0);
        io.B = B;
        io.s0 = (int64_t)ep * N + s0;
        ppo_row_kernel<7><<<(unsigned)kt::ceil_div(B, kRowWarps), 32 * kRowWarps, smem, s>>>(io);
        adam->t += 1;
        adam_bias(adam->beta1, adam->beta2, adam->t, &gi.bc1, &gi.bc2);
        gi.B = B;
        param_grad_kernel<<<(unsigned)kt::ceil_div(P + 1, 128), 128, 0, s>>>(gi);
        ++steps;
      }
    }
    kt::check_launch(ctx, "ppo_update", (int)(2 * steps + 2));
    double htot[3];
    KT_CUDA(cudaMemcpyAsync(htot, tot, sizeof(htot), cudaMemcpyDeviceToHost, s));
    KT_CUDA(cudaMemcpyAsync(ac->host_params.data(), ac->d_params, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
    KT_CUDA(cudaStreamSynchronize(s));
    ++ac->version;
    if (stats)
      for (int k = 0; k < 3; ++k) stats[k] = htot[k] / (double)steps;
  });
}

}  // extern "C"
