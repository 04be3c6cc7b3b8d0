/* CPU restatement of the Chameleon reference hot path — TEST INFRASTRUCTURE.
 * See ktune_oracle.h for the pinning contract. Build: oracle/Makefile
 * (-O3 -ffp-contract=off, no -march: scalar SSE2 IEEE double, no FMA, the
 * reference's own default build, CMakeLists.txt:4,7-9). */
#include "ktune_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * rng.hpp:16-94
 * ==================================================================== */
uint64_t ko_mix64(uint64_t z) { /* rng.hpp:16-23 */
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

uint64_t ko_seed_combine(uint64_t a, uint64_t b) { /* rng.hpp:26-28 */
  return ko_mix64(a + 0x9E3779B97F4A7C15ULL + ko_mix64(b));
}

uint64_t ko_stream_seed(uint64_t root, const char* name) { /* rng.hpp:33-40 */
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* p = (const unsigned char*)name; *p; ++p) {
    h ^= *p;
    h *= 0x100000001B3ULL;
  }
  return ko_seed_combine(root, h);
}

double ko_hash01(uint64_t seed, uint64_t counter) { /* rng.hpp:44-47 */
  const uint64_t u = ko_mix64(seed ^ ko_mix64(counter + 0x9E3779B97F4A7C15ULL));
  return (double)(u >> 11) * 0x1.0p-53;
}

typedef struct {
  uint64_t state;
} ko_rng;

static uint64_t rng_next(ko_rng* r) { /* rng.hpp:54-57 */
  r->state += 0x9E3779B97F4A7C15ULL;
  return ko_mix64(r->state);
}
static double rng_uniform01(ko_rng* r) { /* rng.hpp:60 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static uint64_t rng_below(ko_rng* r, uint64_t n) { /* rng.hpp:63-69 */
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = rng_next(r);
    if (x >= threshold) return x % n;
  }
}
static double rng_normal(ko_rng* r) { /* rng.hpp:78-83 (host libm; init only) */
  double u1 = rng_uniform01(r);
  const double u2 = rng_uniform01(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* ======================================================================
 * Portable transcendental functions. The reference has no
 * tanh/exp/log of its own (actor_critic.hpp has no .cpp), so these ARE the
 * definition the rollout is pinned to. Only IEEE + - * / and exact bit
 * operations, fixed evaluation order; the device copy in
 * paper_2001_08743_b200/csrc/kt_math.cuh is an independent restatement that
 * tests/test_gpu_math.py checks bit-for-bit against this one.
 *   exp: fdlibm e_exp.c scheme (Cody-Waite reduction, Remez P1..P5)
 *   log: fdlibm e_log.c scheme (Lg1..Lg7)
 *   tanh: Cephes tanh.c scheme (rational P/Q below 0.625, exp above)
 * ==================================================================== */
static uint64_t dbits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}
static double bitsd(uint64_t u) {
  double x;
  memcpy(&x, &u, 8);
  return x;
}

double ko_exp(double x) {
  const double o_threshold = 7.09782712893383973096e+02;
  const double u_threshold = -7.45133219101941108420e+02;
  const double ln2HI = 6.93147180369123816490e-01;
  const double ln2LO = 1.90821492927058770002e-10;
  const double invln2 = 1.44269504088896338700e+00;
  const double P1 = 1.66666666666666019037e-01;
  const double P2 = -2.77777777770155933842e-03;
  const double P3 = 6.61375632143793436117e-05;
  const double P4 = -1.65339022054652515390e-06;
  const double P5 = 4.13813679705723846039e-08;
  if (x != x) return x;
  if (x > o_threshold) return bitsd(0x7FF0000000000000ULL);
  if (x < u_threshold) return 0.0;
  const double ax = fabs(x);
  double hi = 0.0, lo = 0.0, r;
  int k = 0;
  if (ax > 0.34657359027997264) {
    k = (int)(invln2 * x + (x < 0.0 ? -0.5 : 0.5));
    const double t = (double)k;
    hi = x - t * ln2HI;
    lo = t * ln2LO;
    r = hi - lo;
  } else if (ax < 3.725290298461914e-09) { /* 2^-28 */
    return 1.0 + x;
  } else {
    r = x;
  }
  const double t = r * r;
  const double c = r - t * (P1 + t * (P2 + t * (P3 + t * (P4 + t * P5))));
  if (k == 0) return 1.0 - ((r * c) / (c - 2.0) - r);
  const double y = 1.0 - ((lo - (r * c) / (2.0 - c)) - hi);
  if (k >= -1021) return bitsd(dbits(y) + ((uint64_t)(int64_t)k << 52));
  return bitsd(dbits(y) + ((uint64_t)(int64_t)(k + 1000) << 52)) * 9.33263618503218878990e-302;
}

double ko_log(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
               Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
               Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
               Lg7 = 1.479819860511658591e-01;
  uint64_t u = dbits(x);
  int32_t hx = (int32_t)(u >> 32);
  const uint32_t lx = (uint32_t)u;
  int k = 0;
  if (hx < 0x00100000) {
    if (((hx & 0x7fffffff) | lx) == 0) return bitsd(0xFFF0000000000000ULL); /* -inf */
    if (hx < 0) return bitsd(0x7FF8000000000000ULL);                           /* NaN */
    k -= 54;
    x *= two54;
    u = dbits(x);
    hx = (int32_t)(u >> 32);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int32_t i0 = (hx + 0x95f64) & 0x100000;
  x = bitsd(((uint64_t)(uint32_t)(hx | (i0 ^ 0x3ff00000)) << 32) | (dbits(x) & 0xFFFFFFFFULL));
  k += (i0 >> 20);
  const double f = x - 1.0;
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double dk = (double)k;
      return dk * ln2_hi + dk * ln2_lo;
    }
    const double R = f * f * (0.5 - 0.33333333333333333 * f);
    if (k == 0) return f - R;
    const double dk = (double)k;
    return dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  const double s = f / (2.0 + f);
  const double dk = (double)k;
  const double z = s * s;
  int32_t i = hx - 0x6147a;
  const double w = z * z;
  const int32_t j = 0x6b851 - hx;
  const double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  const double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  const double R = t2 + t1;
  if (i > 0) {
    const double hfsq = 0.5 * f * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

double ko_tanh(double x) {
  const double P0 = -9.64399179425052238628E-1, P1 = -9.92877231001918586564E1,
               P2 = -1.61468768441708447952E3;
  const double Q0 = 1.12811678491632931402E2, Q1 = 2.23548839060100448583E3,
               Q2 = 4.84406305325125486048E3;
  if (x == 0.0) return x;
  double z = fabs(x);
  if (z > 354.891356446691998) return x > 0.0 ? 1.0 : -1.0; /* 0.5*MAXLOG */
  if (z >= 0.625) {
    const double s = ko_exp(z + z);
    z = 1.0 - 2.0 / (s + 1.0);
    if (x < 0.0) z = -z;
    return z;
  }
  const double s = x * x;
  const double p = (P0 * s + P1) * s + P2;
  const double q = ((s + Q0) * s + Q1) * s + Q2;
  z = p / q;
  z = x * s * z;
  return x + z;
}

/* ======================================================================
 * design_space.cpp / validity.cpp
 * ==================================================================== */
static int rule_eval(const ko_space* s, const int32_t* idx) { /* validity.cpp:162-204 */
  __int128 st[64];
  int sp = 0;
  for (int k = 0; k < s->nops; ++k) {
    const ko_rule_op* op = &s->ops[k];
    switch (op->code) {
      case KO_PUSH_CONST:
        st[sp++] = op->arg;
        break;
      case KO_PUSH_KNOB:
        st[sp++] = s->values[s->value_offsets[op->arg] + idx[op->arg]];
        break;
      case KO_ADD:
        --sp;
        st[sp - 1] += st[sp];
        break;
      case KO_MUL:
        --sp;
        st[sp - 1] *= st[sp];
        break;
      case KO_LE:
        --sp;
        return st[sp - 1] <= st[sp];
      case KO_LT:
        --sp;
        return st[sp - 1] < st[sp];
      case KO_EQ:
        --sp;
        return st[sp - 1] == st[sp];
      default:
        return 1;
    }
  }
  return 1;
}

int ko_validate(const ko_space* s, const int32_t* idx) { /* design_space.cpp:169-173 */
  if (s->ops == NULL || s->nops == 0) return 1;
  return rule_eval(s, idx);
}

void ko_validate_batch(const ko_space* s, const int32_t* idx, int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)ko_validate(s, idx + i * s->D);
}

uint64_t ko_id_of(const ko_space* s, const int32_t* idx) { /* design_space.cpp:158-167 */
  uint64_t id = 0;
  for (int i = 0; i < s->D; ++i) id = id * (uint64_t)s->card[i] + (uint64_t)idx[i];
  return id;
}

void ko_config_at(const ko_space* s, uint64_t id, int32_t* out) { /* design_space.cpp:141-156 */
  for (int i = s->D - 1; i >= 0; --i) {
    out[i] = (int32_t)(id % (uint64_t)s->card[i]);
    id /= (uint64_t)s->card[i];
  }
}

void ko_encode(const ko_space* s, const int32_t* idx, double* out) { /* design_space.cpp:189-200 */
  for (int i = 0; i < s->D; ++i)
    out[i] = s->card[i] > 1 ? (double)idx[i] / (double)(s->card[i] - 1) : 0.0;
}

void ko_encode_batch(const ko_space* s, const int32_t* idx, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) ko_encode(s, idx + i * s->D, out + i * s->D);
}

/* ======================================================================
 * cost_model.cpp:117-124, 179-199
 * ==================================================================== */
double ko_gbt_predict_one(const ko_gbt* m, const double* x) {
  double sum = 0.0;
  for (int t = 0; t < m->num_trees; ++t) {
    const int32_t base = m->offsets[t];
    int node = 0;
    while (m->feature[base + node] >= 0) {
      const int32_t k = base + node;
      node = x[m->feature[k]] <= m->threshold[k] ? m->left[k] : m->right[k];
    }
    sum += m->value[base + node];
  }
  return m->base + m->lr * sum;
}

void ko_gbt_predict_features(const ko_gbt* m, const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ko_gbt_predict_one(m, x + i * m->num_features);
}

void ko_gbt_predict_idx(const ko_gbt* m, const ko_space* s, const int32_t* idx, int64_t n,
                        double* out) {
  double x[256];
  for (int64_t i = 0; i < n; ++i) {
    ko_encode(s, idx + i * s->D, x);
    out[i] = ko_gbt_predict_one(m, x);
  }
}

/* ======================================================================
 * Actor-critic (actor_critic.hpp:10-57 interface; arithmetic builder-pinned,
 * DESIGN.md §5). Flat layout actor_critic.hpp:52-53:
 *   [W0 (h x n), b0 (h), Wp1 (g x h), bp1 (g), Wp2 (3n x g), bp2 (3n),
 *    Wv1 (g x h), bv1 (g), wv2 (g), bv2 (1)]
 * matrices column-major (Eigen::Map default): W(r, c) = base[c * rows + r].
 * ==================================================================== */
typedef struct {
  int64_t w0, b0, wp1, bp1, wp2, bp2, wv1, bv1, wv2, bv2, total;
} ac_off;

static ac_off ac_layout(int n, int h, int g) {
  ac_off o;
  o.w0 = 0;
  o.b0 = o.w0 + (int64_t)h * n;
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

int64_t ko_ac_num_params(int n, int h, int g) { return ac_layout(n, h, g).total; }

/* Pinned init: one Rng(seed) stream, weights drawn in flat-layout order as
 * normal() / sqrt(fan_in); biases are 0 and consume no draws. */
void ko_ac_init(int n, int h, int g, uint64_t seed, double* p) {
  const ac_off o = ac_layout(n, h, g);
  ko_rng r = {seed};
  memset(p, 0, sizeof(double) * (size_t)o.total);
  const double s0 = 1.0 / sqrt((double)n), s1 = 1.0 / sqrt((double)h), s2 = 1.0 / sqrt((double)g);
  for (int64_t i = o.w0; i < o.b0; ++i) p[i] = rng_normal(&r) * s0;
  for (int64_t i = o.wp1; i < o.bp1; ++i) p[i] = rng_normal(&r) * s1;
  for (int64_t i = o.wp2; i < o.bp2; ++i) p[i] = rng_normal(&r) * s2;
  for (int64_t i = o.wv1; i < o.bv1; ++i) p[i] = rng_normal(&r) * s1;
  for (int64_t i = o.wv2; i < o.bv2; ++i) p[i] = rng_normal(&r) * s2;
}

/* One state; scratch h0[h], hp[g], hv[g], logits[3n], logp[3n], probs[3n]. */
static double ac_forward_one(int n, int h, int g, const double* p, const double* x, double* h0,
                             double* hp, double* hv, double* logits, double* logp, double* probs) {
  const ac_off o = ac_layout(n, h, g);
  for (int j = 0; j < h; ++j) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = fma(p[o.w0 + (int64_t)i * h + j], x[i], acc);
    h0[j] = ko_tanh(acc + p[o.b0 + j]);
  }
  for (int j = 0; j < g; ++j) {
    double acc = 0.0;
    for (int i = 0; i < h; ++i) acc = fma(p[o.wp1 + (int64_t)i * g + j], h0[i], acc);
    hp[j] = ko_tanh(acc + p[o.bp1 + j]);
  }
  for (int a = 0; a < 3 * n; ++a) {
    double acc = 0.0;
    for (int j = 0; j < g; ++j) acc = fma(p[o.wp2 + (int64_t)j * 3 * n + a], hp[j], acc);
    logits[a] = acc + p[o.bp2 + a];
  }
  for (int j = 0; j < g; ++j) {
    double acc = 0.0;
    for (int i = 0; i < h; ++i) acc = fma(p[o.wv1 + (int64_t)i * g + j], h0[i], acc);
    hv[j] = ko_tanh(acc + p[o.bv1 + j]);
  }
  double v = 0.0;
  for (int j = 0; j < g; ++j) v = fma(p[o.wv2 + j], hv[j], v);
  v = v + p[o.bv2];
  /* per-knob log-softmax over {dec, stay, inc} (actor_critic.hpp:13-14) */
  for (int d = 0; d < n; ++d) {
    const double* l = logits + 3 * d;
    double m = l[0];
    if (l[1] > m) m = l[1];
    if (l[2] > m) m = l[2];
    const double e0 = ko_exp(l[0] - m), e1 = ko_exp(l[1] - m), e2 = ko_exp(l[2] - m);
    const double s = (e0 + e1) + e2;
    const double lse = m + ko_log(s);
    logp[3 * d + 0] = l[0] - lse;
    logp[3 * d + 1] = l[1] - lse;
    logp[3 * d + 2] = l[2] - lse;
    probs[3 * d + 0] = e0 / s;
    probs[3 * d + 1] = e1 / s;
    probs[3 * d + 2] = e2 / s;
  }
  return v;
}

void ko_ac_forward(int n, int h, int g, const double* params, const double* states, int64_t B,
                   double* h0, double* hp, double* hv, double* logits, double* log_probs,
                   double* probs, double* values) {
  double* sh0 = (double*)malloc(sizeof(double) * (size_t)(h + 2 * g + 9 * n));
  double* shp = sh0 + h;
  double* shv = shp + g;
  double* sl = shv + g;
  double* slp = sl + 3 * n;
  double* spr = slp + 3 * n;
  for (int64_t b = 0; b < B; ++b) {
    const double v = ac_forward_one(n, h, g, params, states + b * n, sh0, shp, shv, sl, slp, spr);
    if (h0) memcpy(h0 + b * h, sh0, sizeof(double) * (size_t)h);
    if (hp) memcpy(hp + b * g, shp, sizeof(double) * (size_t)g);
    if (hv) memcpy(hv + b * g, shv, sizeof(double) * (size_t)g);
    if (logits) memcpy(logits + b * 3 * n, sl, sizeof(double) * (size_t)(3 * n));
    if (log_probs) memcpy(log_probs + b * 3 * n, slp, sizeof(double) * (size_t)(3 * n));
    if (probs) memcpy(probs + b * 3 * n, spr, sizeof(double) * (size_t)(3 * n));
    if (values) values[b] = v;
  }
  free(sh0);
}

/* ======================================================================
 * run_episodes (builder-pinned):
 *  u(e,t,d) = hash01(explore_seed, (e*T + t)*D + d), e = global episode id;
 *  action a = 0 if u < p0, 1 if u < p0 + p1, else 2; direction = a - 1;
 *  joint logp = sum_d logp[d][a_d] in knob order; saturating apply
 *  (design_space.cpp:175-187); every episode runs exactly T steps; scores of
 *  Θ_0..Θ_T come from the cost model (one batched predict per episode).
 * ==================================================================== */
typedef struct {
  const ko_space* s;
  const ko_gbt* m;
  int h, g;
  const double* params;
  int64_t e_begin, e_end;
  int32_t T;
  int64_t episode_offset;
  uint64_t seed;
  const int32_t* init_idx;
  int32_t* idx_out;
  double* score_out;
  int8_t* actions_out;
  double* logp_out;
  double* value_out;
} ep_job;

static void* run_episode_range(void* arg) {
  const ep_job* J = (const ep_job*)arg;
  const int D = J->s->D, h = J->h, g = J->g;
  double* buf = (double*)malloc(sizeof(double) * (size_t)(h + 2 * g + 10 * D));
  double *h0 = buf, *hp = h0 + h, *hv = hp + g, *lg = hv + g, *lp = lg + 3 * D, *pr = lp + 3 * D,
         *x = pr + 3 * D;
  for (int64_t e = J->e_begin; e < J->e_end; ++e) {
    const int64_t ge = J->episode_offset + e;
    int32_t* traj = J->idx_out + e * (int64_t)(J->T + 1) * D;
    memcpy(traj, J->init_idx + e * D, sizeof(int32_t) * (size_t)D);
    for (int32_t t = 0; t < J->T; ++t) {
      const int32_t* cur = traj + (int64_t)t * D;
      int32_t* nxt = traj + (int64_t)(t + 1) * D;
      ko_encode(J->s, cur, x);
      const double v = ac_forward_one(D, h, g, J->params, x, h0, hp, hv, lg, lp, pr);
      double logp = 0.0;
      for (int d = 0; d < D; ++d) {
        const double u = ko_hash01(J->seed, ((uint64_t)ge * (uint64_t)J->T + (uint64_t)t) * (uint64_t)D + (uint64_t)d);
        const double p0 = pr[3 * d], p01 = pr[3 * d] + pr[3 * d + 1];
        const int a = u < p0 ? 0 : (u < p01 ? 1 : 2);
        logp = logp + lp[3 * d + a];
        int idx = cur[d] + (a - 1);
        if (idx < 0) idx = 0;
        if (idx > J->s->card[d] - 1) idx = J->s->card[d] - 1;
        nxt[d] = idx;
        if (J->actions_out) J->actions_out[(e * (int64_t)J->T + t) * D + d] = (int8_t)(a - 1);
      }
      if (J->logp_out) J->logp_out[e * (int64_t)J->T + t] = logp;
      if (J->value_out) J->value_out[e * (int64_t)J->T + t] = v;
    }
    if (J->score_out && J->m)
      ko_gbt_predict_idx(J->m, J->s, traj, J->T + 1, J->score_out + e * (int64_t)(J->T + 1));
  }
  free(buf);
  return NULL;
}

int ko_run_episodes(const ko_space* s, const ko_gbt* m, int h, int g, const double* params,
                    int64_t E, int32_t T, int64_t episode_offset, uint64_t explore_seed,
                    const int32_t* init_idx, int32_t* idx_out, double* score_out,
                    int8_t* actions_out, double* logp_out, double* value_out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > E) threads = (int)(E > 0 ? E : 1);
  ep_job* jobs = (ep_job*)calloc((size_t)threads, sizeof(ep_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int w = 0; w < threads; ++w) {
    ep_job* J = &jobs[w];
    J->s = s;
    J->m = m;
    J->h = h;
    J->g = g;
    J->params = params;
    J->e_begin = E * w / threads;
    J->e_end = E * (w + 1) / threads;
    J->T = T;
    J->episode_offset = episode_offset;
    J->seed = explore_seed;
    J->init_idx = init_idx;
    J->idx_out = idx_out;
    J->score_out = score_out;
    J->actions_out = actions_out;
    J->logp_out = logp_out;
    J->value_out = value_out;
  }
  if (threads == 1) {
    run_episode_range(&jobs[0]);
  } else {
    for (int w = 0; w < threads; ++w) pthread_create(&th[w], NULL, run_episode_range, &jobs[w]);
    for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  }
  free(jobs);
  free(th);
  return 0;
}

/* ======================================================================
 * sa_search (the AutoTVM simulated-annealing baseline; no
 * reference code — builder-pinned):
 *  chain c (global id gc = chain_offset + c): Θ_0 = seeds[c], f_0 = pred(Θ_0),
 *  temp = T0. Step t draws u_j = hash01(sa_seed, (gc*T + t)*3 + j), j = 0,1,2:
 *  knob = (int)(u_0 * D); dir = u_1 < 0.5 ? -1 : +1; the proposal moves that
 *  knob saturating (design_space.cpp:175-187); Δ = pred(proposal) - f_t;
 *  accept iff Δ >= 0 || u_2 < exp(Δ / temp) (portable exp);
 *  Θ_{t+1} = accept ? proposal : Θ_t; temp = temp * cooling_rate.
 *  Outputs: states [E][T+1][D], their predicted fitness [E][T+1], accepted [E][T].
 * ==================================================================== */
typedef struct {
  const ko_space* s;
  const ko_gbt* m;
  int64_t c_begin, c_end;
  int32_t T;
  int64_t chain_offset;
  uint64_t seed;
  double t0, rate;
  const int32_t* init_idx;
  int32_t* idx_out;
  double* score_out;
  uint8_t* acc_out;
} sa_job;

static void* sa_chain_range(void* arg) {
  const sa_job* J = (const sa_job*)arg;
  const int D = J->s->D;
  double* x = (double*)malloc(sizeof(double) * (size_t)D);
  int32_t* prop = (int32_t*)malloc(sizeof(int32_t) * (size_t)D);
  for (int64_t c = J->c_begin; c < J->c_end; ++c) {
    const uint64_t gc = (uint64_t)(J->chain_offset + c);
    int32_t* traj = J->idx_out + c * (int64_t)(J->T + 1) * D;
    double* sc = J->score_out + c * (int64_t)(J->T + 1);
    memcpy(traj, J->init_idx + c * D, sizeof(int32_t) * (size_t)D);
    ko_encode(J->s, traj, x);
    double f = ko_gbt_predict_one(J->m, x);
    sc[0] = f;
    double temp = J->t0;
    for (int32_t t = 0; t < J->T; ++t) {
      const int32_t* cur = traj + (int64_t)t * D;
      int32_t* nxt = traj + (int64_t)(t + 1) * D;
      const uint64_t base = (gc * (uint64_t)J->T + (uint64_t)t) * 3u;
      const double u0 = ko_hash01(J->seed, base), u1 = ko_hash01(J->seed, base + 1),
                   u2 = ko_hash01(J->seed, base + 2);
      const int knob = (int)(u0 * (double)D);
      const int dir = u1 < 0.5 ? -1 : 1;
      memcpy(prop, cur, sizeof(int32_t) * (size_t)D);
      int v = prop[knob] + dir;
      if (v < 0) v = 0;
      if (v > J->s->card[knob] - 1) v = J->s->card[knob] - 1;
      prop[knob] = v;
      ko_encode(J->s, prop, x);
      const double fp = ko_gbt_predict_one(J->m, x);
      const double delta = fp - f;
      const int accept = delta >= 0.0 || u2 < ko_exp(delta / temp);
      memcpy(nxt, accept ? prop : cur, sizeof(int32_t) * (size_t)D);
      if (accept) f = fp;
      sc[t + 1] = f;
      if (J->acc_out) J->acc_out[c * (int64_t)J->T + t] = (uint8_t)accept;
      temp = temp * J->rate;
    }
  }
  free(x);
  free(prop);
  return NULL;
}

int ko_sa_search(const ko_space* s, const ko_gbt* m, int64_t E, int32_t T, int64_t chain_offset,
                 uint64_t sa_seed, double t0, double rate, const int32_t* init_idx, int32_t* idx_out,
                 double* score_out, uint8_t* acc_out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > E) threads = (int)(E > 0 ? E : 1);
  sa_job* jobs = (sa_job*)calloc((size_t)threads, sizeof(sa_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int w = 0; w < threads; ++w) {
    sa_job* J = &jobs[w];
    J->s = s;
    J->m = m;
    J->c_begin = E * w / threads;
    J->c_end = E * (w + 1) / threads;
    J->T = T;
    J->chain_offset = chain_offset;
    J->seed = sa_seed;
    J->t0 = t0;
    J->rate = rate;
    J->init_idx = init_idx;
    J->idx_out = idx_out;
    J->score_out = score_out;
    J->acc_out = acc_out;
  }
  if (threads == 1) {
    sa_chain_range(&jobs[0]);
  } else {
    for (int w = 0; w < threads; ++w) pthread_create(&th[w], NULL, sa_chain_range, &jobs[w]);
    for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  }
  free(jobs);
  free(th);
  return 0;
}

/* ======================================================================
 * make_candidate_set (sampling.cpp:16-31)
 * ==================================================================== */
typedef struct {
  uint64_t id;
  int64_t row;
  double pred;
} cand_key;

static int cmp_id_row(const void* a, const void* b) {
  const cand_key* x = (const cand_key*)a;
  const cand_key* y = (const cand_key*)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->row < y->row ? -1 : (x->row > y->row);
}
static int cmp_rank(const void* a, const void* b) {
  const cand_key* x = (const cand_key*)a;
  const cand_key* y = (const cand_key*)b;
  if (x->pred != y->pred) return x->pred > y->pred ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

int64_t ko_make_candidate_set(int D, const int32_t* idx, const uint64_t* ids, const double* pred,
                              int64_t n, int64_t* out_rows) {
  (void)D;
  (void)idx;
  cand_key* k = (cand_key*)malloc(sizeof(cand_key) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    k[i].id = ids[i];
    k[i].row = i;
    k[i].pred = pred[i];
  }
  qsort(k, (size_t)n, sizeof(cand_key), cmp_id_row);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (i == 0 || k[i].id != k[i - 1].id) k[m++] = k[i]; /* first occurrence wins */
  qsort(k, (size_t)m, sizeof(cand_key), cmp_rank);
  for (int64_t i = 0; i < m; ++i) out_rows[i] = k[i].row;
  free(k);
  return m;
}

/* ======================================================================
 * K-means (sampling.cpp:39-175) with the Eigen reduction orders of
 * strided-row squaredNorm is sequential over d
 * (A.2); contiguous VectorXd sum()/squaredNorm() is the SSE2 two-packet
 * order (A.3).
 * ==================================================================== */
static double row_d2(const double* p, const double* c, int D) { /* A.2 */
  double d = p[0] - c[0];
  double s = d * d;
  for (int j = 1; j < D; ++j) {
    d = p[j] - c[j];
    s = s + d * d;
  }
  return s;
}

static double eigen_vec_sum(const double* x, int64_t n) { /* A.3 */
  if (n == 0) return 0.0;
  const int64_t aligned2 = (n / 4) * 4, aligned = (n / 2) * 2;
  if (aligned == 0) {
    double r = x[0];
    for (int64_t i = 1; i < n; ++i) r = r + x[i];
    return r;
  }
  double a0 = x[0], a1 = x[1];
  if (aligned > 2) {
    double b0 = x[2], b1 = x[3];
    for (int64_t i = 4; i < aligned2; i += 4) {
      a0 = a0 + x[i];
      a1 = a1 + x[i + 1];
      b0 = b0 + x[i + 2];
      b1 = b1 + x[i + 3];
    }
    a0 = a0 + b0;
    a1 = a1 + b1;
    if (aligned > aligned2) {
      a0 = a0 + x[aligned2];
      a1 = a1 + x[aligned2 + 1];
    }
  }
  double r = a0 + a1;
  for (int64_t i = aligned; i < n; ++i) r = r + x[i];
  return r;
}

static void assign_points(const double* P, int64_t N, int D, const double* C, int k, int32_t* a) {
  for (int64_t i = 0; i < N; ++i) { /* sampling.cpp:39-54 */
    double best = INFINITY;
    int bc = 0;
    for (int c = 0; c < k; ++c) {
      const double d2 = row_d2(P + i * D, C + (int64_t)c * D, D);
      if (d2 < best) {
        best = d2;
        bc = c;
      }
    }
    a[i] = bc;
  }
}

static double assignment_loss(const double* P, int64_t N, int D, const double* C,
                              const int32_t* a) { /* sampling.cpp:56-63 */
  double loss = 0.0;
  for (int64_t i = 0; i < N; ++i) loss += row_d2(P + i * D, C + (int64_t)a[i] * D, D);
  return loss;
}

static void kmeanspp_init(const double* P, int64_t N, int D, int k, ko_rng* r, double* C,
                          double* d2) { /* sampling.cpp:65-96 */
  memcpy(C, P + (int64_t)rng_below(r, (uint64_t)N) * D, sizeof(double) * (size_t)D);
  for (int64_t i = 0; i < N; ++i) d2[i] = row_d2(P + i * D, C, D);
  for (int c = 1; c < k; ++c) {
    const double total = eigen_vec_sum(d2, N);
    int64_t pick;
    if (total <= 0.0) {
      pick = (int64_t)rng_below(r, (uint64_t)N);
    } else {
      const double rr = rng_uniform01(r) * total;
      double cum = 0.0;
      pick = N - 1;
      for (int64_t i = 0; i < N; ++i) {
        cum += d2[i];
        if (cum > rr) {
          pick = i;
          break;
        }
      }
    }
    memcpy(C + (int64_t)c * D, P + pick * D, sizeof(double) * (size_t)D);
    for (int64_t i = 0; i < N; ++i) {
      const double v = row_d2(P + i * D, C + (int64_t)c * D, D);
      if (v < d2[i]) d2[i] = v; /* std::min(d2, v): keeps d2 unless v < d2 */
    }
  }
}

/* Returns 0, or 4 when the Lloyd monotonicity assertion fires (sampling.cpp:142-144). */
static int lloyd(const double* P, int64_t N, int D, int k, ko_rng* r, int max_iters, double* C,
                 int32_t* a, double* loss, double* iter_losses, int32_t* n_losses) {
  double* d2 = (double*)malloc(sizeof(double) * (size_t)N);
  double* next = (double*)malloc(sizeof(double) * (size_t)k * D);
  int32_t* na = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  uint8_t* claimed = (uint8_t*)malloc((size_t)N);
  int rc = 0;
  kmeanspp_init(P, N, D, k, r, C, d2);
  assign_points(P, N, D, C, k, a);
  *loss = assignment_loss(P, N, D, C, a);
  int nl = 0;
  iter_losses[nl++] = *loss;
  for (int it = 0; it < max_iters; ++it) {
    memset(next, 0, sizeof(double) * (size_t)k * D);
    memset(counts, 0, sizeof(int32_t) * (size_t)k);
    for (int64_t i = 0; i < N; ++i) { /* :112-116, member order */
      const int c = a[i];
      for (int j = 0; j < D; ++j) next[(int64_t)c * D + j] = next[(int64_t)c * D + j] + P[i * D + j];
      ++counts[c];
    }
    memset(claimed, 0, (size_t)N);
    for (int c = 0; c < k; ++c) {
      if (counts[c] > 0) {
        for (int j = 0; j < D; ++j)
          next[(int64_t)c * D + j] = next[(int64_t)c * D + j] / (double)counts[c];
      } else { /* :122-136 farthest unclaimed point from its OLD centroid */
        double worst = -1.0;
        int64_t wi = 0;
        for (int64_t i = 0; i < N; ++i) {
          if (claimed[i]) continue;
          const double v = row_d2(P + i * D, C + (int64_t)a[i] * D, D);
          if (v > worst) {
            worst = v;
            wi = i;
          }
        }
        claimed[wi] = 1;
        memcpy(next + (int64_t)c * D, P + wi * D, sizeof(double) * (size_t)D);
      }
    }
    assign_points(P, N, D, next, k, na);
    const double nloss = assignment_loss(P, N, D, next, na);
    if (nloss > *loss + 1e-9) {
      rc = 4;
      break;
    }
    const int converged = memcmp(na, a, sizeof(int32_t) * (size_t)N) == 0;
    memcpy(C, next, sizeof(double) * (size_t)k * D);
    memcpy(a, na, sizeof(int32_t) * (size_t)N);
    *loss = nloss;
    iter_losses[nl++] = nloss;
    if (converged) break;
  }
  *n_losses = nl;
  free(d2);
  free(next);
  free(na);
  free(counts);
  free(claimed);
  return rc;
}

int ko_kmeans_run(const double* points, int64_t N, int D, int k, uint64_t seed, int max_iters,
                  int restarts, double* centroids, int32_t* assignments, double* loss,
                  double* iteration_losses, int32_t* num_losses) { /* sampling.cpp:157-175 */
  if (N == 0) return 1;
  if (k < 1 || k > N) return 1;
  double* C = (double*)malloc(sizeof(double) * (size_t)k * D);
  int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  double* il = (double*)malloc(sizeof(double) * (size_t)(max_iters + 1));
  int have = 0;
  double best = 0.0;
  const int R = restarts > 1 ? restarts : 1;
  int rc = 0;
  for (int rr = 0; rr < R; ++rr) {
    ko_rng rng = {ko_seed_combine(seed, (uint64_t)rr)};
    double l;
    int32_t nl;
    rc = lloyd(points, N, D, k, &rng, max_iters, C, a, &l, il, &nl);
    if (rc) break;
    if (!have || l < best) { /* strictly smaller replaces (earliest wins ties) */
      have = 1;
      best = l;
      memcpy(centroids, C, sizeof(double) * (size_t)k * D);
      memcpy(assignments, a, sizeof(int32_t) * (size_t)N);
      memcpy(iteration_losses, il, sizeof(double) * (size_t)nl);
      *num_losses = nl;
      *loss = l;
    }
  }
  free(C);
  free(a);
  free(il);
  return rc;
}

int ko_adaptive_sweep(const double* points, int64_t N, int D, double threshold, int k_min,
                      int k_max_exclusive, int max_iters, int restarts, uint64_t rng_seed,
                      int32_t* k_chosen, double* centroids, int32_t* assignments, double* loss,
                      double* k_losses, int32_t* num_k) { /* sampling.cpp:413-446 */
  if (N == 0) return 1;
  if (k_min >= k_max_exclusive || k_min < 1) return 1;
  if (threshold <= 1.0) return 1;
  const int k_lo = k_min < N ? k_min : (int)N;
  const int k_hi = (k_max_exclusive - 1) < N ? (k_max_exclusive - 1) : (int)N;
  double prev = INFINITY;
  double* il = (double*)malloc(sizeof(double) * (size_t)(max_iters + 1));
  int nk = 0;
  int rc = 0;
  for (int k = k_lo; k <= k_hi; ++k) {
    int32_t nl;
    rc = ko_kmeans_run(points, N, D, k, ko_seed_combine(rng_seed, (uint64_t)k), max_iters,
                       restarts, centroids, assignments, loss, il, &nl);
    if (rc) break;
    k_losses[nk++] = *loss;
    *k_chosen = k;
    if (threshold * *loss >= prev) break;
    prev = *loss;
  }
  *num_k = nk;
  free(il);
  return rc;
}

/* ======================================================================
 * snap_centroid (sampling.cpp:202-235)
 * ==================================================================== */
void ko_snap_centroid(const ko_space* s, const double* centroid, const int32_t* cand_idx,
                      const uint64_t* cand_ids, int64_t n, int32_t* out) {
  const int D = s->D;
  for (int i = 0; i < D; ++i) {
    const int card = s->card[i];
    int idx = (int)floor(centroid[i] * (double)(card - 1) + 0.5); /* A.8 */
    if (idx < 0) idx = 0;
    if (idx > card - 1) idx = card - 1;
    out[i] = idx;
  }
  if (ko_validate(s, out)) return;
  int64_t best = -1;
  double best_d2 = INFINITY;
  int best_valid = 0;
  double x[256], diff2[256];
  for (int64_t c = 0; c < n; ++c) {
    const int32_t* ci = cand_idx + c * D;
    const int cv = ko_validate(s, ci);
    if (best_valid && !cv) continue;
    ko_encode(s, ci, x);
    for (int j = 0; j < D; ++j) {
      const double d = x[j] - centroid[j];
      diff2[j] = d * d;
    }
    const double d2 = eigen_vec_sum(diff2, D); /* contiguous temporary: A.3 */
    const int upgrade = cv && !best_valid;
    const int better = d2 < best_d2 || (d2 == best_d2 && best >= 0 && cand_ids[c] < cand_ids[best]);
    if (best < 0 || upgrade || (cv == best_valid && better)) {
      best = c;
      best_d2 = d2;
      best_valid = cv;
    }
  }
  if (best >= 0) memcpy(out, cand_idx + best * D, sizeof(int32_t) * (size_t)D);
}

/* ======================================================================
 * PPO training step (ActorCritic::backward and AdamOptimizer
 * are declared at actor_critic.hpp:45-49,66-79 with no definition anywhere in
 * the reference). Builder-pinned arithmetic: every reduction
 * over the batch is a sequential chain in ascending sample order, products
 * accumulated with fma(), everything else separately rounded; the CUDA
 * implementation (csrc/ppo.cu) performs the same operations in the same order.
 * ==================================================================== */

/* actor_critic.hpp:45-49: upstream gradients w.r.t. the logits (B x 3n) and the
 * values (B) -> flat parameter gradient (layout of ac_layout). The cache is the
 * forward pass of the same parameters: states B x n, h0 B x h, hp/hv B x g. */
void ko_ac_backward(int n, int h, int g, const double* p, const double* x, const double* h0,
                    const double* hp, const double* hv, int64_t B, const double* dl, const double* dv,
                    double* grad) {
  const ac_off o = ac_layout(n, h, g);
  double* dzv = (double*)malloc(sizeof(double) * (size_t)(B * (2 * g + h)));
  double* dzp = dzv + B * g;
  double* dz0 = dzp + B * g;
  for (int64_t b = 0; b < B; ++b) {
    for (int j = 0; j < g; ++j) {
      const double t = hv[b * g + j] * hv[b * g + j];
      dzv[b * g + j] = (dv[b] * p[o.wv2 + j]) * (1.0 - t);
    }
    for (int j = 0; j < g; ++j) {
      double acc = 0.0;
      for (int a = 0; a < 3 * n; ++a) acc = fma(p[o.wp2 + (int64_t)j * 3 * n + a], dl[b * 3 * n + a], acc);
      const double t = hp[b * g + j] * hp[b * g + j];
      dzp[b * g + j] = acc * (1.0 - t);
    }
    for (int i = 0; i < h; ++i) {
      double acc = 0.0;
      for (int j = 0; j < g; ++j) acc = fma(p[o.wp1 + (int64_t)i * g + j], dzp[b * g + j], acc);
      for (int j = 0; j < g; ++j) acc = fma(p[o.wv1 + (int64_t)i * g + j], dzv[b * g + j], acc);
      const double t = h0[b * h + i] * h0[b * h + i];
      dz0[b * h + i] = acc * (1.0 - t);
    }
  }
  /* parameter gradients: sum over the batch, ascending b */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < h; ++j) {
      double acc = 0.0;
      for (int64_t b = 0; b < B; ++b) acc = fma(dz0[b * h + j], x[b * n + i], acc);
      grad[o.w0 + (int64_t)i * h + j] = acc;
    }
  for (int j = 0; j < h; ++j) {
    double acc = 0.0;
    for (int64_t b = 0; b < B; ++b) acc = acc + dz0[b * h + j];
    grad[o.b0 + j] = acc;
  }
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < g; ++j) {
      double ap = 0.0, av = 0.0;
      for (int64_t b = 0; b < B; ++b) {
        ap = fma(dzp[b * g + j], h0[b * h + i], ap);
        av = fma(dzv[b * g + j], h0[b * h + i], av);
      }
      grad[o.wp1 + (int64_t)i * g + j] = ap;
      grad[o.wv1 + (int64_t)i * g + j] = av;
    }
  for (int j = 0; j < g; ++j) {
    double ap = 0.0, av = 0.0, aw = 0.0;
    for (int64_t b = 0; b < B; ++b) {
      ap = ap + dzp[b * g + j];
      av = av + dzv[b * g + j];
      aw = fma(dv[b], hv[b * g + j], aw);
    }
    grad[o.bp1 + j] = ap;
    grad[o.bv1 + j] = av;
    grad[o.wv2 + j] = aw;
  }
  for (int j = 0; j < g; ++j)
    for (int a = 0; a < 3 * n; ++a) {
      double acc = 0.0;
      for (int64_t b = 0; b < B; ++b) acc = fma(dl[b * 3 * n + a], hp[b * g + j], acc);
      grad[o.wp2 + (int64_t)j * 3 * n + a] = acc;
    }
  for (int a = 0; a < 3 * n; ++a) {
    double acc = 0.0;
    for (int64_t b = 0; b < B; ++b) acc = acc + dl[b * 3 * n + a];
    grad[o.bp2 + a] = acc;
  }
  {
    double acc = 0.0;
    for (int64_t b = 0; b < B; ++b) acc = acc + dv[b];
    grad[o.bv2] = acc;
  }
  free(dzv);
}

/* AdamOptimizer::step (actor_critic.hpp:66-79) for step number t (1-based); the bias
 * corrections 1 - beta^t are products of t factors (no pow). */
void ko_adam_bias(double beta1, double beta2, int64_t t, double* bc1, double* bc2) {
  double p1 = 1.0, p2 = 1.0;
  for (int64_t i = 0; i < t; ++i) {
    p1 = p1 * beta1;
    p2 = p2 * beta2;
  }
  *bc1 = 1.0 - p1;
  *bc2 = 1.0 - p2;
}

void ko_adam_step(int64_t dim, double* params, const double* grad, double* m, double* v, double lr,
                  double beta1, double beta2, double eps, double bc1, double bc2) {
  for (int64_t i = 0; i < dim; ++i) {
    const double gi = grad[i];
    m[i] = beta1 * m[i] + (1.0 - beta1) * gi;
    v[i] = beta2 * v[i] + (1.0 - beta2) * (gi * gi);
    const double mh = m[i] / bc1, vh = v[i] / bc2;
    params[i] = params[i] - lr * mh / (sqrt(vh) + eps);
  }
}

/* compute_gae, E episodes of T steps (row-major E x T). */
void ko_compute_gae(int64_t E, int32_t T, const double* rewards, const double* values,
                    const double* terminal_values, double gamma, double lambda, double* adv, double* ret) {
  const double gl = gamma * lambda;
  for (int64_t e = 0; e < E; ++e) {
    double a_next = 0.0;
    for (int32_t t = T - 1; t >= 0; --t) {
      const int64_t k = e * T + t;
      const double vn = t == T - 1 ? terminal_values[e] : values[k + 1];
      const double delta = (rewards[k] + gamma * vn) - values[k];
      a_next = delta + gl * a_next;
      adv[k] = a_next;
      ret[k] = a_next + values[k];
    }
  }
}

/* Advantage normalisation: population mean/variance, sequential sums. */
void ko_normalize_advantages(int64_t N, const double* adv, double* out) {
  double s = 0.0;
  for (int64_t i = 0; i < N; ++i) s = s + adv[i];
  const double mean = s / (double)N;
  double q = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double d = adv[i] - mean;
    q = q + d * d;
  }
  const double sd = sqrt(q / (double)N);
  for (int64_t i = 0; i < N; ++i) out[i] = (adv[i] - mean) / (sd + 1e-8);
}

/* One PPO minibatch step's loss gradients for B samples: the forward
 * outputs (log_probs/probs B x 3n, values B), actions B x n in {-1,0,+1}, old joint
 * log-probs, normalised advantages and returns -> d_logits (B x 3n), d_values (B) of
 * the loss  -mean(min(rho A, clip(rho) A)) + c_v mean((V - R)^2) - c_e mean(H),
 * and the minibatch sums (surrogate, squared value error, entropy). */
void ko_ppo_loss_grad(int n, int64_t B, const double* logp, const double* probs, const double* values,
                      const int8_t* actions, const double* old_logp, const double* adv, const double* ret,
                      double clip_eps, double c_v, double c_e, double* dl, double* dv, double* sums) {
  const double invB = 1.0 / (double)B;
  double ss = 0.0, sv = 0.0, se = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    double lp = 0.0, H = 0.0;
    for (int d = 0; d < n; ++d) lp = lp + logp[b * 3 * n + 3 * d + (actions[b * n + d] + 1)];
    const double rho = ko_exp(lp - old_logp[b]);
    const double A = adv[b];
    const double un = rho * A;
    const double rc = rho < 1.0 - clip_eps ? 1.0 - clip_eps : (rho > 1.0 + clip_eps ? 1.0 + clip_eps : rho);
    const double cl = rc * A;
    const double s = un <= cl ? un : cl;
    const double gs = un <= cl ? A * rho : 0.0;
    for (int d = 0; d < n; ++d) {
      const double* pk = probs + b * 3 * n + 3 * d;
      const double* lk = logp + b * 3 * n + 3 * d;
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc = acc + pk[k] * lk[k];
      const double Hd = -acc;
      H = H + Hd;
      for (int k = 0; k < 3; ++k) {
        const double ind = (k == actions[b * n + d] + 1) ? 1.0 : 0.0;
        const double t2 = gs * (ind - pk[k]);
        const double t5 = c_e * (pk[k] * (lk[k] + Hd));
        dl[b * 3 * n + 3 * d + k] = invB * (t5 - t2);
      }
    }
    const double diff = values[b] - ret[b];
    dv[b] = invB * ((2.0 * c_v) * diff);
    ss = ss + s;
    sv = sv + diff * diff;
    se = se + H;
  }
  sums[0] = ss;
  sums[1] = sv;
  sums[2] = se;
}

/* ppo_update: N samples (states N x n, actions N x n, old log-probs,
 * advantages, returns); advantages normalised once; num_epochs epochs, each a
 * Fisher-Yates permutation (rng.hpp:88-92) from Rng(seed_combine(seed, epoch)),
 * minibatches of mb consecutive permuted samples (the last may be shorter); per
 * minibatch: forward, loss gradients, backward, one Adam step (state m, v, t in/out).
 * stats[3] = mean over minibatch steps of (policy loss, value loss, entropy). */
int ko_ppo_update(int n, int h, int g, double* params, double* adam_m, double* adam_v, int64_t* adam_t,
                  int64_t N, const double* states, const int8_t* actions, const double* old_logp,
                  const double* adv, const double* ret, int num_epochs, int64_t mb, double lr,
                  double clip_eps, double c_v, double c_e, uint64_t seed, double* stats) {
  if (N <= 0 || mb <= 0 || num_epochs <= 0) return 1;
  const int64_t P = ko_ac_num_params(n, h, g);
  double* an = (double*)malloc(sizeof(double) * (size_t)N);
  ko_normalize_advantages(N, adv, an);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  const int64_t S = mb < N ? mb : N;
  double* xs = (double*)malloc(sizeof(double) * (size_t)(S * (n + h + 2 * g + 9 * n + 6) + P));
  double* h0 = xs + S * n;
  double* hp = h0 + S * h;
  double* hv = hp + S * g;
  double* lg = hv + S * g;
  double* lp = lg + S * 3 * n;
  double* pr = lp + S * 3 * n;
  double* va = pr + S * 3 * n;
  double* ol = va + S;
  double* aa = ol + S;
  double* rr = aa + S;
  double* dv = rr + S;
  double* dl = lg; /* logits are not needed after the forward */
  double* gr = dv + S;
  int8_t* ac = (int8_t*)malloc((size_t)(S * n));
  double tot[3] = {0.0, 0.0, 0.0};
  int64_t steps = 0;
  for (int ep = 0; ep < num_epochs; ++ep) {
    for (int64_t i = 0; i < N; ++i) perm[i] = i;
    ko_rng r = {ko_seed_combine(seed, (uint64_t)ep)};
    for (int64_t i = N; i > 1; --i) {
      const int64_t j = (int64_t)rng_below(&r, (uint64_t)i);
      const int64_t t = perm[i - 1];
      perm[i - 1] = perm[j];
      perm[j] = t;
    }
    for (int64_t s0 = 0; s0 < N; s0 += mb) {
      const int64_t B = N - s0 < mb ? N - s0 : mb;
      for (int64_t b = 0; b < B; ++b) {
        const int64_t k = perm[s0 + b];
        memcpy(xs + b * n, states + k * n, sizeof(double) * (size_t)n);
        memcpy(ac + b * n, actions + k * n, (size_t)n);
        ol[b] = old_logp[k];
        aa[b] = an[k];
        rr[b] = ret[k];
      }
      ko_ac_forward(n, h, g, params, xs, B, h0, hp, hv, lg, lp, pr, va);
      double sums[3];
      ko_ppo_loss_grad(n, B, lp, pr, va, ac, ol, aa, rr, clip_eps, c_v, c_e, dl, dv, sums);
      ko_ac_backward(n, h, g, params, xs, h0, hp, hv, B, dl, dv, gr);
      *adam_t += 1;
      double bc1, bc2;
      ko_adam_bias(0.9, 0.999, *adam_t, &bc1, &bc2);
      ko_adam_step(P, params, gr, adam_m, adam_v, lr, 0.9, 0.999, 1e-8, bc1, bc2);
      const double invB = 1.0 / (double)B;
      tot[0] = tot[0] + (-sums[0]) * invB;
      tot[1] = tot[1] + sums[1] * invB;
      tot[2] = tot[2] + sums[2] * invB;
      ++steps;
    }
  }
  for (int k = 0; k < 3; ++k) stats[k] = tot[k] / (double)steps;
  free(an);
  free(perm);
  free(xs);
  free(ac);
  return 0;
}
