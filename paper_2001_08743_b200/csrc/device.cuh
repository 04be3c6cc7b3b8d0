// Device helpers: RNG (rng.hpp), exact-order fp64 arithmetic, the portable
// transcendental functions and the validity-rule evaluator.
#pragma once

#include <cstdint>

#include "internal.cuh"

namespace kt {

// ---------------------------------------------------------------- exact fp64
// Explicit round-to-nearest intrinsics: never contracted into FMA, so every
// expression below evaluates exactly as the x86-64 SSE2 reference build does.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------- rng.hpp:16-47
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t seed_combine(uint64_t a, uint64_t b) {
  return mix64(a + 0x9E3779B97F4A7C15ULL + mix64(b));
}
__device__ __forceinline__ double hash01(uint64_t seed, uint64_t counter) {
  const uint64_t u = mix64(seed ^ mix64(counter + 0x9E3779B97F4A7C15ULL));
  return dmul((double)(u >> 11), 0x1.0p-53);
}
// Rng (rng.hpp:50-69) with the state held by the caller.
__host__ __device__ __forceinline__ uint64_t rng_next(uint64_t& s) {
  s += 0x9E3779B97F4A7C15ULL;
  return mix64(s);
}
__device__ __forceinline__ double rng_uniform01(uint64_t& s) {
  return dmul((double)(rng_next(s) >> 11), 0x1.0p-53);
}
__host__ __device__ __forceinline__ uint64_t rng_below(uint64_t& s, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t r = rng_next(s);
    if (r >= threshold) return r % n;
  }
}

// ---------------------------------------------------------------- portable math
// Device restatement of oracle/ktune_oracle.c ko_exp/ko_log/ko_tanh (same
// schemes, constants and operation order); tests/test_gpu_math.py checks the
// two bit-for-bit.
__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double((long long)u); }

__device__ inline double kt_exp(double x) {
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
    k = (int)dadd(dmul(invln2, x), (x < 0.0 ? -0.5 : 0.5));
    const double t = (double)k;
    hi = dsub(x, dmul(t, ln2HI));
    lo = dmul(t, ln2LO);
    r = dsub(hi, lo);
  } else if (ax < 3.725290298461914e-09) {
    return dadd(1.0, x);
  } else {
    r = x;
  }
  const double t = dmul(r, r);
  const double poly = dadd(P1, dmul(t, dadd(P2, dmul(t, dadd(P3, dmul(t, dadd(P4, dmul(t, P5))))))));
  const double c = dsub(r, dmul(t, poly));
  if (k == 0) return dsub(1.0, dsub(ddiv(dmul(r, c), dsub(c, 2.0)), r));
  const double y = dsub(1.0, dsub(dsub(lo, ddiv(dmul(r, c), dsub(2.0, c))), hi));
  if (k >= -1021) return bitsd(dbits(y) + ((uint64_t)(int64_t)k << 52));
  return dmul(bitsd(dbits(y) + ((uint64_t)(int64_t)(k + 1000) << 52)), 9.33263618503218878990e-302);
}

__device__ inline double kt_log(double x) {
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
    if (((hx & 0x7fffffff) | lx) == 0) return bitsd(0xFFF0000000000000ULL);
    if (hx < 0) return bitsd(0x7FF8000000000000ULL);
    k -= 54;
    x = dmul(x, two54);
    u = dbits(x);
    hx = (int32_t)(u >> 32);
  }
  if (hx >= 0x7ff00000) return dadd(x, x);
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int32_t i0 = (hx + 0x95f64) & 0x100000;
  x = bitsd(((uint64_t)(uint32_t)(hx | (i0 ^ 0x3ff00000)) << 32) | (dbits(x) & 0xFFFFFFFFULL));
  k += (i0 >> 20);
  const double f = dsub(x, 1.0);
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double dk = (double)k;
      return dadd(dmul(dk, ln2_hi), dmul(dk, ln2_lo));
    }
    const double R = dmul(dmul(f, f), dsub(0.5, dmul(0.33333333333333333, f)));
    if (k == 0) return dsub(f, R);
    const double dk = (double)k;
    return dsub(dmul(dk, ln2_hi), dsub(dsub(R, dmul(dk, ln2_lo)), f));
  }
  const double s = ddiv(f, dadd(2.0, f));
  const double dk = (double)k;
  const double z = dmul(s, s);
  int32_t i = hx - 0x6147a;
  const double w = dmul(z, z);
  const int32_t j = 0x6b851 - hx;
  const double t1 = dmul(w, dadd(Lg2, dmul(w, dadd(Lg4, dmul(w, Lg6)))));
  const double t2 = dmul(z, dadd(Lg1, dmul(w, dadd(Lg3, dmul(w, dadd(Lg5, dmul(w, Lg7)))))));
  i |= j;
  const double R = dadd(t2, t1);
  if (i > 0) {
    const double hfsq = dmul(dmul(0.5, f), f);
    if (k == 0) return dsub(f, dsub(hfsq, dmul(s, dadd(hfsq, R))));
    return dsub(dmul(dk, ln2_hi), dsub(dsub(hfsq, dadd(dmul(s, dadd(hfsq, R)), dmul(dk, ln2_lo))), f));
  }
  if (k == 0) return dsub(f, dmul(s, dsub(f, R)));
  return dsub(dmul(dk, ln2_hi), dsub(dsub(dmul(s, dsub(f, R)), dmul(dk, ln2_lo)), f));
}

__device__ inline double kt_tanh(double x) {
  const double P0 = -9.64399179425052238628E-1, P1 = -9.92877231001918586564E1,
               P2 = -1.61468768441708447952E3;
  const double Q0 = 1.12811678491632931402E2, Q1 = 2.23548839060100448583E3,
               Q2 = 4.84406305325125486048E3;
  if (x == 0.0) return x;
  double z = fabs(x);
  if (z > 354.891356446691998) return x > 0.0 ? 1.0 : -1.0;
  if (z >= 0.625) {
    const double s = kt_exp(dadd(z, z));
    z = dsub(1.0, ddiv(2.0, dadd(s, 1.0)));
    if (x < 0.0) z = -z;
    return z;
  }
  const double s = dmul(x, x);
  const double p = dadd(dmul(dadd(dmul(P0, s), P1), s), P2);
  const double q = dadd(dmul(dadd(dmul(dadd(s, Q0), s), Q1), s), Q2);
  z = ddiv(p, q);
  z = dmul(dmul(x, s), z);
  return dadd(x, z);
}

// Branch-free evaluation of kt_tanh for SIMT lanes with mixed |x| (same
// operations as kt_tanh on every input, so bit-identical): both the rational
// branch and the exp branch are evaluated and selected. For |x| >= 0.625 the
// exp argument 2|x| lies in [1.25, 709.78], where kt_exp always takes the
// reduction path with 2 <= k <= 1024, so that path is inlined without its
// range checks.
__device__ __forceinline__ double kt_tanh_bf(double x) {
  const double ln2HI = 6.93147180369123816490e-01;
  const double ln2LO = 1.90821492927058770002e-10;
  const double invln2 = 1.44269504088896338700e+00;
  const double P1 = 1.66666666666666019037e-01;
  const double P2 = -2.77777777770155933842e-03;
  const double P3 = 6.61375632143793436117e-05;
  const double P4 = -1.65339022054652515390e-06;
  const double P5 = 4.13813679705723846039e-08;
  const double Q0 = 1.12811678491632931402E2, Q1 = 2.23548839060100448583E3,
               Q2 = 4.84406305325125486048E3;
  const double T0 = -9.64399179425052238628E-1, T1 = -9.92877231001918586564E1,
               T2 = -1.61468768441708447952E3;
  const double z = fabs(x);
  // exp branch on ze = clamp(z, 0.625, 354.89...) (identity where it is selected)
  const double ze = fmin(fmax(z, 0.625), 354.891356446691998);
  const double xx = dadd(ze, ze);
  const int k = (int)dadd(dmul(invln2, xx), 0.5);
  const double t = (double)k;
  const double hi = dsub(xx, dmul(t, ln2HI));
  const double lo = dmul(t, ln2LO);
  const double r = dsub(hi, lo);
  const double tt = dmul(r, r);
  const double poly = dadd(P1, dmul(tt, dadd(P2, dmul(tt, dadd(P3, dmul(tt, dadd(P4, dmul(tt, P5))))))));
  const double c = dsub(r, dmul(tt, poly));
  const double y = dsub(1.0, dsub(dsub(lo, ddiv(dmul(r, c), dsub(2.0, c))), hi));
  const double s = bitsd(dbits(y) + ((uint64_t)(int64_t)k << 52));
  double ze_t = dsub(1.0, ddiv(2.0, dadd(s, 1.0)));
  ze_t = x < 0.0 ? -ze_t : ze_t;
  // rational branch
  const double s2 = dmul(x, x);
  const double p = dadd(dmul(dadd(dmul(T0, s2), T1), s2), T2);
  const double q = dadd(dmul(dadd(dmul(dadd(s2, Q0), s2), Q1), s2), Q2);
  const double zp = dadd(x, dmul(dmul(x, s2), ddiv(p, q)));
  double res = z >= 0.625 ? ze_t : zp;
  res = z > 354.891356446691998 ? (x > 0.0 ? 1.0 : -1.0) : res;
  return x == 0.0 ? x : res;
}

// Per-knob log-softmax over {dec, stay, inc} (actor_critic.hpp:13-14).
struct Knob3 {
  double lp[3], p[3];
};
__device__ __forceinline__ Knob3 softmax3(double l0, double l1, double l2) {
  double m = l0;
  if (l1 > m) m = l1;
  if (l2 > m) m = l2;
  const double e0 = kt_exp(dsub(l0, m)), e1 = kt_exp(dsub(l1, m)),
               e2 = kt_exp(dsub(l2, m));
  const double s = dadd(dadd(e0, e1), e2);
  const double lse = dadd(m, kt_log(s));
  Knob3 r;
  r.lp[0] = dsub(l0, lse);
  r.lp[1] = dsub(l1, lse);
  r.lp[2] = dsub(l2, lse);
  r.p[0] = ddiv(e0, s);
  r.p[1] = ddiv(e1, s);
  r.p[2] = ddiv(e2, s);
  return r;
}

// ---------------------------------------------------------------- validity.cpp:162-204
template <class IdxAt>
__device__ inline bool rule_eval(const KtSpaceParams& sp, IdxAt idx_at) {
  if (sp.nops == 0) return true;
  __int128 st[16];
  int top = 0;
  for (int k = 0; k < sp.nops; ++k) {
    const int code = sp.op_code[k];
    if (code == KTUNE_RULE_PUSH_CONST) {
      st[top++] = sp.op_arg[k];
    } else if (code == KTUNE_RULE_PUSH_KNOB) {
      const int d = (int)sp.op_arg[k];
      st[top++] = sp.values[sp.val_off[d] + idx_at(d)];
    } else if (code == KTUNE_RULE_ADD) {
      --top;
      st[top - 1] += st[top];
    } else if (code == KTUNE_RULE_MUL) {
      --top;
      st[top - 1] *= st[top];
    } else if (code == KTUNE_RULE_LE) {
      return st[top - 2] <= st[top - 1];
    } else if (code == KTUNE_RULE_LT) {
      return st[top - 2] < st[top - 1];
    } else {
      return st[top - 2] == st[top - 1];
    }
  }
  return true;
}

// Row loads of knob indices (uint8 / uint16).
template <class IdxT>
__device__ __forceinline__ int load_idx(const IdxT* row, int d) {
  return (int)row[d];
}

}  // namespace kt
