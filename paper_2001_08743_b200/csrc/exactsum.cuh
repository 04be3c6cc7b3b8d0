// Exact parallel emulation of SEQUENTIAL fp64 summation of non-negative values.
//
// The reference accumulates centroid sums (sampling.cpp:112-121) and losses
// (sampling.cpp:56-63) as plain left-to-right fp64 chains:
//     s_0 = 0,  s_{i+1} = fl(s_i + x_i),  x_i >= 0.
// Such a chain is order-sensitive, so a tree reduction gives different bits.
// It can nevertheless be evaluated in parallel EXACTLY:
//
//  * while s stays inside one binade [2^e, 2^(e+1)) every value is a multiple
//    of U = 2^(e-52): s = m*U with integer m in [2^52, 2^53). Write x/U = q + f
//    (q integer, 0 <= f < 1; exact because U is a power of two). Round-to-
//    nearest-even gives  fl(s + x) = (m + q + [f > 1/2] + [f == 1/2 and (m+q)
//    odd]) * U  as long as the result stays below 2^(e+1).
//  * so a segment of the sequence acts on m as  m -> m + F(m mod 2): two
//    integers F0, F1 (start parity even / odd), computed independently per
//    segment in parallel under the binade predicted by an approximate prefix;
//  * one thread then composes the segment maps in order starting from the
//    exact running value; whenever the running value is not in the predicted
//    binade or the segment would leave it, that segment is summed by the plain
//    sequential chain (exact by definition). Both branches yield the reference
//    bits; the maps only skip work.
// Cost: O(n) parallel + O(n / L) sequential integer steps + O(L) per binade
// crossing (~log2 n crossings per chain).
#pragma once

#include <cstdint>

#include "device.cuh"

namespace kt {
namespace xsum {

constexpr int kSeg = 256;  // elements per segment

struct SegMap {
  uint64_t F0, F1;  // increments of m (units of U) for even / odd start parity
  int32_t e;        // binade the map assumes (unbiased exponent of the running sum)
  int32_t ok;       // 0: must be summed sequentially; 1: valid in binade e;
                    // 2: identity (every element is +0: s + 0 == s for any s >= 0)
};

// Identity map if every element of the segment is zero.
template <class At>
__device__ SegMap zero_segment_map(At at, int len) {
  for (int i = 0; i < len; ++i)
    if (at(i) != 0.0) return SegMap{0, 0, 0, 0};
  return SegMap{0, 0, 0, 2};
}

__device__ __forceinline__ int binade_of(double s) {
  return (int)((__double_as_longlong(s) >> 52) & 0x7FF) - 1023;
}

// Map of one segment under binade e. `at(i)` returns element i (0 <= i < len).
template <class At>
__device__ SegMap segment_map(At at, int len, int e) {
  SegMap r{0, 0, e, 1};
  if (e < -960 || e > 1000) {
    r.ok = 0;
    return r;
  }
  const double inv_u = __longlong_as_double((long long)(uint64_t)(1023 + 52 - e) << 52);  // 2^(52-e)
  uint64_t f0 = 0, f1 = 0;
  uint32_t p0 = 0, p1 = 1;  // parity of the running m for each start parity
  for (int i = 0; i < len; ++i) {
    const double xs = dmul(at(i), inv_u);  // exact power-of-two scaling
    if (!(xs < 4503599627370496.0)) {      // >= 2^52 (or NaN): certainly leaves the binade
      r.ok = 0;
      return r;
    }
    const double qd = floor(xs);
    const double fr = dsub(xs, qd);
    const uint64_t q = (uint64_t)qd;
    const uint32_t gt = fr > 0.5 ? 1u : 0u;
    const uint32_t tie = fr == 0.5 ? 1u : 0u;
    const uint32_t qp = (uint32_t)(q & 1u);
    const uint64_t d0 = q + gt + (tie & (p0 ^ qp));
    const uint64_t d1 = q + gt + (tie & (p1 ^ qp));
    f0 += d0;
    f1 += d1;
    p0 ^= (uint32_t)(d0 & 1u);
    p1 ^= (uint32_t)(d1 & 1u);
    if (f0 >= (1ull << 53) || f1 >= (1ull << 53)) {
      r.ok = 0;
      return r;
    }
  }
  r.F0 = f0;
  r.F1 = f1;
  return r;
}

// Apply a segment map to the exact running value s if valid; returns false
// when the caller must sum the segment sequentially.
__device__ __forceinline__ bool apply_map(double& s, const SegMap& m) {
  if (m.ok == 2) return true;
  if (!m.ok || !(s > 0.0)) return false;
  const uint64_t b = (uint64_t)__double_as_longlong(s);
  const int e = (int)((b >> 52) & 0x7FF) - 1023;
  if (e != m.e || ((b >> 52) & 0x7FF) == 0) return false;
  const uint64_t mant = (b & ((1ull << 52) - 1)) | (1ull << 52);
  const uint64_t nm = mant + ((mant & 1u) ? m.F1 : m.F0);
  if (nm >= (1ull << 53)) return false;
  s = __longlong_as_double((long long)((b & 0xFFF0000000000000ull) | (nm - (1ull << 52))));
  return true;
}

}  // namespace xsum
}  // namespace kt
