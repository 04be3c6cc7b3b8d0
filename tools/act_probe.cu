// Microbenchmark: cycles per activation unit of the rollout epilogue (act2 pair + fp16 hi/lo
// split), vs warps per SM sub-partition. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/act_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpf(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 act2(float2 y, float S) {
  const float ea = ex2f(fminf(y.x, 63.f)), eb = ex2f(fminf(y.y, 63.f));
  const float2 d = __fadd2_rn(make_float2(ea, eb), make_float2(1.f, 1.f));
  const float R = rcpf(d.x * d.y);
  const float2 r = __fmul2_rn(make_float2(d.y, d.x), make_float2(R, R));
  return __ffma2_rn(r, make_float2(2.f * S, 2.f * S), make_float2(-S, -S));
}
__device__ __forceinline__ float act1(float y, float S) { return fmaf(rcpf(1.0f + ex2f(y)), 2.f * S, -S); }
// 2^y on the FMA pipe: y = n + f (round to nearest via the 1.5*2^23 trick), degree-6 polynomial on
// [-0.5, 0.5] (max rel. error ~1e-7 in fp32), exponent added as an integer. y in [-126, 63].
__device__ __forceinline__ float ex2poly(float y) {
  y = fmaxf(y, -125.f);
  const float t = y + 12582912.f;
  const float f = y - (t - 12582912.f);
  const int n = __float_as_int(t) - 0x4B400000;
  float p = 0.00015337577497120947f;
  p = fmaf(p, f, 0.0013399859890341759f);
  p = fmaf(p, f, 0.009618519805371761f);
  p = fmaf(p, f, 0.05550329014658928f);
  p = fmaf(p, f, 0.24022646248340607f);
  p = fmaf(p, f, 0.6931471824645996f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (n << 23));
}
__device__ __forceinline__ float2 ex2poly2(float2 y) {  // packed: both lanes of a pair on the FMA pipe
  y.x = fmaxf(y.x, -125.f);
  y.y = fmaxf(y.y, -125.f);
  const float2 M = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(y, M);
  const float2 f = __fadd2_rn(y, __fadd2_rn(M, make_float2(-t.x, -t.y)));
  float2 p = make_float2(0.00015337577497120947f, 0.00015337577497120947f);
  p = __ffma2_rn(p, f, make_float2(0.0013399859890341759f, 0.0013399859890341759f));
  p = __ffma2_rn(p, f, make_float2(0.009618519805371761f, 0.009618519805371761f));
  p = __ffma2_rn(p, f, make_float2(0.05550329014658928f, 0.05550329014658928f));
  p = __ffma2_rn(p, f, make_float2(0.24022646248340607f, 0.24022646248340607f));
  p = __ffma2_rn(p, f, make_float2(0.6931471824645996f, 0.6931471824645996f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + ((__float_as_int(t.x) - 0x4B400000) << 23)),
                     __int_as_float(__float_as_int(p.y) + ((__float_as_int(t.y) - 0x4B400000) << 23)));
}
// hybrid pair: unit a on the SFU, unit b on the FMA pipe, one shared reciprocal
__device__ __forceinline__ float2 act2h(float2 y, float S) {
  const float ea = ex2f(fminf(y.x, 63.f)), eb = ex2poly(fminf(y.y, 63.f));
  const float2 d = __fadd2_rn(make_float2(ea, eb), make_float2(1.f, 1.f));
  const float R = rcpf(d.x * d.y);
  const float2 r = __fmul2_rn(make_float2(d.y, d.x), make_float2(R, R));
  return __ffma2_rn(r, make_float2(2.f * S, 2.f * S), make_float2(-S, -S));
}
// both units' exponentials on the FMA pipe (packed), one shared reciprocal on the SFU
__device__ __forceinline__ float2 act2p(float2 y, float S) {
  const float2 e = ex2poly2(make_float2(fminf(y.x, 63.f), fminf(y.y, 63.f)));
  const float2 d = __fadd2_rn(e, make_float2(1.f, 1.f));
  const float R = rcpf(d.x * d.y);
  const float2 r = __fmul2_rn(make_float2(d.y, d.x), make_float2(R, R));
  return __ffma2_rn(r, make_float2(2.f * S, 2.f * S), make_float2(-S, -S));
}
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[32];
  for (int j = 0; j < 32; ++j) v[j] = 0.001f * (threadIdx.x + j) - 0.3f;
  uint32_t acc = 0;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float2 a;
      if (MODE == 0) a = act2(make_float2(v[j], v[j + 1]), 16384.f);
      else if (MODE == 2) a = act2h(make_float2(v[j], v[j + 1]), 16384.f);
      else if (MODE == 3) a = act2p(make_float2(v[j], v[j + 1]), 16384.f);
      else { a.x = act1(v[j], 16384.f); a.y = act1(v[j + 1], 16384.f); }
      const __half2 h = __floats2half2_rn(a.x, a.y);
      const float2 f = __half22float2(h);
      const __half2 l = __float22half2_rn(__fadd2_rn(a, make_float2(-f.x, -f.y)));
      acc += *reinterpret_cast<const uint32_t*>(&h) ^ *reinterpret_cast<const uint32_t*>(&l);
      v[j] = a.x * 1e-5f; v[j + 1] = a.y * 1e-5f;
    }
  }
  long long c1 = clock64();
  float s = 0; for (int j = 0; j < 32; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[4] = {"act2(1.5 MUFU)", "act1(2 MUFU)", "act2h(1 MUFU)", "act2p(0.5 MUFU)"};
  for (int mode = 0; mode < 4; ++mode)
    for (int wps : {1, 2, 3, 4}) {
      const int thr = wps * 4 * 32;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, thr>>>(out, iters, cyc);
        else if (mode == 1) k<1><<<148, thr>>>(out, iters, cyc);
        else if (mode == 2) k<2><<<148, thr>>>(out, iters, cyc);
        else k<3><<<148, thr>>>(out, iters, cyc);
        cudaDeviceSynchronize();
      }
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double units = (double)iters * 32;  // per thread
      printf("%s warps/SMSP %d: %.2f cycles per unit per warp, %.2f cycles per unit-warp per SMSP\n",
             names[mode], wps, c / units, c / units / wps);
    }
  return 0;
}
