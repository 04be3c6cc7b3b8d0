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
  for (int mode = 0; mode < 2; ++mode)
    for (int wps : {1, 2, 3, 4, 6, 8}) {
      const int thr = wps * 4 * 32;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, thr>>>(out, iters, cyc); else k<1><<<148, thr>>>(out, iters, cyc);
        cudaDeviceSynchronize();
      }
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double units = (double)iters * 32;  // per thread
      printf("%s warps/SMSP %d: %.2f cycles per unit per warp, %.2f cycles per unit-warp per SMSP\n",
             mode ? "act1(2 MUFU)" : "act2(1.5 MUFU)", wps, c / units, c / units / wps);
    }
  return 0;
}
