// Microbenchmark: SFU (MUFU) and conversion throughput per SM per clock on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpf(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int OP>
__global__ void k(float* out, int iters) {
  float v[16];
  for (int j = 0; j < 16; ++j) v[j] = 0.001f * (threadIdx.x + j);
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (OP == 0) v[j] = ex2f(v[j]);
      else if (OP == 1) v[j] = rcpf(v[j] + 1.0f);
      else if (OP == 2) { __half2 h = __floats2half2_rn(v[j], v[j] + 1.f); acc += *reinterpret_cast<uint32_t*>(&h); v[j] += 1e-7f; }
      else if (OP == 3) { v[j] = fmaf(v[j], 1.0001f, 1e-7f); }
      else if (OP == 4) {  // the rollout's activation: y -> 2S/(1+2^y) - S, then the fp16 hi/lo split
        const float y = fmaf(v[j], -0.37f, 0.11f);
        const float t = fmaf(rcpf(1.0f + ex2f(y)), 32768.f, -16384.f);
        __half2 hh = __floats2half2_rn(t, t * 0.5f);
        float2 f = __half22float2(hh);
        __half2 ll = __floats2half2_rn(t - f.x, 0.5f * t - f.y);
        acc += *reinterpret_cast<uint32_t*>(&hh) ^ *reinterpret_cast<uint32_t*>(&ll);
        v[j] = t * 1e-4f;
      }
    }
  }
  float s = 0; for (int j = 0; j < 16; ++j) s += v[j];
  if (s == 12345.f || acc == 77) out[0] = s + acc;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"ex2.approx", "rcp.approx", "f2fp pack (+fadd)", "ffma", "activation+split"};
  for (int op = 0; op < 5; ++op) {
    void (*kk)(float*, int) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
    int iters = 2000;
    kk<<<sms * 2, 512>>>(out, 10); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kk<<<sms * 2, 512>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 2 * 512 * iters * 16;
    double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-20s %.3e ops/s  = %.2f lanes/clk/SM (at the %d MHz base attribute)\n", names[op], ops / (ms * 1e-3), per_sm_clk, clk / 1000);
  }
  return 0;
}
