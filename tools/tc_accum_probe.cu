// Characterisation probe for the rollout certificate:
//  (1) `accum <in> <out>`: chains of tcgen05.mma.kind::f16 (M=128, N=16, K=16,
//      fp32 accumulate in TMEM); the accumulator is read back after EVERY
//      instruction, so tools/tc_accum_analyze.py can compare each instruction's
//      result d against the exact value c + sum_k a_k b_k of its inputs.
//  (2) `mufu`: exhaustive error of ex2.approx.ftz.f32, rcp.approx.ftz.f32,
//      lg2.approx.ftz.f32 and of the rollout's fast tanh over every fp32 input.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2001_08743_b200/csrc/tcgen05.cuh"

constexpr int M = 128, N = 16, K = 16;

__global__ void accum_kernel(const __half* A, const __half* B, float* D, int nmma) {
  __shared__ __align__(128) __half sA[M * K];
  __shared__ __align__(128) __half sB[N * K];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, b = blockIdx.x;
  unsigned char* pa = reinterpret_cast<unsigned char*>(sA);
  unsigned char* pb = reinterpret_cast<unsigned char*>(sB);
  if (t < 32) kt::tc::tmem_alloc(&tbase, 32);
  if (t == 0) {
    kt::tc::mbar_init(&mbar, 1);
    kt::tc::fence_mbar_init();
  }
  kt::tc::fence_before();
  __syncthreads();
  kt::tc::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = kt::tc::idesc_f16_f32(M, N);
  for (int j = 0; j < nmma; ++j) {
    const __half* a = A + ((size_t)b * nmma + j) * M * K;
    const __half* bb = B + ((size_t)b * nmma + j) * N * K;
    for (int i = t; i < M * K; i += blockDim.x)
      *reinterpret_cast<__half*>(pa + kt::tc::kmajor_offset(i / K, i % K, K)) = a[i];
    for (int i = t; i < N * K; i += blockDim.x)
      *reinterpret_cast<__half*>(pb + kt::tc::kmajor_offset(i / K, i % K, K)) = bb[i];
    kt::tc::fence_proxy_async();
    kt::tc::fence_before();
    __syncthreads();
    kt::tc::fence_after();
    if (t == 0) {
      const uint64_t ad = kt::tc::smem_desc(kt::tc::smem_u32(pa), 128, (K / 8) * 128);
      const uint64_t bd = kt::tc::smem_desc(kt::tc::smem_u32(pb), 128, (K / 8) * 128);
      kt::tc::mma_f16(tmem, ad, bd, idesc, j > 0);
      kt::tc::commit(&mbar);
    }
    kt::tc::mbar_wait(&mbar, j & 1);
    kt::tc::fence_after();
    uint32_t r[16];
    kt::tc::ld_32x32b_x16(tmem + ((uint32_t)(32 * (t >> 5)) << 16), r);
    kt::tc::ld_wait();
    float* d = D + ((size_t)b * nmma + j) * M * N + t * N;
    for (int c = 0; c < N; ++c) d[c] = __uint_as_float(r[c]);
    kt::tc::fence_before();
    __syncthreads();
    kt::tc::fence_after();
  }
  if (t < 32) kt::tc::tmem_dealloc(tmem, 32);
}

// ------------------------------------------------------------------ MUFU
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

__device__ void amax(unsigned long long* p, double v) {
  if (v > 0) atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// out[0]: ex2 max rel err (result normal); out[1]: rcp max rel err (normal in/out);
// out[2]: lg2 max abs err on [0.5, 2); out[3]: lg2 max rel err elsewhere (normal x);
// out[4]: fast tanh (S = 1) max abs err vs tanh(y / K2L) for every fp32 y;
// out[5]: fast tanh with S = 2^14, max abs err / S.
// out[6]: ex2 max rel err for y in [-1, 0] (the softmax's range is y <= 0)
__global__ void mufu_kernel(unsigned long long* out) {
  const double k2l = -2.0 / 0.69314718055994530942;  // -2 log2(e), exact to fp64
  const float k2lf = -2.8853900817779268f;
  (void)k2lf;
  double m[7] = {0, 0, 0, 0, 0, 0, 0};
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < (1ull << 32);
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)i);
    if (!isfinite(x)) continue;
    // ex2
    if (x >= -126.f && x < 128.f) {
      const double ref = exp2((double)x);
      const double e = fabs((double)ex2f(x) - ref) / ref;
      m[0] = fmax(m[0], e);
      if (x >= -1.f && x <= 0.f) m[6] = fmax(m[6], e);
    }
    // rcp
    if (x > 0.f && fabsf(x) >= 0x1.0p-125f && fabsf(x) < 0x1.0p126f) {
      const double ref = 1.0 / (double)x;
      m[1] = fmax(m[1], fabs((double)rcpf(x) - ref) / ref);
    }
    // lg2
    if (x >= 0x1.0p-126f) {
      const double ref = log2((double)x);
      const double e = fabs((double)lg2f(x) - ref);
      if (x >= 0.5f && x < 2.f) m[2] = fmax(m[2], e);
      else m[3] = fmax(m[3], e / fabs(ref));
    }
    // fast tanh: S tanh(y / K2L) ~= 2S/(1+2^y) - S
    {
      const double ref = tanh((double)x / k2l);
      const float r = rcpf(1.0f + ex2f(x));
      const float a1 = fmaf(r, 2.f, -1.f);
      m[4] = fmax(m[4], fabs((double)a1 - ref));
      const float a2 = fmaf(r, 32768.f, -16384.f);
      m[5] = fmax(m[5], fabs((double)a2 / 16384.0 - ref));
    }
  }
  for (int k = 0; k < 7; ++k) amax(out + k, m[k]);
}

static int run_accum(const char* in, const char* outp) {
  FILE* f = std::fopen(in, "rb");
  if (!f) return 2;
  int hdr[2];
  if (std::fread(hdr, 4, 2, f) != 2) return 2;
  const int nb = hdr[0], nm = hdr[1];
  std::vector<__half> A((size_t)nb * nm * M * K), B((size_t)nb * nm * N * K);
  // file layout per (batch, mma): A then B
  for (size_t i = 0; i < (size_t)nb * nm; ++i) {
    if (std::fread(A.data() + i * M * K, 2, M * K, f) != (size_t)M * K) return 2;
    if (std::fread(B.data() + i * N * K, 2, N * K, f) != (size_t)N * K) return 2;
  }
  std::fclose(f);
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, (size_t)nb * nm * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  accum_kernel<<<nb, 128>>>(dA, dB, dD, nm);
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("accum: %d batches x %d mma: %s\n", nb, nm, cudaGetErrorString(e));
  std::vector<float> D((size_t)nb * nm * M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  FILE* g = std::fopen(outp, "wb");
  std::fwrite(D.data(), 4, D.size(), g);
  std::fclose(g);
  return e == cudaSuccess ? 0 : 1;
}

static int run_mufu() {
  unsigned long long* d;
  cudaMalloc(&d, 7 * 8);
  cudaMemset(d, 0, 7 * 8);
  mufu_kernel<<<148 * 8, 256>>>(d);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[7];
  cudaMemcpy(h, d, 7 * 8, cudaMemcpyDeviceToHost);
  const char* names[7] = {"ex2.approx.ftz rel (normal results)", "rcp.approx.ftz rel (normal)",
                          "lg2.approx.ftz abs on [0.5,2)", "lg2.approx.ftz rel elsewhere",
                          "fast tanh S=1 abs", "fast tanh S=2^14 abs/S", "ex2.approx.ftz rel on [-1,0]"};
  std::printf("mufu exhaustive (%s):\n", cudaGetErrorString(e));
  for (int k = 0; k < 7; ++k) {
    double v;
    std::memcpy(&v, &h[k], 8);
    std::printf("  %-40s %.6e = 2^%.3f\n", names[k], v, v > 0 ? std::log2(v) : -999.0);
  }
  return e == cudaSuccess ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc >= 4 && !std::strcmp(argv[1], "accum")) return run_accum(argv[2], argv[3]);
  if (argc >= 2 && !std::strcmp(argv[1], "mufu")) return run_mufu();
  std::fprintf(stderr, "usage: tc_accum_probe accum <in> <out> | mufu\n");
  return 2;
}
