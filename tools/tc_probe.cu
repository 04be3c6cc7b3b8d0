// Probe: D[128 x N] = A[128 x 32] . B[N x 32]^T with tcgen05 (kind::f16, fp32
// accumulate in TMEM), A/B K-major no-swizzle — checks csrc/tcgen05.cuh.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2001_08743_b200/csrc/tcgen05.cuh"

constexpr int M = 128, K = 32, N = 64;

__global__ void probe(const __half* A, const __half* B, float* D) {
  __shared__ __align__(128) __half sA[M * K];
  __shared__ __align__(128) __half sB[N * K];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  unsigned char* pa = reinterpret_cast<unsigned char*>(sA);
  unsigned char* pb = reinterpret_cast<unsigned char*>(sB);
  for (int i = t; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(pa + kt::tc::kmajor_offset(r, k, K)) = A[i];
  }
  for (int i = t; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(pb + kt::tc::kmajor_offset(r, k, K)) = B[i];
  }
  if (t < 32) kt::tc::tmem_alloc(&tbase, 64);
  if (t == 0) {
    kt::tc::mbar_init(&mbar, 1);
    kt::tc::fence_mbar_init();
  }
  kt::tc::fence_proxy_async();
  kt::tc::fence_before();
  __syncthreads();
  kt::tc::fence_after();
  const uint32_t tmem = tbase;
  if (t == 0) {
    const uint32_t idesc = kt::tc::idesc_f16_f32(M, N);
    for (int kb = 0; kb < K / 16; ++kb) {
      const uint64_t ad = kt::tc::smem_desc(kt::tc::smem_u32(pa + kb * 256), 128, (K / 8) * 128);
      const uint64_t bd = kt::tc::smem_desc(kt::tc::smem_u32(pb + kb * 256), 128, (K / 8) * 128);
      kt::tc::mma_f16(tmem, ad, bd, idesc, kb > 0);
    }
    kt::tc::commit(&mbar);
  }
  kt::tc::mbar_wait(&mbar, 0);
  kt::tc::fence_after();
  const int w = t >> 5;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    kt::tc::ld_32x32b_x16(tmem + ((uint32_t)(32 * w) << 16) + c0, r);
    kt::tc::ld_wait();
    for (int j = 0; j < 16; ++j) D[(32 * w + (t & 31)) * N + c0 + j] = __uint_as_float(r[j]);
  }
  kt::tc::fence_before();
  __syncthreads();
  if (t < 32) kt::tc::tmem_dealloc(tmem, 64);
}

int main() {
  std::mt19937 g(3);
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  for (int i = 0; i < M * K; ++i) { Af[i] = (float)(g() % 300); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = __half2float(__float2half((g() % 1000) / 997.0f)); B[i] = __float2half(Bf[i]); }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(__half) * M * K);
  cudaMalloc(&dB, sizeof(__half) * N * K);
  cudaMalloc(&dD, sizeof(float) * M * N);
  cudaMemcpy(dA, A.data(), sizeof(__half) * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), sizeof(__half) * N * K, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
  double maxrel = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)Af[m * K + k] * Bf[n * K + k];
      const double rel = std::fabs(D[m * N + n] - ref) / std::max(1.0, std::fabs(ref));
      maxrel = std::max(maxrel, rel);
      bad += rel > 1e-5;
    }
  std::printf("tcgen05 probe: %s, max rel err %.3g, bad %d / %d, D[0]=%g D[last]=%g\n", cudaGetErrorString(e),
              maxrel, bad, M * N, D[0], D[M * N - 1]);
  return bad ? 1 : 0;
}
