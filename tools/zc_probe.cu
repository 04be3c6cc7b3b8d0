// Debug: SM-issued writes into pinned (mapped) host memory: GB/s vs CTA count and row width.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void copy_rows(const uint8_t* __restrict__ src, uint8_t* dst, int rows, int w, int spitch, int dpitch) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nw) {
    const uint64_t* s = reinterpret_cast<const uint64_t*>(src + (size_t)r * spitch);
    uint64_t* d = reinterpret_cast<uint64_t*>(dst + (size_t)r * dpitch);
    for (int i = lane; i < w / 8; i += 32) d[i] = s[i];
  }
}
int main() {
  const int rows = 49152 * 5;
  const size_t dbytes = (size_t)rows * 1024, hbytes = (size_t)rows * 4096;
  uint8_t *src, *dst;
  cudaMalloc(&src, dbytes);
  cudaHostAlloc(&dst, hbytes, cudaHostAllocDefault);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w : {200, 400, 800}) for (int ctas : {4, 8, 16, 32, 148, 296}) {
    copy_rows<<<ctas, 512>>>(src, dst, rows, w, 1024, 4000);
    cudaEventRecord(a);
    for (int k = 0; k < 3; ++k) copy_rows<<<ctas, 512>>>(src, dst, rows, w, 1024, 4000);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("w %4d ctas %3d: %.1f GB/s\n", w, ctas, 3.0 * rows * w / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
