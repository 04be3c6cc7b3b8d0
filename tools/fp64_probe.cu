// Debug: dependent-chain latency (cycles/op) of fp64 ops on one warp, B200.
#include <cstdio>
#include "../paper_2001_08743_b200/csrc/device.cuh"
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = __fma_rn(x, b, a);
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) x = __dadd_rn(x, b);
  long long t2 = clock64();
  for (int i = 0; i < 200; ++i) x = __ddiv_rn(a, x + 1.5);
  long long t3 = clock64();
  for (int i = 0; i < 200; ++i) x = kt::kt_tanh_bf(x + 0.3);
  long long t4 = clock64();
  for (int i = 0; i < 1000; ++i) x = __fmaf_rn((float)x, (float)b, (float)a);
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(o, c, 0.5, 0.999); cudaDeviceSynchronize(); }
  printf("DFMA %.1f  DADD %.1f  ddiv %.1f  tanh_bf %.1f  FFMA(+cvt) %.1f cycles/op\n", c[0] / 1000.0, c[1] / 1000.0,
         c[2] / 200.0, c[3] / 200.0, c[4] / 1000.0);
}
