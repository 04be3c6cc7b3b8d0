// Diagnostic: exact parallel sequential-sum (csrc/exactsum.cuh) on one long
// lattice chain vs the plain sequential chain; prints how many segments fell
// back to sequential summation.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2001_08743_b200/csrc/exactsum.cuh"



__global__ void partial(const double* x, int n, double* approx) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  int lo = g * kt::xsum::kSeg;
  if (lo >= n) return;
  int hi = min(n, lo + kt::xsum::kSeg);
  double s = 0;
  for (int i = lo; i < hi; ++i) s = kt::dadd(s, x[i]);
  approx[g] = s;
}
__global__ void maps_k(const double* x, int n, const double* pre, kt::xsum::SegMap* maps) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  int lo = g * kt::xsum::kSeg;
  if (lo >= n) return;
  int len = min(n, lo + kt::xsum::kSeg) - lo;
  kt::xsum::SegMap m{0, 0, 0, 0};
  if (pre[g] > 0) m = kt::xsum::segment_map([&](int i) { return x[lo + i]; }, len, kt::xsum::binade_of(pre[g]));
  maps[g] = m;
}
__global__ void compose(const double* x, int n, const kt::xsum::SegMap* maps, double* out, int* nseq, int* nok) {
  double s = 0;
  int nsg = (n + kt::xsum::kSeg - 1) / kt::xsum::kSeg;
  for (int g = 0; g < nsg; ++g) {
    if (maps[g].ok) ++*nok;
    if (kt::xsum::apply_map(s, maps[g])) continue;
    ++*nseq;
    int lo = g * kt::xsum::kSeg, hi = min(n, lo + kt::xsum::kSeg);
    for (int i = lo; i < hi; ++i) s = kt::dadd(s, x[i]);
  }
  out[0] = s;
  double t = 0;
  for (int i = 0; i < n; ++i) t = kt::dadd(t, x[i]);
  out[1] = t;
}

int main() {
  const int n = 125000, card = 84;
  std::mt19937 r(1);
  std::vector<double> x(n);
  for (auto& v : x) v = (double)(r() % card) / (double)(card - 1);
  int nsg = (n + kt::xsum::kSeg - 1) / kt::xsum::kSeg;
  double *dx, *da, *dp, *dout;
  kt::xsum::SegMap* dm;
  int *dseq, *dok;
  cudaMalloc(&dx, n * 8);
  cudaMalloc(&da, nsg * 8);
  cudaMalloc(&dp, nsg * 8);
  cudaMalloc(&dm, nsg * sizeof(kt::xsum::SegMap));
  cudaMalloc(&dout, 16);
  cudaMalloc(&dseq, 4);
  cudaMalloc(&dok, 4);
  cudaMemset(dseq, 0, 4);
  cudaMemset(dok, 0, 4);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  partial<<<(nsg + 127) / 128, 128>>>(dx, n, da);
  std::vector<double> a(nsg), p(nsg);
  cudaMemcpy(a.data(), da, nsg * 8, cudaMemcpyDeviceToHost);
  double run = 0;
  for (int g = 0; g < nsg; ++g) { p[g] = run; run += a[g]; }
  cudaMemcpy(dp, p.data(), nsg * 8, cudaMemcpyHostToDevice);
  maps_k<<<(nsg + 127) / 128, 128>>>(dx, n, dp, dm);
  compose<<<1, 1>>>(dx, n, dm, dout, dseq, dok);
  double out[2];
  int nseq, nok;
  cudaMemcpy(out, dout, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(&nseq, dseq, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&nok, dok, 4, cudaMemcpyDeviceToHost);
  std::vector<kt::xsum::SegMap> m(nsg);
  cudaMemcpy(m.data(), dm, nsg * sizeof(kt::xsum::SegMap), cudaMemcpyDeviceToHost);
  printf("segments %d ok %d sequential %d exact %d (%.17g vs %.17g) err=%s\n", nsg, nok, nseq,
         out[0] == out[1], out[0], out[1], cudaGetErrorString(cudaGetLastError()));
  for (int g = 1; g < 6; ++g) printf("seg %d pre %.6g e %d ok %d F0 %llu F1 %llu\n", g, p[g], m[g].e, m[g].ok,
                                     (unsigned long long)m[g].F0, (unsigned long long)m[g].F1);
  return 0;
}
