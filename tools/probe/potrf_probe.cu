// Latency of the Cholesky DAG's in-tile kernels (pf_chol.cu potrf64, trinv64) on one CTA, no
// co-resident work: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   -Ipaper_2203_11875_b200/csrc tools/probe/potrf_probe.cu -o tools/probe/potrf_probe.bin
#include "pf_chol.cu"
#include <cstdio>

namespace pf {
__global__ void probe(const double* A, long long* cyc, double* out) {
  extern __shared__ double sm[];
  __shared__ int sh[2];
  double* Cs = sm;
  double* Li = sm + TILE_D;
  double* sv = Li + TILE_D;
  double* tmp = sv + NB;
  if (threadIdx.x >= kCons) return;
  for (int rep = 0; rep < 3; ++rep) {
    for (int e = threadIdx.x; e < NB * NB; e += kCons) Cs[(e >> 6) * LDC + (e & 63)] = A[e];
    cons_sync();
    long long t0 = clock64();
    const int fail = potrf64(Cs, sv, sh);
    cons_sync();
    long long t1 = clock64();
    trinv64(Cs, sv, Li, tmp);
    cons_sync();
    long long t2 = clock64();
    if (threadIdx.x == 0) { cyc[2 * rep] = t1 - t0; cyc[2 * rep + 1] = t2 - t1; out[0] = fail; out[1] = Li[0]; }
  }
}
}  // namespace pf

int main() {
  double h[64 * 64];
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c < 64; ++c) h[r * 64 + c] = (r == c) ? 64.0 : 1.0 / (1 + r + c);
  double *dA, *dout;
  long long* dc;
  cudaMalloc(&dA, sizeof(h)); cudaMalloc(&dc, 64); cudaMalloc(&dout, 16);
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  const int smem = (2 * pf::TILE_D + pf::NB + 768) * 8;
  cudaFuncSetAttribute(pf::probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pf::probe<<<1, pf::kDagThreads, smem>>>(dA, dc, dout);
  long long c[6];
  double o[2];
  cudaMemcpy(c, dc, 48, cudaMemcpyDeviceToHost);
  cudaMemcpy(o, dout, 16, cudaMemcpyDeviceToHost);
  printf("potrf64 %lld cycles, trinv64 %lld cycles (rep 2), fail %g, err %s\n", c[4], c[5], o[0],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
