// Cycles of the DAG kernel's in-tile potrf64 / trsm64 (pf_chol.cu) on one CTA, plus
// the FP64 dependent-latency basics they are built from.
#include "pf_chol.cu"
#include <cstdio>
using namespace pf;
__global__ void bench(int variant, double* out, long long* cyc) {
  extern __shared__ double smx[];
  double *Cs = smx, *Ls = Cs + NB * LDC, *rd = Ls + TILE_D;
  __shared__ int sh[2];
  for (int i = threadIdx.x; i < NB * LDC; i += blockDim.x) { int r = i / LDC, c = i % LDC; Cs[i] = (r == c) ? 64.0 : 1.0 / (1 + r + c); }
  for (int i = threadIdx.x; i < TILE_D; i += blockDim.x) { int c = i / LDT, r = i % LDT; Ls[i] = (r == c) ? 8.0 : (r > c ? 0.01 : 0); }
  for (int i = threadIdx.x; i < NB; i += blockDim.x) rd[i] = 0.125;
  __syncthreads();
  long long t0 = clock64();
  double acc = threadIdx.x;
  if (variant == 1) potrf64(Cs, rd, sh);
  else if (variant == 2) trsm64(Cs, Ls, rd);
  else if (variant == 3) { for (int i = 0; i < 1000; ++i) acc = fma(acc, 0.999, 1e-3); }
  else if (variant == 4) { for (int i = 0; i < 1000; ++i) acc = rsqrt(acc + 1.0); }
  else if (variant == 5) { for (int i = 0; i < 1000; ++i) acc = __shfl_sync(0xffffffffu, acc, 3) + 1.0; }
  else if (variant == 6) { for (int i = 0; i < 1000; ++i) { cons_sync(); } }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = Cs[threadIdx.x] + acc;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  const char* names[] = {"", "potrf64", "trsm64", "1000 dependent DFMA", "1000 dependent rsqrt(double)", "1000 shfl+DADD", "1000 bar.sync 256"};
  for (int v = 1; v <= 6; ++v) {
    for (int rep = 0; rep < 3; ++rep) bench<<<1, 256, 110000>>>(v, out, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-30s %8lld cycles  (%.2f us at 1.965 GHz)\n", names[v], c, c / 1965.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
