// Latency of the in-tile 64×64 Cholesky / trsm variants (one CTA, clock64).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NB = 64, LDC = 65, LDT = 68;

// V1: Crout by columns, thread r owns row r, 2 named barriers per column
__device__ void potrf_v1(double* Cs, double* sv) {
  const int r = threadIdx.x;
  double* Lr = Cs + r * LDC;
  for (int c = 0; c < NB; ++c) {
    double num = 0.0;
    if (r >= c) {
      const double* Lc = Cs + c * LDC;
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      int k = 0;
      for (; k + 3 < c; k += 4) { s0 += Lr[k] * Lc[k]; s1 += Lr[k + 1] * Lc[k + 1]; s2 += Lr[k + 2] * Lc[k + 2]; s3 += Lr[k + 3] * Lc[k + 3]; }
      for (; k < c; ++k) s0 += Lr[k] * Lc[k];
      num = Lr[c] - ((s0 + s1) + (s2 + s3));
      if (r == c) sv[c] = num;
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const double d = sv[c];
    const double ld = sqrt(d);
    if (r > c) Lr[c] = num / ld; else if (r == c) Lr[c] = ld;
    asm volatile("bar.sync 1, 64;" ::: "memory");
  }
}
// V2: as V1 with rsqrt + multiply
__device__ void potrf_v2(double* Cs, double* sv) {
  const int r = threadIdx.x;
  double* Lr = Cs + r * LDC;
  for (int c = 0; c < NB; ++c) {
    double num = 0.0;
    if (r >= c) {
      const double* Lc = Cs + c * LDC;
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      int k = 0;
      for (; k + 3 < c; k += 4) { s0 += Lr[k] * Lc[k]; s1 += Lr[k + 1] * Lc[k + 1]; s2 += Lr[k + 2] * Lc[k + 2]; s3 += Lr[k + 3] * Lc[k + 3]; }
      for (; k < c; ++k) s0 += Lr[k] * Lc[k];
      num = Lr[c] - ((s0 + s1) + (s2 + s3));
      if (r == c) sv[c] = num;
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const double d = sv[c];
    const double rs = rsqrt(d);
    if (r >= c) Lr[c] = num * rs;
    asm volatile("bar.sync 1, 64;" ::: "memory");
  }
}
// V3: right-looking, one warp, lane owns rows lane and lane+32 in SMEM; no block barriers
__device__ void potrf_v3(double* Cs, double*) {
  const int l = threadIdx.x;
  if (l >= 32) return;
  for (int c = 0; c < NB; ++c) {
    __syncwarp();
    const double rs = rsqrt(Cs[c * LDC + c]);
    double l0 = 0, l1 = 0;
    const int r0 = l, r1 = l + 32;
    if (r0 >= c) l0 = Cs[r0 * LDC + c] * rs;
    if (r1 >= c) l1 = Cs[r1 * LDC + c] * rs;
    __syncwarp();
    if (r0 >= c) Cs[r0 * LDC + c] = l0;
    if (r1 >= c) Cs[r1 * LDC + c] = l1;
    __syncwarp();
    // trailing update of columns c+1.. : A[r][k] -= L[r][c] L[k][c] for c < k <= r
    for (int k = c + 1; k < NB; ++k) {
      const double lk = Cs[k * LDC + c];
      if (r0 >= k) Cs[r0 * LDC + k] -= l0 * lk;
      if (r1 >= k) Cs[r1 * LDC + k] -= l1 * lk;
    }
  }
}
// trsm X L^T = C, thread per row, dot form
__device__ void trsm_v1(double* Cs, const double* Ls) {
  const int r = threadIdx.x;
  double* X = Cs + r * LDC;
  for (int c = 0; c < NB; ++c) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int k = 0;
    for (; k + 3 < c; k += 4) { s0 += X[k] * Ls[k * LDT + c]; s1 += X[k + 1] * Ls[(k + 1) * LDT + c]; s2 += X[k + 2] * Ls[(k + 2) * LDT + c]; s3 += X[k + 3] * Ls[(k + 3) * LDT + c]; }
    for (; k < c; ++k) s0 += X[k] * Ls[k * LDT + c];
    X[c] = (X[c] - ((s0 + s1) + (s2 + s3))) / Ls[c * LDT + c];
  }
}
// trsm with transposed L staged row-major (Lt[c][k] = L(c,k), stride LDC) and reciprocal diag
__device__ void trsm_v2(double* Cs, const double* Lt, const double* rd) {
  const int r = threadIdx.x;
  double* X = Cs + r * LDC;
  for (int c = 0; c < NB; ++c) {
    const double* Lc = Lt + c * LDC;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int k = 0;
    for (; k + 3 < c; k += 4) { s0 += X[k] * Lc[k]; s1 += X[k + 1] * Lc[k + 1]; s2 += X[k + 2] * Lc[k + 2]; s3 += X[k + 3] * Lc[k + 3]; }
    for (; k < c; ++k) s0 += X[k] * Lc[k];
    X[c] = (X[c] - ((s0 + s1) + (s2 + s3))) * rd[c];
  }
}

__global__ void bench(int variant, double* out, long long* cyc) {
  extern __shared__ double smx[];
  double *Cs = smx, *Ls = Cs + NB * LDC, *Lt = Ls + NB * LDT, *sv = Lt + NB * LDC, *rd = sv + NB;
  for (int i = threadIdx.x; i < NB * LDC; i += blockDim.x) { int r = i / LDC, c = i % LDC; Cs[i] = (r == c) ? 64.0 : 1.0 / (1 + r + c); Lt[i] = (r == c) ? 8.0 : (r > c ? 0.01 : 0); }
  for (int i = threadIdx.x; i < NB * LDT; i += blockDim.x) { int c = i / LDT, r = i % LDT; Ls[i] = (r == c) ? 8.0 : (r > c ? 0.01 : 0); }
  for (int i = threadIdx.x; i < NB; i += blockDim.x) rd[i] = 0.125;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 64) {
    if (variant == 1) potrf_v1(Cs, sv);
    else if (variant == 2) potrf_v2(Cs, sv);
    else if (variant == 3) potrf_v3(Cs, sv);
    else if (variant == 4) trsm_v1(Cs, Ls);
    else if (variant == 5) trsm_v2(Cs, Lt, rd);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  double s = 0;
  for (int i = threadIdx.x; i < NB * LDC; i += blockDim.x) s += Cs[i];
  out[threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  const char* names[] = {"", "potrf crout 2bar", "potrf crout rsqrt", "potrf right-looking 1 warp", "trsm dot (packed L)", "trsm dot (row-major L, rcp)"};
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  for (int v = 1; v <= 5; ++v) {
    for (int rep = 0; rep < 3; ++rep) bench<<<1, 256, 110000>>>(v, out, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-32s %8lld cycles  (%.2f us at 1.965 GHz)\n", names[v], c, c / 1965.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
