// FP64 peak microbenchmark for the Cholesky roofline denominator (DFMA vs DMMA m8n8k4).
// MEASURED_PEAKS.json carries no FP64 figure, so this is how DESIGN.md's FP64 peak is obtained.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 - a;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the sm_90+ f64 shapes: m16n8k4 (A 2, B 1, C 4 doubles per lane), m16n8k8 (A 4, B 2), m16n8k16 (A 8, B 4)
template <int K>
__global__ void dmma16_kernel(double* out, int iters) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-9 - i;
  double c[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if constexpr (K == 4)
          asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                       : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
        else if constexpr (K == 8)
          asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                       : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
        else
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                       : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                       : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                         "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K>
void run16(int blocks, int threads, int iters, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  dmma16_kernel<K><<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0); dmma16_kernel<K><<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * K * 4 * 16 * (double)iters * blocks * (threads / 32);
  printf("DMMA m16n8k%d: %.3f ms  %.2f TFLOP/s\n", K, ms, flops / ms / 1e9);
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = p.multiProcessorCount * 4, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("DFMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 8 * 4 * 8 * 16 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    run16<4>(blocks, threads, iters / 2, out, e0, e1);
    run16<8>(blocks, threads, iters / 4, out, e0, e1);
    run16<16>(blocks, threads, iters / 8, out, e0, e1);
  }
  cudaError_t err = cudaGetLastError(); printf("err %s\n", cudaGetErrorString(err));
  return 0;
}
