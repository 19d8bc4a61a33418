// Standalone timing + task trace of the condensed-KKT Cholesky (pf_chol.cu)
// on S random SPD matrices of order n:  chol_bench [n] [S] [reps] [trace.csv]
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DPF_CHOL_TRACE \
//        -Ipaper_2203_11875_b200/csrc tools/chol_bench.cu -o /tmp/chol_bench
#include "pf_chol.cu"

#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2889, S = argc > 2 ? atoi(argv[2]) : 8;
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  const char* trace = argc > 4 ? argv[4] : nullptr;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> K((size_t)S * n * n), b((size_t)S * n, 1.0);
  for (int s = 0; s < S; ++s)
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r) K[((size_t)s * n + c) * n + r] = (r == c) ? n : U(rng);
  pf::DevNet net{};
  net.n_u = n;
  pf::Work w{};
  double *dK, *dK0, *drhs;
  int *dinfo, *dws;
  cudaMalloc(&dK, K.size() * 8); cudaMalloc(&dK0, K.size() * 8); cudaMalloc(&drhs, b.size() * 8);
  cudaMalloc(&dinfo, S * 4); cudaMalloc(&dws, S * 4);
  cudaMalloc(&w.ctile, S * pf::chol_tile_doubles(n) * 8);
  cudaMalloc(&w.cflag, S * pf::chol_flag_ints(n) * 4);
  cudaMalloc(&w.cticket, 4 * (1 + 1024));
  cudaMalloc(&w.cy, S * pf::chol_vec_doubles(n) * 8);
  cudaMemcpy(dK0, K.data(), K.size() * 8, cudaMemcpyHostToDevice);
  const int ntask_max = S * (int)(pf::chol_flag_ints(n));
  unsigned long long* dtr = nullptr;
  cudaMalloc(&dtr, (size_t)ntask_max * 8 * 8);
  cudaMemset(dtr, 0, (size_t)ntask_max * 8 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int gmax = pf::chol_grid_max();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpy(dK, dK0, K.size() * 8, cudaMemcpyDeviceToDevice);
    cudaMemcpy(drhs, b.data(), b.size() * 8, cudaMemcpyHostToDevice);
#ifdef PF_CHOL_TRACE
    if (r == reps - 1 && trace) cudaMemcpyToSymbol(pf::g_chol_trace, &dtr, sizeof(dtr));
#endif
    cudaEventRecord(e0);
    pf::launch_chol(net, w, S, dK, nullptr, 0.0, drhs, 1, dinfo, dws, 0, gmax);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (!(r == reps - 1 && trace)) best = std::min(best, ms);
    printf("rep %d: %.3f ms\n", r, ms);
  }
  // correctness: L Lᵀ = sym(K) on sampled entries, and the solve residual, for scenarios 0 and S-1
  {
    std::vector<double> L((size_t)n * n), p(n);
    double worst = 0.0, resid = 0.0;
    for (int s : {0, S - 1}) {
      cudaMemcpy(L.data(), dK + (size_t)s * n * n, (size_t)n * n * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(p.data(), drhs + (size_t)s * n, (size_t)n * 8, cudaMemcpyDeviceToHost);
      auto Kc = [&](int r, int c) { const double* A = &K[(size_t)s * n * n]; return 0.5 * (A[(size_t)c * n + r] + A[(size_t)r * n + c]); };
      std::mt19937 g(3);
      for (int t = 0; t < 2000; ++t) {
        int r = g() % n, c = g() % n;
        if (c > r) std::swap(r, c);
        if (t < 64) { r = n - 1 - t % 7; c = t % 64 < r ? r - t % 64 : r; }
        double acc = 0.0;
        for (int k = 0; k <= c; ++k) acc += L[(size_t)k * n + r] * L[(size_t)k * n + c];
        worst = std::max(worst, std::fabs(acc - Kc(r, c)) / n);
      }
      for (int r = 0; r < n; ++r) {
        double acc = 0.0;
        for (int c = 0; c < n; ++c) acc += Kc(r, c) * p[c];
        resid = std::max(resid, std::fabs(acc - 1.0));
      }
    }
    printf("check: max |LLt - K|/max|K| = %.3e, max |K p - b| = %.3e\n", worst, resid);
  }
  std::vector<int> info(S);
  cudaMemcpy(info.data(), dinfo, S * 4, cudaMemcpyDeviceToHost);
  printf("n=%d S=%d best %.3f ms  (%.2f TFLOP/s on n^3/3)  info[0]=%d err=%s\n", n, S, best,
         S * (double)n * n * n / 3.0 / (best * 1e-3) / 1e12, info[0], cudaGetErrorString(cudaGetLastError()));
  if (trace) {
    std::vector<unsigned long long> tr((size_t)ntask_max * 8);
    cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
    FILE* f = fopen(trace, "w");
    fprintf(f, "ticket,kind,s,i,j,sm,t0,t1,m0,m1,m2,m3\n");
    for (int t = 0; t < ntask_max; ++t) {
      const unsigned long long* e = &tr[8 * (size_t)t];
      if (!e[2]) continue;
      fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", t, e[0] >> 56, (e[0] >> 40) & 0xffff,
              (e[0] >> 20) & 0xfffff, e[0] & 0xfffff, e[1], e[2], e[3], e[4], e[5], e[6], e[7]);
    }
    fclose(f);
  }
  return 0;
}
