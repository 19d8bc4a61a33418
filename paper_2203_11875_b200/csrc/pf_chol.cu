// pf_chol.cu — condensed-KKT factor + solve (A9 of SURVEY §8(a)):
// K_cond = sym(K̂) + diag(Σ_u) + δ_w I (Theorem 2 with R9, P:L784–787;
// δ_w regularisation P:L1341–1342), blocked right-looking FP64 Cholesky
// (the role of cusolver's potrf in P:L1339–1341) and L Lᵀ p = b.
//
// B200: there is no tcgen05 kind::f64 (ptxas rejects it), so the
// O(n³) trailing update runs on the FP64 tensor pipe through warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), operands staged in SMEM; the panel
// and the triangular solves are DFMA.  Batched over scenarios (grid.y).
#include "pf_launch.h"

#include <algorithm>

namespace pf {

namespace {

constexpr int NB = 64;       // panel width
constexpr int LDS = NB + 4;  // padded SMEM row stride (conflict-free 8-byte fragment loads)
constexpr int kSyrkSmem = 2 * NB * LDS * (int)sizeof(double);
constexpr int kTrsmSmem = 2 * NB * (NB + 1) * (int)sizeof(double);

__global__ void k_chol_init(int n, int n_scen, double* __restrict__ K, const double* __restrict__ sig_u,
                            double delta, int* __restrict__ info_ws) {
  const long long total = (long long)n_scen * n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / ((long long)n * n));
    const long long rem = t % ((long long)n * n);
    const int jc = (int)(rem / n), i = (int)(rem % n);  // column-major (row i, column jc)
    double* A = K + (size_t)s * n * n;
    if (i > jc) {
      const double a = 0.5 * (A[(size_t)jc * n + i] + A[(size_t)i * n + jc]);
      A[(size_t)jc * n + i] = a;
      A[(size_t)i * n + jc] = 0.0;
    } else if (i == jc) {
      A[(size_t)jc * n + i] += (sig_u ? sig_u[(size_t)s * n + i] : 0.0) + delta;
    }
    if (rem == 0) info_ws[s] = 0;
  }
}

// Panel step of the right-looking factorization, one launch per 64-column
// panel: every CTA factors the 64×64 diagonal block in SMEM (unblocked, 256
// threads; CTA 0 writes L_kk back and reports the first failing column in
// info), then solves its 64-row block of the panel, X L_kkᵀ = A (4 lanes per
// row, shuffle-reduced dot products).
__global__ void __launch_bounds__(256) k_chol_panel(int n, int k0, double* __restrict__ K, int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  extern __shared__ double smem_panel[];
  double (*L)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_panel);
  double (*X)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_panel + NB * (NB + 1));
  __shared__ int fail;
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - k0);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int c = idx / nb, r = idx % nb;
    L[r][c] = r >= c ? A[(size_t)(k0 + c) * n + k0 + r] : 0.0;
  }
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  for (int jj = 0; jj < nb; ++jj) {
    if (threadIdx.x == 0) {
      const double d = L[jj][jj];
      if (!(d > 0.0) || !isfinite(d)) fail = k0 + jj + 1;
      else L[jj][jj] = sqrt(d);
    }
    __syncthreads();
    if (fail) break;
    const double piv = L[jj][jj];
    for (int r = jj + 1 + threadIdx.x; r < nb; r += blockDim.x) L[r][jj] /= piv;
    __syncthreads();
    const int m = nb - jj - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int r = jj + 1 + idx / m, c = jj + 1 + idx % m;
      if (c <= r) L[r][c] -= L[r][jj] * L[c][jj];
    }
    __syncthreads();
  }
  if (fail) {
    if (blockIdx.x == 0 && threadIdx.x == 0) info[s] = fail;
    return;
  }
  if (blockIdx.x == 0)
    for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
      const int c = idx / nb, r = idx % nb;
      if (r >= c) A[(size_t)(k0 + c) * n + k0 + r] = L[r][c];
    }
  const int i0 = k0 + nb + blockIdx.x * NB;
  if (i0 >= n) return;
  for (int idx = threadIdx.x; idx < nb * NB; idx += blockDim.x) {
    const int c = idx / NB, r = idx % NB;
    X[r][c] = (i0 + r < n) ? A[(size_t)(k0 + c) * n + i0 + r] : 0.0;
  }
  __syncthreads();
  const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
  for (int c = 0; c < nb; ++c) {
    double part = 0.0;
    for (int mm = q; mm < c; mm += 4) part += X[r][mm] * L[c][mm];
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (q == 0) X[r][c] = (X[r][c] - part) / L[c][c];
    __syncwarp();
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nb * NB; idx += blockDim.x) {
    const int c = idx / NB, rr = idx % NB;
    if (i0 + rr < n) A[(size_t)(k0 + c) * n + i0 + rr] = X[rr][c];
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Trailing update A[I,J] −= A[I,k] A[J,k]ᵀ for lower tiles I ≥ J (SYRK/GEMM)
// on the FP64 tensor pipe: 4 warps × (32×32) per 64×64 tile, m8n8k4 fragments
// from SMEM (row stride LDS keeps each 8-byte half-warp phase bank-conflict free).
__global__ void __launch_bounds__(128) k_chol_syrk(int n, int k0, double* __restrict__ K, const int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  extern __shared__ double smem_syrk[];
  double* As = smem_syrk;
  double* Bs = smem_syrk + NB * LDS;
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - k0);
  const int t0 = k0 + nb;
  const int tt = blockIdx.x;
  int I = (int)((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= tt) ++I;
  while (I * (I + 1) / 2 > tt) --I;
  const int J = tt - I * (I + 1) / 2;
  const int I0 = t0 + I * NB, J0 = t0 + J * NB;
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x) {
    const int kk = idx / NB, r = idx % NB;
    const bool kin = kk < nb;
    As[r * LDS + kk] = (kin && I0 + r < n) ? A[(size_t)(k0 + kk) * n + I0 + r] : 0.0;
    Bs[r * LDS + kk] = (kin && J0 + r < n) ? A[(size_t)(k0 + kk) * n + J0 + r] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }
#pragma unroll 4
  for (int kk = 0; kk < NB; kk += 4) {
    double af[4], bf[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[mt] = As[(wr * 32 + mt * 8 + g) * LDS + kk + q];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[(wc * 32 + nt * 8 + g) * LDS + kk + q];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = I0 + wr * 32 + mt * 8 + g;
        const int c = J0 + wc * 32 + nt * 8 + 2 * q + h;
        if (r < n && c < n && (I != J || r >= c)) A[(size_t)c * n + r] -= acc[mt][nt][h];
      }
}

// L Lᵀ p = b for one (scenario, right-hand side): blocked forward / backward
// substitution; b and each 64×64 diagonal block staged in SMEM, the
// off-diagonal updates as coalesced column sweeps over L.
__global__ void __launch_bounds__(256) k_chol_solve(int n, const double* __restrict__ K, double* __restrict__ rhs,
                                                    int nrhs, const int* __restrict__ info) {
  extern __shared__ double sm_solve[];
  double (*D)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(sm_solve);
  double* b = sm_solve + NB * (NB + 1);
  const int s = blockIdx.y, rr = blockIdx.x;
  if (info[s] != 0) return;
  const double* L = K + (size_t)s * n * n;
  double* bg = rhs + ((size_t)s * nrhs + rr) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = bg[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  auto stage = [&](int j0, int nb) {
    for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
      const int c = idx / nb, r = idx % nb;
      D[r][c] = r >= c ? L[(size_t)(j0 + c) * n + j0 + r] : 0.0;
    }
  };
  __syncthreads();
  // forward: L y = b
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int j1 = min(n, j0 + NB), nb = j1 - j0;
    stage(j0, nb);
    __syncthreads();
    if (warp == 0) {
      for (int j = 0; j < nb; ++j) {
        const double yj = b[j0 + j] / D[j][j];
        __syncwarp();
        if (lane == 0) b[j0 + j] = yj;
        for (int i = j + 1 + lane; i < nb; i += 32) b[j0 + i] -= D[i][j] * yj;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = j1 + threadIdx.x; i < n; i += blockDim.x) {
      double acc = b[i];
      for (int j = j0; j < j1; ++j) acc -= L[(size_t)j * n + i] * b[j];
      b[i] = acc;
    }
    __syncthreads();
  }
  // backward: Lᵀ p = y
  const int nblk = (n + NB - 1) / NB;
  for (int bk = nblk - 1; bk >= 0; --bk) {
    const int j0 = bk * NB, j1 = min(n, j0 + NB), nb = j1 - j0;
    for (int j = j0 + warp; j < j1; j += nwarp) {
      double acc = 0.0;
      for (int i = j1 + lane; i < n; i += 32) acc += L[(size_t)j * n + i] * b[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) b[j] -= acc;
    }
    stage(j0, nb);
    __syncthreads();
    if (warp == 0) {
      for (int j = nb - 1; j >= 0; --j) {
        double acc = 0.0;
        for (int i = j + 1 + lane; i < nb; i += 32) acc += D[i][j] * b[j0 + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) b[j0 + j] = (b[j0 + j] - acc) / D[j][j];
        __syncwarp();
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) bg[i] = b[i];
}

__global__ void k_info_out(int n_scen, const int* __restrict__ ws, int* __restrict__ out) {
  for (int s = threadIdx.x; s < n_scen; s += blockDim.x) out[s] = ws[s];
}

}  // namespace

int launch_chol(const DevNet& net, int n_scen, double* K, const double* sigma_u, double delta_w,
                double* rhs, int nrhs, int* info, int* info_ws, cudaStream_t st) {
  const int n = net.n_u;
  int launches = 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_chol_syrk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem);
    cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem);
    attr = true;
  }
  long long tot = (long long)n_scen * n * n;
  int blocks = (int)std::min<long long>((tot + 255) / 256, 148LL * 32);
  k_chol_init<<<blocks, 256, 0, st>>>(n, n_scen, K, sigma_u, delta_w, info_ws);
  ++launches;
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int nb = std::min(NB, n - k0);
    const int rest = n - k0 - nb;
    const int T = (rest + NB - 1) / NB;
    k_chol_panel<<<dim3(std::max(T, 1), n_scen), 256, kTrsmSmem, st>>>(n, k0, K, info_ws);
    ++launches;
    if (rest > 0) {
      k_chol_syrk<<<dim3(T * (T + 1) / 2, n_scen), 128, kSyrkSmem, st>>>(n, k0, K, info_ws);
      ++launches;
    }
  }
  if (nrhs > 0) {
    const size_t smem = (size_t)(n + NB * (NB + 1)) * sizeof(double);
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_chol_solve<<<dim3(nrhs, n_scen), 256, smem, st>>>(n, K, rhs, nrhs, info_ws);
    ++launches;
  }
  if (info) { k_info_out<<<1, 256, 0, st>>>(n_scen, info_ws, info); ++launches; }
  return launches;
}

}  // namespace pf
