// pf_chol.cu — condensed-KKT factor + solve (A9 of SURVEY §8(a)):
// K_cond = sym(K̂) + diag(Σ_u) + δ_w I (Theorem 2 with R9, P:L784–787;
// δ_w regularisation P:L1341–1342), blocked FP64 Cholesky (the role of
// cusolver's potrf in P:L1339–1341; success certifies the inertia, Theorem 3
// P:L856–866) and the solve L Lᵀ p = b.
//
// Left-looking blocked algorithm, 64-column panels, per panel j:
//   k_chol_update  A[j:, j] −= L[j:, :j] L[j, :j]ᵀ  — the O(n³) part, a deep-K
//                  GEMM on the FP64 tensor pipe (mma.sync m8n8k4 f64 = SASS
//                  DMMA.8x8x4; tcgen05 has no kind::f64), operands streamed
//                  through a 2-stage cp.async SMEM pipeline; each panel tile
//                  is written once.
//   k_chol_panel   factor the 64×64 diagonal block in SMEM and solve the
//                  panel rows below it (X L_jjᵀ = A).
// k_chol_solve     forward/backward substitution, cooperative: the CTAs of a
//                  scenario own 64-row blocks, one grid barrier per block.
// Batched over scenarios; a scenario whose factorization failed (info ≠ 0)
// skips all later work.
#include "pf_launch.h"

#include <algorithm>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace pf {

namespace {

constexpr int NB = 64;        // panel width
constexpr int KC = 32;        // K chunk of the update GEMM
constexpr int LDT = NB + 4;   // SMEM stride of the [k][row] operand tiles (conflict-free fragments)
constexpr int kUpdSmem = 2 * 2 * KC * LDT * (int)sizeof(double);
constexpr int kPanelSmem = 2 * NB * (NB + 1) * (int)sizeof(double);

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

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N_>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_)); }

// A[I-tile, j-panel] −= L[I-tile, 0:j0] · L[j-panel, 0:j0]ᵀ for one 64×64 tile.
// 4 warps × 32×32 outputs; K streamed in 32-wide chunks, 2 SMEM stages.
__global__ void __launch_bounds__(128) k_chol_update(int n, int j0, double* __restrict__ K, const int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  extern __shared__ double sm_upd[];
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - j0);
  const int I0 = j0 + blockIdx.x * NB;
  auto As = [&](int st) { return sm_upd + st * 2 * KC * LDT; };
  auto Bs = [&](int st) { return sm_upd + st * 2 * KC * LDT + KC * LDT; };
  auto load = [&](int st, int k0) {
    double* a = As(st);
    double* b = Bs(st);
    for (int idx = threadIdx.x; idx < KC * NB; idx += blockDim.x) {
      const int k = idx / NB, r = idx % NB;
      const double* col = A + (size_t)(k0 + k) * n;
      if (I0 + r < n) cp_async8(a + k * LDT + r, col + I0 + r); else a[k * LDT + r] = 0.0;
      if (r < nb) cp_async8(b + k * LDT + r, col + j0 + r); else b[k * LDT + r] = 0.0;
    }
    cp_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }
  const int nchunk = j0 / KC;
  load(0, 0);
  for (int c = 0; c < nchunk; ++c) {
    if (c + 1 < nchunk) { load((c + 1) & 1, (c + 1) * KC); cp_wait<1>(); }
    else cp_wait<0>();
    __syncthreads();
    const double* a = As(c & 1);
    const double* b = Bs(c & 1);
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = a[(kk + q) * LDT + wr * 32 + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = b[(kk + q) * LDT + wc * 32 + nt * 8 + g];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = I0 + wr * 32 + mt * 8 + g;
        const int c = wc * 32 + nt * 8 + 2 * q + h;
        if (r < n && c < nb && r >= j0 + c) A[(size_t)(j0 + c) * n + r] -= acc[mt][nt][h];
      }
}

// Panel step: every CTA factors the 64×64 diagonal block in SMEM (CTA 0 writes
// L_jj back and reports the first failing column in info), then solves its
// 64-row block of the panel, X L_jjᵀ = A (4 lanes per row, shuffle-reduced).
__global__ void __launch_bounds__(256) k_chol_panel(int n, int k0, double* __restrict__ K, int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  extern __shared__ double smem_panel[];
  double (*L)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_panel);
  double (*X)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_panel + NB * (NB + 1));
  __shared__ int fail;
  __shared__ double inv_piv;
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - k0);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int c = idx / nb, r = idx % nb;
    L[r][c] = r >= c ? A[(size_t)(k0 + c) * n + k0 + r] : 0.0;
  }
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int jj = 0; jj < nb; ++jj) {
    if (threadIdx.x == 0) {
      const double d = L[jj][jj];
      if (!(d > 0.0) || !isfinite(d)) fail = k0 + jj + 1;
      else { const double sq = sqrt(d); L[jj][jj] = sq; inv_piv = 1.0 / sq; }
    }
    __syncthreads();
    if (fail) break;
    const double ip = inv_piv;
    for (int r = jj + 1 + threadIdx.x; r < nb; r += blockDim.x) L[r][jj] *= ip;
    __syncthreads();
    for (int r = jj + 1 + ty; r < nb; r += 16) {
      const double lr = L[r][jj];
      for (int c = jj + 1 + tx; c <= r; c += 16) L[r][c] -= lr * L[c][jj];
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

// L Lᵀ P = B for every right-hand side of every scenario.  The P CTAs of a
// scenario own 64-row blocks round-robin.  Forward: the owner of block J
// solves L_JJ y_J = b_J, grid barrier, then every CTA updates its own blocks
// I > J: b_I −= L_IJ y_J.  Backward (right-looking on Lᵀ): the owner of J
// solves L_JJᵀ p_J = b_J, barrier, every CTA updates its blocks I < J:
// b_I −= L_JIᵀ p_J.  One grid barrier per block and direction.
constexpr int kSolveThreads = 256;

__global__ void __launch_bounds__(kSolveThreads) k_chol_solve(int n, const double* __restrict__ K, double* __restrict__ rhs,
                                                              int nrhs, const int* __restrict__ info, int n_scen, int P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double D[NB][NB + 1];
  __shared__ double yb[NB];
  const int s = blockIdx.x / P, sub = blockIdx.x % P;
  const bool active = s < n_scen && info[s] == 0;
  const double* L = K + (size_t)(s < n_scen ? s : 0) * n * n;
  const int nblk = (n + NB - 1) / NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  auto stage = [&](int j0, int nb) {
    for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
      const int c = idx / nb, r = idx % nb;
      D[r][c] = r >= c ? L[(size_t)(j0 + c) * n + j0 + r] : 0.0;
    }
    __syncthreads();
  };
  for (int rr = 0; rr < nrhs; ++rr) {
    double* b = rhs + ((size_t)(s < n_scen ? s : 0) * nrhs + rr) * n;
    // ---- forward L y = b
    for (int J = 0; J < nblk; ++J) {
      const int j0 = J * NB, nb = min(NB, n - j0);
      if (active && sub == J % P) {
        stage(j0, nb);
        if (warp == 0) {
          for (int j = 0; j < nb; ++j) {
            const double yj = __ldcg(b + j0 + j) / D[j][j];
            __syncwarp();
            if (lane == 0) __stcg(b + j0 + j, yj);
            for (int i = j + 1 + lane; i < nb; i += 32) __stcg(b + j0 + i, __ldcg(b + j0 + i) - D[i][j] * yj);
            __syncwarp();
          }
        }
      }
      grid.sync();
      if (active) {
        for (int t = threadIdx.x; t < nb; t += blockDim.x) yb[t] = __ldcg(b + j0 + t);
        __syncthreads();
        for (int I = J + 1 + ((sub - (J + 1)) % P + P) % P; I < nblk; I += P) {
          const int i0 = I * NB, ni = min(NB, n - i0);
          for (int t = threadIdx.x; t < ni; t += blockDim.x) {
            const int i = i0 + t;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int j = 0;
            for (; j + 3 < nb; j += 4) {
              a0 += L[(size_t)(j0 + j) * n + i] * yb[j];
              a1 += L[(size_t)(j0 + j + 1) * n + i] * yb[j + 1];
              a2 += L[(size_t)(j0 + j + 2) * n + i] * yb[j + 2];
              a3 += L[(size_t)(j0 + j + 3) * n + i] * yb[j + 3];
            }
            for (; j < nb; ++j) a0 += L[(size_t)(j0 + j) * n + i] * yb[j];
            __stcg(b + i, __ldcg(b + i) - ((a0 + a1) + (a2 + a3)));
          }
        }
        __syncthreads();
      }
    }
    // ---- backward Lᵀ p = y
    for (int J = nblk - 1; J >= 0; --J) {
      const int j0 = J * NB, nb = min(NB, n - j0);
      if (active && sub == J % P) {
        stage(j0, nb);
        if (warp == 0) {
          for (int j = nb - 1; j >= 0; --j) {
            double acc = 0.0;
            for (int i = j + 1 + lane; i < nb; i += 32) acc += D[i][j] * __ldcg(b + j0 + i);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) __stcg(b + j0 + j, (__ldcg(b + j0 + j) - acc) / D[j][j]);
            __syncwarp();
          }
        }
      }
      grid.sync();
      if (active) {
        for (int t = threadIdx.x; t < nb; t += blockDim.x) yb[t] = __ldcg(b + j0 + t);
        __syncthreads();
        for (int I = sub; I < J; I += P) {
          const int i0 = I * NB, ni = min(NB, n - i0);
          for (int t = warp; t < ni; t += nwarp) {  // column i of L, rows j0.. (contiguous)
            const int i = i0 + t;
            double acc = 0.0;
            for (int j = lane; j < nb; j += 32) acc += L[(size_t)i * n + j0 + j] * yb[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) __stcg(b + i, __ldcg(b + i) - acc);
          }
        }
        __syncthreads();
      }
    }
    grid.sync();
  }
}

__global__ void k_info_out(int n_scen, const int* __restrict__ ws, int* __restrict__ out) {
  for (int s = threadIdx.x; s < n_scen; s += blockDim.x) out[s] = ws[s];
}

}  // namespace

int launch_chol(const DevNet& net, int n_scen, double* K, const double* sigma_u, double delta_w,
                double* rhs, int nrhs, int* info, int* info_ws, cudaStream_t st) {
  const int n = net.n_u;
  int launches = 0;
  static int solve_cap = 0;
  if (!solve_cap) {
    cudaFuncSetAttribute(k_chol_update, cudaFuncAttributeMaxDynamicSharedMemorySize, kUpdSmem);
    cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem);
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_solve, kSolveThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    solve_cap = std::max(1, per_sm) * sms;
  }
  const long long tot = (long long)n_scen * n * n;
  const int blocks = (int)std::min<long long>((tot + 255) / 256, 148LL * 32);
  k_chol_init<<<blocks, 256, 0, st>>>(n, n_scen, K, sigma_u, delta_w, info_ws);
  ++launches;
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int rows = n - j0;
    const int T = (rows + NB - 1) / NB;
    if (j0 > 0) {
      k_chol_update<<<dim3(T, n_scen), 128, kUpdSmem, st>>>(n, j0, K, info_ws);
      ++launches;
    }
    const int nb = std::min(NB, rows);
    const int Tb = (rows - nb + NB - 1) / NB;
    k_chol_panel<<<dim3(std::max(Tb, 1), n_scen), 256, kPanelSmem, st>>>(n, j0, K, info_ws);
    ++launches;
  }
  if (nrhs > 0) {
    const int nblk = (n + NB - 1) / NB;
    int P = std::max(1, std::min(solve_cap / n_scen, nblk));
    void* args[] = {(void*)&n, (void*)&K, (void*)&rhs, (void*)&nrhs, (void*)&info_ws, (void*)&n_scen, (void*)&P};
    cudaLaunchCooperativeKernel((void*)k_chol_solve, dim3(P * n_scen), dim3(kSolveThreads), args, 0, st);
    ++launches;
  }
  if (info) { k_info_out<<<1, 256, 0, st>>>(n_scen, info_ws, info); ++launches; }
  return launches;
}

}  // namespace pf
