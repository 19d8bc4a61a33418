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
//                  through a 3-stage cp.async SMEM pipeline.  K is split so
//                  that ~2 CTAs per SM work on every panel; the last CTA of a
//                  tile (arrival counter) sums the split-K partials in fixed
//                  order — deterministic — and writes the updated panel tile.
//   k_chol_panel   factor the 64×64 diagonal block (register-blocked, one
//                  barrier per column) and solve the panel rows below it.
// k_chol_solve     forward/backward substitution on one thread-block cluster per
//                  scenario: its CTAs own 64-row blocks, one cluster barrier per block.
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
constexpr int NST = 3;       // cp.async pipeline stages of the update GEMM
constexpr int kUpdSmem = NST * 2 * KC * LDT * (int)sizeof(double);
constexpr int TS = 32;        // symmetrize tile

// sym + shift: lower ← (A + Aᵀ)/2 (+ Σ_u + δ_w on the diagonal), upper ← 0,
// through 32×32 SMEM tiles so both the tile and its mirror are read coalesced.
__global__ void __launch_bounds__(256) k_chol_sym(int n, double* __restrict__ K, const double* __restrict__ sig_u,
                                                  double delta, int* __restrict__ info_ws) {
  __shared__ double a[TS][TS + 1], b[TS][TS + 1];
  const int s = blockIdx.y;
  const int nt = (n + TS - 1) / TS;
  int I = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);  // lower tile (I ≥ J)
  while ((I + 1) * (I + 2) / 2 <= (int)blockIdx.x) ++I;
  while (I * (I + 1) / 2 > (int)blockIdx.x) --I;
  const int J = blockIdx.x - I * (I + 1) / 2;
  if (I >= nt) return;
  double* A = K + (size_t)s * n * n;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 × 8
  for (int c = ty; c < TS; c += 8) {
    const int col = J * TS + c, row = I * TS + tx;           // tile (I, J): A[col][row] column-major
    a[c][tx] = (row < n && col < n) ? A[(size_t)col * n + row] : 0.0;
    const int col2 = I * TS + c, row2 = J * TS + tx;         // mirror tile (J, I)
    b[c][tx] = (row2 < n && col2 < n) ? A[(size_t)col2 * n + row2] : 0.0;
  }
  __syncthreads();
  for (int c = ty; c < TS; c += 8) {
    const int col = J * TS + c, row = I * TS + tx;
    if (row < n && col < n) {
      // element (row, col) of the lower triangle; its mirror (col, row) is b[tx][c]
      double v;
      if (row > col) v = 0.5 * (a[c][tx] + b[tx][c]);
      else if (row == col) v = a[c][tx] + (sig_u ? sig_u[(size_t)s * n + row] : 0.0) + delta;
      else v = 0.0;  // strict upper part of a diagonal tile
      A[(size_t)col * n + row] = v;
    }
    if (I != J) {
      const int col2 = I * TS + c, row2 = J * TS + tx;
      if (row2 < n && col2 < n) A[(size_t)col2 * n + row2] = 0.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) info_ws[s] = 0;
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

// Split-K Gram products of the left-looking update for the 64×64 tiles t of
// panel j (tile 0 = the diagonal block):
//   P[ks][t] = Σ_{k ∈ chunk range ks} L[j0 + 64t : +64, k] · L[j0 : j0+64, k]ᵀ.
// 4 warps × 32×32 outputs, K streamed in 32-wide chunks through 3 cp.async
// SMEM stages.  KS = 1: the CTA writes A − P itself; otherwise each CTA stores
// its partial and the last to arrive sums them in ks order (deterministic).
__global__ void __launch_bounds__(128) k_chol_update(int n, int j0, int T, int KS, double* __restrict__ K,
                                                     double* __restrict__ part, int slots, int* __restrict__ count,
                                                     int cnt_stride, const int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  extern __shared__ double sm_upd[];
  __shared__ int last;
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - j0);
  const int tile = blockIdx.x % T, ks = blockIdx.x / T;
  const int I0 = j0 + tile * NB;
  const int nchunk = j0 / KC, per = (nchunk + KS - 1) / KS;
  const int c0 = ks * per, c1 = min(nchunk, c0 + per);
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
  if (c0 < c1) load(0, c0 * KC);
  if (c0 + 1 < c1) load(1, (c0 + 1) * KC);
  for (int c = c0; c < c1; ++c) {
    if (c + 2 < c1) { load((c + 2 - c0) % NST, (c + 2) * KC); cp_wait<2>(); }
    else if (c + 1 < c1) cp_wait<1>();
    else cp_wait<0>();
    __syncthreads();
    const double* a = As((c - c0) % NST);
    const double* b = Bs((c - c0) % NST);
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
  auto store_final = [&](int r, int c, double sub) {  // tile-local (r, c)
    const int gr = I0 + r;
    if (gr < n && c < nb && gr >= j0 + c) {
      double* p = A + (size_t)(j0 + c) * n + gr;
      *p = *p - sub;
    }
  };
  if (KS == 1) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          store_final(wr * 32 + mt * 8 + g, wc * 32 + nt * 8 + 2 * q + h, acc[mt][nt][h]);
    return;
  }
  double* P = part + ((size_t)s * slots + (size_t)ks * T + tile) * (NB * NB);
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wr * 32 + mt * 8 + g, c = wc * 32 + nt * 8 + 2 * q + h;
        __stcg(P + c * NB + r, acc[mt][nt][h]);
      }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* cnt = count + (size_t)s * cnt_stride + tile;
    last = atomicAdd(cnt, 1) == KS - 1;
    if (last) *cnt = 0;  // ready for the next panel / call
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double* P0 = part + ((size_t)s * slots + tile) * (NB * NB);
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x) {
    const int c = idx / NB, r = idx % NB;
    double sum = 0.0;
    for (int k = 0; k < KS; ++k) sum += __ldcg(P0 + (size_t)k * T * (NB * NB) + idx);
    store_final(r, c, sum);
  }
}

// Panel step.  Every CTA factors the 64×64 diagonal block, then solves its
// 64-row block of the panel, X L_jjᵀ = A.  Both are register-blocked: thread
// (ty, tx) of the 16×16 thread grid owns the 16 elements (ty + 16a, tx + 16b);
// each of the 64 sequential steps publishes one column through SMEM (double-
// buffered, ONE barrier per step) and every thread updates its elements.
// The factorization runs in the unscaled LDLᵀ form (A[r][c] −= A[r][J] A[c][J]
// / d_J needs no broadcast pivot), the Cholesky scaling L = D^{1/2} applied at
// the end; CTA 0 writes L_jj back and reports the first pivot ≤ 0 in info.
__global__ void __launch_bounds__(256) k_chol_panel(int n, int k0, double* __restrict__ K, int* __restrict__ info) {
  const int s = blockIdx.y;
  if (info[s] != 0) return;
  __shared__ double col[2][NB];
  __shared__ double dv[NB];
  __shared__ double Ls[NB][NB + 1];
  __shared__ int fail;
  double* A = K + (size_t)s * n * n;
  const int nb = min(NB, n - k0);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double a[4][4];  // element (ty + 16i, tx + 16j)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      double v;
      if (r < nb && c < nb) v = r >= c ? A[(size_t)(k0 + c) * n + k0 + r] : 0.0;
      else v = (r == c) ? 1.0 : 0.0;  // identity padding past the matrix edge
      a[i][j] = v;
    }
  if (threadIdx.x == 0) fail = 0;
  // ---- factor: 64 steps, one barrier each
  for (int J = 0; J < NB; ++J) {
    const int bj = J >> 4, tj = J & 15, buf = J & 1;
    if (tx == tj) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j == bj) col[buf][ty + 16 * i] = a[i][j];  // static indexing keeps a[][] in registers
    }
    __syncthreads();
    const double d = col[buf][J];
    if (!(d > 0.0) || !isfinite(d)) {  // every thread sees the same pivot
      if (threadIdx.x == 0) fail = k0 + J + 1;
      break;
    }
    if (threadIdx.x == 0) dv[J] = d;
    const double invd = 1.0 / d;
    double cr[4], cc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { cr[i] = col[buf][ty + 16 * i]; cc[i] = col[buf][tx + 16 * i] * invd; }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = ty + 16 * i, c = tx + 16 * j;
        if (c > J && r >= c) a[i][j] -= cr[i] * cc[j];
      }
  }
  __syncthreads();
  if (fail) {
    if (blockIdx.x == 0 && threadIdx.x == 0) info[s] = fail;
    return;
  }
  // ---- L = (unscaled column) / sqrt(d_c), diagonal sqrt(d_c)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      const double sq = sqrt(dv[c]);
      const double v = r == c ? sq : (r > c ? a[i][j] / sq : 0.0);
      Ls[r][c] = v;
      if (blockIdx.x == 0 && r < nb && c < nb && r >= c) A[(size_t)(k0 + c) * n + k0 + r] = v;
    }
  const int i0 = k0 + nb + blockIdx.x * NB;
  if (i0 >= n) return;
  // ---- panel rows: X L_jjᵀ = A, column by column (right-looking), one barrier per column
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      a[i][j] = (i0 + r < n && c < nb) ? A[(size_t)(k0 + c) * n + i0 + r] : 0.0;
    }
  __syncthreads();
  for (int J = 0; J < nb; ++J) {
    const int bj = J >> 4, tj = J & 15, buf = J & 1;
    const double inv = 1.0 / Ls[J][J];
    if (tx == tj) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j == bj) { a[i][j] *= inv; col[buf][ty + 16 * i] = a[i][j]; }
    }
    __syncthreads();
    double xr[4], lc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { xr[i] = col[buf][ty + 16 * i]; lc[i] = Ls[tx + 16 * i][J]; }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (tx + 16 * j > J) a[i][j] -= xr[i] * lc[j];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      if (i0 + r < n && c < nb) A[(size_t)(k0 + c) * n + i0 + r] = a[i][j];
    }
}

// L Lᵀ P = B for every right-hand side of every scenario.  The P CTAs of a
// scenario's thread-block cluster own 64-row blocks round-robin.  Forward: the owner of block J
// solves L_JJ y_J = b_J, grid barrier, then every CTA updates its own blocks
// I > J: b_I −= L_IJ y_J.  Backward (right-looking on Lᵀ): the owner of J
// solves L_JJᵀ p_J = b_J, barrier, every CTA updates its blocks I < J:
// b_I −= L_JIᵀ p_J.  One cluster barrier per block and direction.
constexpr int kSolveThreads = 256;

__global__ void __launch_bounds__(kSolveThreads) k_chol_solve(int n, const double* __restrict__ K, double* __restrict__ rhs,
                                                              int nrhs, const int* __restrict__ info, int n_scen, int P) {
  cg::cluster_group grid = cg::this_cluster();  // one cluster of P CTAs per scenario
  __shared__ double D[NB][NB + 1];
  __shared__ double yb[NB];
  const int s = blockIdx.x / P, sub = (int)grid.block_rank();
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
        for (int t = threadIdx.x; t < nb; t += blockDim.x) yb[t] = __ldcg(b + j0 + t);
        stage(j0, nb);
        if (warp == 0) {
          for (int j = 0; j < nb; ++j) {
            const double yj = yb[j] / D[j][j];
            __syncwarp();
            if (lane == 0) yb[j] = yj;
            for (int i = j + 1 + lane; i < nb; i += 32) yb[i] -= D[i][j] * yj;
            __syncwarp();
          }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nb; t += blockDim.x) __stcg(b + j0 + t, yb[t]);
      }
      grid.sync();
      if (active) {
        for (int t = threadIdx.x; t < nb; t += blockDim.x) yb[t] = __ldcg(b + j0 + t);
        __syncthreads();
        // rows of the owned blocks I > J, 4 lanes per row (16 columns each)
        const int q = threadIdx.x & 3;
        for (int I = J + 1 + ((sub - (J + 1)) % P + P) % P; I < nblk; I += P) {
          const int i0 = I * NB, ni = min(NB, n - i0);
          // warp-uniform trip count: the shuffles below need all 32 lanes
          for (int t0 = 0; t0 < ni; t0 += blockDim.x >> 2) {
            const int t = t0 + (threadIdx.x >> 2);
            const int i = i0 + t;
            double a0 = 0.0, a1 = 0.0;
            if (t < ni)
              for (int j = q; j < nb; j += 8) {
                a0 += L[(size_t)(j0 + j) * n + i] * yb[j];
                if (j + 4 < nb) a1 += L[(size_t)(j0 + j + 4) * n + i] * yb[j + 4];
              }
            double a = a0 + a1;
            a += __shfl_xor_sync(0xffffffffu, a, 1);
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            if (q == 0 && t < ni) __stcg(b + i, __ldcg(b + i) - a);
          }
        }
        __syncthreads();
      }
    }
    // ---- backward Lᵀ p = y
    for (int J = nblk - 1; J >= 0; --J) {
      const int j0 = J * NB, nb = min(NB, n - j0);
      if (active && sub == J % P) {
        for (int t = threadIdx.x; t < nb; t += blockDim.x) yb[t] = __ldcg(b + j0 + t);
        stage(j0, nb);
        if (warp == 0) {
          for (int j = nb - 1; j >= 0; --j) {
            double acc = 0.0;
            for (int i = j + 1 + lane; i < nb; i += 32) acc += D[i][j] * yb[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) yb[j] = (yb[j] - acc) / D[j][j];
            __syncwarp();
          }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nb; t += blockDim.x) __stcg(b + j0 + t, yb[t]);
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

int chol_part_slots(int n_u) { return (n_u + NB - 1) / NB + 296; }

int launch_chol(const DevNet& net, const Work& w, int n_scen, double* K, const double* sigma_u, double delta_w,
                double* rhs, int nrhs, int* info, int* info_ws, cudaStream_t st) {
  const int n = net.n_u;
  int launches = 0;
  static int CSS = 0;
  if (!CSS) {
    cudaFuncSetAttribute(k_chol_update, cudaFuncAttributeMaxDynamicSharedMemorySize, kUpdSmem);
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {16, 8, 4, 2, 1}) {  // largest cluster the part schedules
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cs); cfg.blockDim = dim3(kSolveThreads); cfg.attrs = at; cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, (void*)k_chol_solve, &cfg) == cudaSuccess && nc > 0) { CSS = cs; break; }
    }
    cudaGetLastError();
    if (!CSS) CSS = 1;
  }
  const int nts = (n + TS - 1) / TS;
  k_chol_sym<<<dim3(nts * (nts + 1) / 2, n_scen), 256, 0, st>>>(n, K, sigma_u, delta_w, info_ws);
  ++launches;
  const int cnt_stride = (n + NB - 1) / NB + 1;
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int rows = n - j0;
    const int T = (rows + NB - 1) / NB;   // tiles of the panel, tile 0 = diagonal block
    if (j0 > 0) {  // split K so that ~2 CTAs per SM work on every panel
      const int nchunk = j0 / KC;
      int KS = std::max(1, std::min({(296 + T * n_scen - 1) / (T * n_scen), nchunk, 16}));
      KS = std::min(KS, std::max(1, w.cpart_slots / T));
      k_chol_update<<<dim3(T * KS, n_scen), 128, kUpdSmem, st>>>(n, j0, T, KS, K, w.cpart, w.cpart_slots,
                                                                   w.ccount, cnt_stride, info_ws);
      ++launches;
    }
    k_chol_panel<<<dim3(std::max(T - 1, 1), n_scen), 256, 0, st>>>(n, j0, K, info_ws);
    ++launches;
  }
  if (nrhs > 0) {
    const int P = CSS;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(P * n_scen); cfg.blockDim = dim3(kSolveThreads); cfg.stream = st;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_chol_solve, n, (const double*)K, rhs, nrhs, (const int*)info_ws, n_scen, P);
    ++launches;
  }
  if (info) { k_info_out<<<1, 256, 0, st>>>(n_scen, info_ws, info); ++launches; }
  return launches;
}

}  // namespace pf
