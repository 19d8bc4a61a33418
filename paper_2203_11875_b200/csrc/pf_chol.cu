// pf_chol.cu — condensed-KKT factor + solve (A9 of SURVEY §8(a)):
// K_cond = sym(K̂) + diag(Σ_u) + δ_w I (Theorem 2 with R9, P:L784–787;
// δ_w regularisation P:L1341–1342), FP64 Cholesky K_cond = L Lᵀ (the role of
// cusolver's potrf in P:L1339–1341; success certifies the inertia, Theorem 3
// P:L856–866) and the solve L Lᵀ p = b.
//
// Tile algorithm on 64×64 tiles, run as ONE persistent, dependency-driven
// kernel (k_chol_dag) over every scenario at once:
//   k_chol_reset   clear the ready flags, info, ticket (the K_cond entries are not
//                  packed ahead: each tile task reads its tile of sym(K̂) + Σ_u + δ_w I
//                  straight from K̂ into its DMMA accumulators, identity past n).
//   k_chol_dag     CTAs take tasks from a ticket counter in a topological order
//                  (column by column, all scenarios interleaved) and wait on
//                  per-tile ready flags (release/acquire):
//     tile (i, j)  C = A_ij − Σ_{k<j} L_ik L_jkᵀ  (left-looking; DMMA m8n8k4 f64 —
//                  tcgen05 has no kind::f64 — operands streamed by cp.async.bulk
//                  through a 3-stage mbarrier ring), then
//                  i = j: L_jj = chol(C) (blocked, info) and L_jj⁻¹ (block triangular
//                         inversion), stored beside the tiles;
//                  i > j: L_ij = C L_jj⁻ᵀ as one more DMMA tile product (L_jj⁻¹ streamed
//                         in as the task's last ring chunk).
//     fwd j        y_j = L_jj⁻¹(b_j − Σ_{k<j} L_jk y_k)   (runs during the factorization)
//     bwd j        p_j = L_jj⁻ᵀ(y_j − Σ_{i>j} L_ijᵀ p_i)   (GEMVs with the stored inverse)
//   k_chol_unpack  L back into K (column-major, strict upper zeroed).
// The critical path is ~3 short tile steps per block column, instead of one
// launch-separated panel per column; every tile's arithmetic order is fixed,
// so the result is deterministic and independent of the schedule.
#include "pf_launch.h"

#include <algorithm>
#include <cstdint>

namespace pf {

namespace {

constexpr int NB = 64;                    // tile size
constexpr int LDT = 68;                   // leading dimension inside a packed tile
constexpr int TILE_D = NB * LDT;          // doubles per packed tile (34816 B)
constexpr int HALF_D = 32 * LDT;          // 32 tile columns (one pipeline chunk, 17408 B)
constexpr int NST = 3;                    // bulk-copy ring stages
constexpr int kDagSmem = NST * 2 * HALF_D * (int)sizeof(double);  // 104448 B → 2 CTAs / SM
constexpr int LDC = NB + 1;               // SMEM row stride of the C / work tile

enum { T_DONE = 0, T_TILE = 1, T_FWD = 2, T_BWD = 3 };

constexpr int kRhsCap = 2;               // right-hand sides per DAG run (cy workspace)

struct DagArgs {
  int n, nt, ntri, S, nrhs, ntask;
  int factor;      // 1: tile tasks included; 0: solve-only run over an existing factor
  int rhs_ld;      // right-hand sides per scenario in rhs (this run handles [rhs0, rhs0 + nrhs))
  double* tiles;   // [S][ntri][TILE_D]
  int* flags;      // [S][ntri + 2 nt]   tile / fwd / bwd ready flags
  int* ticket;     // task counter
  int* info;       // [S]
  double* cy;      // [S][2][kRhsCap][nt*64]  y (forward) and p (backward), padded
  double* rhs;     // [S][rhs_ld][n], already offset to the first vector of this run
  int* crit;       // [kMaxSm] per-SM count of critical-path tasks in their triangular phase
  const int* sidx; // [S] caller scenario of each (virtual) scenario s, or null = identity (rhs indexing)
  // K_cond's entries are read straight from the caller's K̂ by each tile task (sym + shift + identity
  // padding, k_cond_entry): K [caller scenarios][n][n] column-major, Σ_u [caller scenarios][n], δ_w or
  // per-scenario dvec (regularization retries)
  const double* K;
  const double* sig_u;
  double delta;
  const double* dvec;
};
constexpr int kMaxSm = 1024;
#ifndef PF_CHOL_LOOK
#define PF_CHOL_LOOK 2
#endif
constexpr int kLook = PF_CHOL_LOOK;  // look-ahead band of the task order (k_chol_dag)

__host__ __device__ __forceinline__ int tidx(int nt, int i, int j) { return j * nt - j * (j - 1) / 2 + (i - j); }
// tiles per scenario: the ntri packed lower tiles of K_cond / L, then the nt inverses L_jj⁻¹
__host__ __device__ __forceinline__ size_t tstride(int nt) { return (size_t)nt * (nt + 1) / 2 + nt; }

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Poll relaxed, then acquire once: an acquire load compiles to LDG.STRONG + CCTL.IVALL (the
// whole L1 invalidated), so acquiring on every poll cost ~4% of the DAG's stall samples.
__device__ __forceinline__ void wait_flag(const int* p) {
  while (ld_relaxed(p) == 0) __nanosleep(40);
  (void)ld_acquire(p);
}
__device__ __forceinline__ int smid() {
  int v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
#ifndef PF_CHOL_SPIN_NS
#define PF_CHOL_SPIN_NS 64
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned done = 0;
  for (;;) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(saddr(b)), "r"(parity) : "memory");
    if (done) break;
    if (PF_CHOL_SPIN_NS) __nanosleep(PF_CHOL_SPIN_NS);  // let the co-resident CTA's warps issue
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// info[s] = min over failures (first failing column), 0 = none yet
__device__ __forceinline__ void record_fail(int* info, int code) {
  int old = *(volatile int*)info;
  while (old == 0 || code < old) {
    const int prev = atomicCAS(info, old, code);
    if (prev == old) break;
    old = prev;
  }
}

// K_cond(R, C) for R ≥ C of (virtual) scenario s: sym(K̂) + diag(Σ_u) + δ_w I (Theorem 2 with
// R9), the identity past n.  K̂ stays untouched, so a failed scenario can be retried.
__device__ __forceinline__ double k_cond_entry(const DagArgs& a, int s, int R, int C) {
  const int n = a.n;
  if (R >= n || C >= n) return R == C ? 1.0 : 0.0;  // identity padding
  const int sr = a.sidx ? a.sidx[s] : s;
  const double* A = a.K + (size_t)sr * n * n;
  if (R > C) return 0.5 * (__ldg(A + (size_t)C * n + R) + __ldg(A + (size_t)R * n + C));
  if (R == C) return __ldg(A + (size_t)C * n + R) + (a.sig_u ? __ldg(a.sig_u + (size_t)sr * n + R) : 0.0) +
                     (a.dvec ? __ldg(a.dvec + s) : a.delta);
  return 0.0;
}

// per run: clear every scenario's tile / fwd / bwd flags, its info, the ticket and the per-SM counters
__global__ void __launch_bounds__(256) k_chol_reset(int nt, int S, int* __restrict__ flags, int* __restrict__ ticket,
                                                    int* __restrict__ info, int* __restrict__ crit) {
  const int nflag = nt * (nt + 1) / 2 + 2 * nt;
  const long long total = (long long)S * nflag;
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < total; f += (long long)gridDim.x * blockDim.x)
    flags[f] = 0;
  if (blockIdx.x == 0) {
    for (int k = threadIdx.x; k < S; k += blockDim.x) info[k] = 0;
    for (int k = threadIdx.x; k < kMaxSm; k += blockDim.x) crit[k] = 0;
    if (threadIdx.x == 0) *ticket = 0;
  }
}

// L back into K: lower (incl. diagonal) from the tiles, strict upper zeroed — only for the
// scenarios that factorized (a failed one keeps its K̂, so a caller can retry with a larger δ_w).
__global__ void __launch_bounds__(256) k_chol_unpack(int n, int nt, const double* __restrict__ tiles,
                                                     double* __restrict__ K, const int* __restrict__ info,
                                                     const int* __restrict__ sidx) {
  const int s = blockIdx.z, I = blockIdx.x, J = blockIdx.y;
  if (info[s] != 0) return;
  double* A = K + (size_t)(sidx ? sidx[s] : s) * n * n;
  const double* T = I >= J ? tiles + ((size_t)s * tstride(nt) + tidx(nt, I, J)) * TILE_D : nullptr;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  for (int c = ty; c < NB; c += 4) {
    const int R = I * NB + tx, C = J * NB + c;
    if (R < n && C < n) A[(size_t)C * n + R] = (R >= C && T) ? T[c * LDT + tx] : 0.0;
  }
}

// solve-only run: clear the fwd / bwd flags and the ticket
__global__ void k_chol_reset_solve(int nt, int S, int* __restrict__ flags, int* __restrict__ ticket) {
  const int ntri = nt * (nt + 1) / 2, nflag = ntri + 2 * nt;
  for (int x = threadIdx.x; x < S * 2 * nt; x += blockDim.x) flags[(size_t)(x / (2 * nt)) * nflag + ntri + x % (2 * nt)] = 0;
  if (threadIdx.x == 0) *ticket = 0;
}

#ifdef PF_CHOL_TRACE
// tools/chol_bench.cu: per-task {kind | s | i | j, smid, t0, t1, phase marks[4]} (globaltimer ns)
__device__ unsigned long long* g_chol_trace;
__shared__ unsigned long long g_marks[4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PF_MARK(k) do { if (threadIdx.x == 0) g_marks[k] = gtimer(); } while (0)
#else
#define PF_MARK(k) do {} while (0)
#endif

// ------------------------------------------------------------------ the DAG kernel
// 8 consumer warps (DMMA, triangular kernels, GEMVs) + 1 producer warp that
// waits on the dependency flags and streams operand tiles into a 3-stage
// SMEM ring with cp.async.bulk (full / empty mbarriers), so flag latency
// never stalls the math.  Both sides walk the same chunk sequence per task.
constexpr int kCons = 256;                 // consumer threads
constexpr int kDagThreads = kCons + 32;    // + producer warp

struct Pipe {
  uint64_t* full;   // [NST]  producer arrive.expect_tx → bytes landed
  uint64_t* empty;  // [NST]  8 consumer-warp arrivals → slot free
  uint64_t* lbar;   // L_jj tile load
  unsigned cc;      // chunks of the ring used so far by this CTA
  unsigned lpar;    // parity of lbar
};

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 2, 256;" ::: "memory"); }
__device__ __forceinline__ double* stage_ptr(double* sm, unsigned st) { return sm + st * 2 * HALF_D; }

// consumer side: wait for chunk cc, hand the slot back after use
__device__ __forceinline__ const double* cons_acquire(Pipe& p, double* sm) {
  const unsigned st = p.cc % NST;
  mbar_wait(p.full + st, (p.cc / NST) & 1);
  return stage_ptr(sm, st);
}
__device__ __forceinline__ void cons_release(Pipe& p) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(p.empty + p.cc % NST);
  ++p.cc;
}
// producer side (one lane): wait for the slot, then copy `bytes` (1 or 2 pieces)
__device__ __forceinline__ void prod_issue(Pipe& p, double* sm, const double* src0, const double* src1,
                                           unsigned bytes_each) {
  const unsigned st = p.cc % NST;
  mbar_wait(p.empty + st, ((p.cc / NST) & 1) ^ 1);
  double* dst = stage_ptr(sm, st);
  fence_proxy_global();
  mbar_expect(p.full + st, src1 ? 2 * bytes_each : bytes_each);
  bulk_g2s(dst, src0, bytes_each, p.full + st);
  if (src1) bulk_g2s(dst + HALF_D, src1, bytes_each, p.full + st);
  ++p.cc;
}

struct TaskCtx {
  const DagArgs* a;
  int s, i, j;
  double* T;  // tiles of scenario s
  int* F;     // flags of scenario s
  __device__ const double* tile(int r, int c) const { return T + (size_t)tidx(a->nt, r, c) * TILE_D; }
  __device__ const double* linv(int c) const { return T + (size_t)(a->ntri + c) * TILE_D; }  // L_cc⁻¹
  __device__ int* tflag(int r, int c) const { return F + tidx(a->nt, r, c); }
  __device__ int* fwdflag(int k) const { return F + a->ntri + k; }
  __device__ int* bwdflag(int k) const { return F + a->ntri + a->nt + k; }
};

// ---- producer: the operand stream of each task kind
// L_jj (or, inv, L_jj⁻¹) into `dst` (epilogue area) once every ring chunk of the task is consumed
__device__ void prod_ljj(const TaskCtx& t, Pipe& p, double* dst, bool inv = false) {
  for (unsigned c = p.cc >= NST ? p.cc - NST : 0; c < p.cc; ++c) mbar_wait(p.empty + c % NST, (c / NST) & 1);
  wait_flag(t.tflag(t.j, t.j));
  fence_proxy_global();
  mbar_expect(p.lbar, TILE_D * sizeof(double));
  bulk_g2s(dst, inv ? t.linv(t.j) : t.tile(t.j, t.j), TILE_D * sizeof(double), p.lbar);
}

__device__ void produce(const TaskCtx& t, int kind, Pipe& p, double* sm) {
  const unsigned half = HALF_D * sizeof(double), full = TILE_D * sizeof(double);
  if (kind == T_TILE) {
    const bool diag = t.i == t.j;
    // the diagonal tile and the first one below it carry the column chain: while one
    // of them runs its triangular kernel on this SM, the other CTA's (non-critical)
    // GEMM stream pauses, so the latency-bound chain does not share the SM's pipes
    const bool critical = t.i <= t.j + 1;
    int* crit = t.a->crit + smid();
    // A critical tile also holds the counter while it streams chunks whose inputs
    // are ready — never while it waits for a dependency, which the throttled
    // neighbour may be computing (so the throttle cannot deadlock).
    bool held = false;
    auto hold = [&](bool on) {
      if (on != held) { atomicAdd(crit, on ? 1 : -1); held = on; }
    };
    for (int k = 0; k < t.j; ++k) {
      if (!critical)
        while (ld_relaxed(crit) > 0) __nanosleep(200);
      if (critical && (ld_relaxed(t.tflag(t.i, k)) == 0 || (!diag && ld_relaxed(t.tflag(t.j, k)) == 0)))
        hold(false);
      wait_flag(t.tflag(t.i, k));
      if (!diag) wait_flag(t.tflag(t.j, k));
      if (critical) hold(true);
      for (int h = 0; h < 2; ++h)
        prod_issue(p, sm, t.tile(t.i, k) + h * HALF_D, diag ? nullptr : t.tile(t.j, k) + h * HALF_D, half);
    }
    hold(false);
    if (!diag) {  // L_jj⁻¹ as the task's last ring chunk (one full slot), in flight during the last GEMM chunks
      wait_flag(t.tflag(t.j, t.j));
      prod_issue(p, sm, t.linv(t.j), t.linv(t.j) + HALF_D, half);
    }
  } else if (kind == T_FWD) {
    for (int k = 0; k < t.j; ++k) {
      wait_flag(t.tflag(t.j, k));
      prod_issue(p, sm, t.tile(t.j, k), nullptr, full);
    }
    prod_ljj(t, p, sm, true);
  } else if (kind == T_BWD) {
    for (int i = t.a->nt - 1; i > t.j; --i) {
      wait_flag(t.tflag(i, t.j));
      prod_issue(p, sm, t.tile(i, t.j), nullptr, full);
    }
    prod_ljj(t, p, sm, true);
  }
}

// ---- in-tile triangular kernels (256 consumer threads, 16-column blocks).
// Each 16-step dependency chain runs in registers (compile-time indices); the
// trailing block updates are spread over all consumer threads.
constexpr int SB = 16;

// Cs (row-major, stride LDC) lower part ← its Cholesky factor; rdv[c] = 1 / L(c, c).
// Returns 0, or c + 1 for the first column whose pivot is ≤ 0 or non-finite.
__device__ int potrf64(double* Cs, double* rdv, int* sh) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) sh[0] = 0;
  for (int b0 = 0; b0 < NB; b0 += SB) {
    if (tid < 32) {  // diagonal block: lane r < 16 owns row b0 + r (Crout, columns in order)
      const int r = lane & (SB - 1);
      double* row = Cs + (b0 + r) * LDC + b0;
      double x[SB];
#pragma unroll
      for (int k = 0; k < SB; ++k) x[k] = lane < SB ? row[k] : 0.0;  // lanes ≥ 16 only join the shuffles
      int bad = 0;
#pragma unroll
      for (int c = 0; c < SB; ++c) {
        const double* Lc = Cs + (b0 + c) * LDC + b0;
        double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < c; ++k) q4[k & 3] += x[k] * Lc[k];
        const double num = x[c] - ((q4[0] + q4[1]) + (q4[2] + q4[3]));
        const double d = __shfl_sync(0xffffffffu, num, c);
        if (!(d > 0.0) || !isfinite(d)) { bad = b0 + c + 1; break; }
        const double rs = rsqrt(d);
        x[c] = r == c ? d * rs : num * rs;
        if (lane < SB && r >= c) row[c] = x[c];
        if (lane == c) rdv[b0 + c] = rs;
        __syncwarp();
      }
      if (tid == 0 && bad) sh[0] = bad;
    }
    cons_sync();
    if (sh[0]) return sh[0];
    const int nb = NB - b0 - SB;  // rows / columns below the block
    if (nb == 0) break;
    if (tid < nb) {  // panel rows: X L_bbᵀ = A, one row per thread in registers
      double* row = Cs + (b0 + SB + tid) * LDC + b0;
      double x[SB];
#pragma unroll
      for (int k = 0; k < SB; ++k) x[k] = row[k];
#pragma unroll
      for (int c = 0; c < SB; ++c) {
        const double* Lc = Cs + (b0 + c) * LDC + b0;
        double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < c; ++k) q4[k & 3] += x[k] * Lc[k];
        x[c] = (x[c] - ((q4[0] + q4[1]) + (q4[2] + q4[3]))) * rdv[b0 + c];
      }
#pragma unroll
      for (int k = 0; k < SB; ++k) row[k] = x[k];
    }
    cons_sync();
    // trailing update A[r][c] −= Σ_k L[r][k] L[c][k] over the block's 16 columns, c ≤ r
    for (int e = tid; e < nb * nb; e += kCons) {
      const int r = e / nb, c = e % nb;
      if (c > r) continue;
      const double* Lr = Cs + (b0 + SB + r) * LDC + b0;
      const double* Lc = Cs + (b0 + SB + c) * LDC + b0;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k < SB; k += 2) { s0 += Lr[k] * Lc[k]; s1 += Lr[k + 1] * Lc[k + 1]; }
      Cs[(b0 + SB + r) * LDC + b0 + SB + c] -= s0 + s1;
    }
    cons_sync();
  }
  return 0;
}

// Li (packed layout: Li[c·LDT + r] = L⁻¹(r, c)) ← the inverse of the lower-triangular L in Cs
// (row-major, stride LDC), rdv[c] = 1 / L(c, c); tmp: 3 × 256 doubles.  On 16×16 blocks: the
// diagonal blocks by forward substitution (one column per thread), then the block diagonals
// d = 1, 2, 3: L⁻¹_ij = −L⁻¹_ii Σ_{k=j}^{i−1} L_ik L⁻¹_kj.  The off-diagonal tiles of the
// column then solve X L_jjᵀ = C as the DMMA product X = C L_jj⁻ᵀ, and the solves use L_jj⁻¹.
__device__ void trinv64(const double* Cs, const double* rdv, double* Li, double* tmp) {
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += kCons) {  // blocks above the block diagonal are zero
    const int c = e >> 6, r = e & 63;
    if ((r >> 4) < (c >> 4)) Li[c * LDT + r] = 0.0;
  }
  if (tid < NB) {
    const int b0 = tid & ~(SB - 1), c = tid & (SB - 1);
    double y[SB];
#pragma unroll
    for (int r = 0; r < SB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < r; ++k) v -= Cs[(b0 + r) * LDC + b0 + k] * y[k];
      y[r] = r < c ? 0.0 : v * rdv[b0 + r];
    }
#pragma unroll
    for (int r = 0; r < SB; ++r) Li[(b0 + c) * LDT + b0 + r] = y[r];
  }
  cons_sync();
  // block diagonals d = 1 … 3 on DMMA (m8n8k4): each 16×16 block is 2×2 output tiles of 8×8,
  // warps round-robin over the diagonal's tiles
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  for (int d = 1; d < NB / SB; ++d) {
    const int ntl = (NB / SB - d) * 4;  // blocks (i, i − d), i = d … 3, × 4 tiles
    for (int tt = warp; tt < ntl; tt += kCons / 32) {  // T_ij = Σ_{k=j}^{i−1} L_ik L⁻¹_kj
      const int bi = tt >> 2, i = d + bi, j = bi, r0 = i * SB + (tt & 2) * 4, c0 = j * SB + (tt & 1) * 8;
      double t0 = 0.0, t1 = 0.0;
      for (int k0 = j * SB; k0 < i * SB; k0 += 4)
        dmma_8x8x4(t0, t1, Cs[(r0 + g) * LDC + k0 + q], Li[(c0 + g) * LDT + k0 + q]);
      const int rr = r0 - i * SB, cc = c0 - j * SB;  // position inside the 16×16 block
      tmp[(bi << 8) + (rr + g) * SB + cc + 2 * q] = t0;
      tmp[(bi << 8) + (rr + g) * SB + cc + 2 * q + 1] = t1;
    }
    cons_sync();
    for (int tt = warp; tt < ntl; tt += kCons / 32) {  // L⁻¹_ij = −L⁻¹_ii T_ij
      const int bi = tt >> 2, i = d + bi, j = bi, rr = (tt & 2) * 4, cc = (tt & 1) * 8;
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < SB; k0 += 4)
        dmma_8x8x4(v0, v1, -Li[(i * SB + k0 + q) * LDT + i * SB + rr + g], tmp[(bi << 8) + (k0 + q) * SB + cc + g]);
      Li[(j * SB + cc + 2 * q) * LDT + i * SB + rr + g] = v0;
      Li[(j * SB + cc + 2 * q + 1) * LDT + i * SB + rr + g] = v1;
    }
    cons_sync();
  }
}

// ---- consumers: tile task (i, j)
__device__ void cons_tile(const TaskCtx& t, Pipe& p, double* sm, int* sh) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, q = lane & 3;
  const bool diag = t.i == t.j;
  // acc = −A_ij + Σ_k L_ik L_jkᵀ, so C = −acc; A is loaded before the first chunk lands
  double* Out = const_cast<double*>(t.tile(t.i, t.j));
  double acc[4][2][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        acc[m][x][h] = -k_cond_entry(*t.a, t.s, t.i * NB + wr * 32 + m * 8 + g, t.j * NB + wc * 16 + x * 8 + 2 * q + h);
#ifdef PF_CHOL_CONS_THROTTLE
  const bool crit_task = t.i <= t.j + 1;
  const int* critc = t.a->crit + smid();
#endif
  for (int c = 0; c < 2 * t.j; ++c) {
#ifdef PF_CHOL_CONS_THROTTLE
    if (!crit_task) {  // experiment: the consumers of a non-critical tile also pause for the chain
      if (lane == 0)
        while (ld_relaxed(critc) > 0) __nanosleep(100);
      __syncwarp();
    }
#endif
    const double* A = cons_acquire(p, sm);
    const double* B = diag ? A : A + HALF_D;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = A[(kk + q) * LDT + wr * 32 + m * 8 + g];
#pragma unroll
      for (int x = 0; x < 2; ++x) bf[x] = B[(kk + q) * LDT + wc * 16 + x * 8 + g];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int x = 0; x < 2; ++x) dmma_8x8x4(acc[m][x][0], acc[m][x][1], af[m], bf[x]);
    }
    cons_release(p);
  }
  cons_sync();  // every warp is past the ring before the epilogue reuses it
  PF_MARK(0);
  const bool critical = t.i <= t.j + 1;
  int* crit = t.a->crit + smid();
  if (diag) {
    double* Cs = sm;               // [64][LDC] row-major
    double* Li = sm + TILE_D;      // L_jj⁻¹ (packed layout)
    double* sv = Li + TILE_D;      // [64]
    double* tmp = sv + NB;         // [3][256]
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wr * 32 + m * 8 + g, c = wc * 16 + x * 8 + 2 * q + h;
          Cs[r * LDC + c] = -acc[m][x][h];
        }
    if (tid == 0) atomicAdd(crit, 1);
    cons_sync();
    PF_MARK(1);
    const int fail = potrf64(Cs, sv, sh);
    if (!fail) trinv64(Cs, sv, Li, tmp);
    PF_MARK(2);
    if (fail && tid == 0) record_fail(t.a->info + t.s, t.j * NB + fail);
    double* Inv = const_cast<double*>(t.linv(t.j));
    for (int idx = tid; idx < NB * NB; idx += kCons) {
      const int c = idx >> 6, r = idx & 63;
      Out[c * LDT + r] = r >= c ? Cs[r * LDC + c] : 0.0;
      Inv[c * LDT + r] = fail ? 0.0 : (r >= c ? Li[c * LDT + r] : Li[r * LDT + c]);  // strict upper: L⁻ᵀ
    }
  } else {
    // C = −acc (packed layout, the DMMA A operand), then X = C L_jj⁻ᵀ on DMMA; L_jj⁻¹ is the
    // task's last ring chunk and C goes to the slot after it (consumed)
    const double* Li = cons_acquire(p, sm);
    double* Ct = stage_ptr(sm, (p.cc + 1) % NST);  // C(r, c) = Ct[c·LDT + r]
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wr * 32 + m * 8 + g, c = wc * 16 + x * 8 + 2 * q + h;
          Ct[c * LDT + r] = -acc[m][x][h];
          acc[m][x][h] = 0.0;
        }
    if (critical && tid == 0) atomicAdd(crit, 1);  // L_jj⁻¹ is here: the chain runs on this SM now
    cons_sync();
    PF_MARK(1);
#pragma unroll 4
    for (int kk = 0; kk < NB; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = Ct[(kk + q) * LDT + wr * 32 + m * 8 + g];
#pragma unroll
      for (int x = 0; x < 2; ++x) {  // L⁻¹(col, k), zero above the diagonal (the slot holds L⁻ᵀ there)
        const int col = wc * 16 + x * 8 + g;
        bf[x] = kk + q <= col ? Li[(kk + q) * LDT + col] : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int x = 0; x < 2; ++x) dmma_8x8x4(acc[m][x][0], acc[m][x][1], af[m], bf[x]);
    }
    cons_release(p);
    PF_MARK(2);
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wr * 32 + m * 8 + g, c = wc * 16 + x * 8 + 2 * q + h;
          Out[c * LDT + r] = acc[m][x][h];
        }
  }
  cons_sync();
  PF_MARK(3);
  if (tid == 0) {
    __threadfence();
    fence_proxy_global();
    st_release(t.tflag(t.i, t.j), 1);
    if (critical) atomicSub(crit, 1);
  }
}

// ---- consumers: forward solve task j, y_j = L_jj^{-1}(b_j − Σ_{k<j} L_jk y_k)
__device__ void cons_fwd(const TaskCtx& t, Pipe& p, double* sm, double* red, double* vs, double* rdv) {
  const DagArgs& a = *t.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, j = t.j, nt = a.nt;
  // warp w: rows [8w, 8w+8) of every streamed tile; lanes: columns lane, lane + 32
  double acc[kRhsCap][8];
#pragma unroll
  for (int rr = 0; rr < kRhsCap; ++rr)
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) acc[rr][r8] = 0.0;
  for (int k = 0; k < j; ++k) {
    const double* Tk = cons_acquire(p, sm);
    if (lane == 0) wait_flag(t.fwdflag(k));
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < kRhsCap; ++rr) {
      if (rr < a.nrhs) {
        const double* yk = a.cy + ((size_t)t.s * 2 * kRhsCap + rr) * nt * NB + k * NB;
        const double y0 = __ldcg(yk + lane), y1 = __ldcg(yk + lane + 32);
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8)
          acc[rr][r8] += Tk[lane * LDT + 8 * warp + r8] * y0 + Tk[(lane + 32) * LDT + 8 * warp + r8] * y1;
      }
    }
    cons_release(p);
  }
#pragma unroll
  for (int rr = 0; rr < kRhsCap; ++rr)
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) {
      double v = acc[rr][r8];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && rr < a.nrhs) red[rr * NB + 8 * warp + r8] = v;
    }
  cons_sync();
  mbar_wait(p.lbar, p.lpar);  // L_jj⁻¹ (lower: Li[c·LDT + r] = L⁻¹(r, c), r ≥ c)
  p.lpar ^= 1;
  const double* Li = sm;
  for (int idx = tid; idx < a.nrhs * NB; idx += kCons) {
    const int rr = idx >> 6, r = idx & 63, R = j * NB + r;
    const double b = R < a.n ? a.rhs[((size_t)(a.sidx ? a.sidx[t.s] : t.s) * a.rhs_ld + rr) * a.n + R] : 0.0;
    vs[rr * NB + r] = b - red[rr * NB + r];
  }
  cons_sync();
  if (warp < a.nrhs) {  // y = L⁻¹ v, one warp per right-hand side: lane owns rows lane, lane + 32
    const double* v = vs + warp * NB;
    double y0[4] = {0.0, 0.0, 0.0, 0.0}, y1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
    for (int c = 0; c < NB; ++c) {
      const double vc = v[c];
      if (c <= lane) y0[c & 3] += Li[c * LDT + lane] * vc;
      y1[c & 3] += Li[c * LDT + lane + 32] * (c <= lane + 32 ? vc : 0.0);
    }
    const double ya = (y0[0] + y0[1]) + (y0[2] + y0[3]), yb = (y1[0] + y1[1]) + (y1[2] + y1[3]);
    double* yo = a.cy + ((size_t)t.s * 2 * kRhsCap + warp) * nt * NB + j * NB;
    __stcg(yo + lane, ya);
    __stcg(yo + lane + 32, yb);
  }
  cons_sync();
  if (tid == 0) {
    __threadfence();
    st_release(t.fwdflag(j), 1);
  }
}

// ---- consumers: backward solve task j, p_j = L_jj^{-T}(y_j − Σ_{i>j} L_ijᵀ p_i)
__device__ void cons_bwd(const TaskCtx& t, Pipe& p, double* sm, double* red, double* vs, double* rdv, int* sh) {
  const DagArgs& a = *t.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, j = t.j, nt = a.nt;
  // warp w: columns c = 8w..8w+7 of every streamed tile, lanes over its rows
  double acc[kRhsCap][8];
#pragma unroll
  for (int rr = 0; rr < kRhsCap; ++rr)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[rr][c] = 0.0;
  for (int i = nt - 1; i > j; --i) {
    const double* Ti = cons_acquire(p, sm);
    if (lane == 0) wait_flag(t.bwdflag(i));
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < kRhsCap; ++rr) {
      if (rr < a.nrhs) {
        const double* pi = a.cy + ((size_t)t.s * 2 * kRhsCap + kRhsCap + rr) * nt * NB + i * NB;
        const double p0 = __ldcg(pi + lane), p1 = __ldcg(pi + lane + 32);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          acc[rr][c] += Ti[(8 * warp + c) * LDT + lane] * p0 + Ti[(8 * warp + c) * LDT + lane + 32] * p1;
      }
    }
    cons_release(p);
  }
#pragma unroll
  for (int rr = 0; rr < kRhsCap; ++rr)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double v = acc[rr][c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && rr < a.nrhs) red[rr * NB + 8 * warp + c] = v;
    }
  if (tid == 0) {
    wait_flag(t.fwdflag(j));
    sh[0] = *(volatile int*)(a.info + t.s) == 0;
  }
  cons_sync();  // red and y_j visible to every consumer
  mbar_wait(p.lbar, p.lpar);  // L_jj⁻¹ with L⁻ᵀ in the strict upper part: Li[c·LDT + r] = L⁻¹(c, r) for r < c
  p.lpar ^= 1;
  const double* Li = sm;
  for (int idx = tid; idx < a.nrhs * NB; idx += kCons) {
    const int rr = idx >> 6, c = idx & 63;
    vs[rr * NB + c] = __ldcg(a.cy + ((size_t)t.s * 2 * kRhsCap + rr) * nt * NB + j * NB + c) - red[rr * NB + c];
  }
  cons_sync();
  const bool ok = sh[0];
  if (ok && warp < a.nrhs) {  // p = L⁻ᵀ v: p_r = Σ_{c ≥ r} L⁻¹(c, r) v_c; lane owns entries lane, lane + 32
    const double* v = vs + warp * NB;
    double q0[4] = {0.0, 0.0, 0.0, 0.0}, q1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
    for (int c = 0; c < NB; ++c) {
      const double vc = v[c];
      q0[c & 3] += Li[c * LDT + lane] * (c >= lane ? vc : 0.0);
      if (c >= lane + 32) q1[c & 3] += Li[c * LDT + lane + 32] * vc;
    }
    const double v0 = (q0[0] + q0[1]) + (q0[2] + q0[3]), v1 = (q1[0] + q1[1]) + (q1[2] + q1[3]);
    double* po = a.cy + ((size_t)t.s * 2 * kRhsCap + kRhsCap + warp) * nt * NB + j * NB;
    __stcg(po + lane, v0);
    __stcg(po + lane + 32, v1);
    double* out = a.rhs + ((size_t)(a.sidx ? a.sidx[t.s] : t.s) * a.rhs_ld + warp) * a.n;
    if (j * NB + lane < a.n) out[j * NB + lane] = v0;
    if (j * NB + lane + 32 < a.n) out[j * NB + lane + 32] = v1;
  }
  cons_sync();
  if (tid == 0) {
    __threadfence();
    st_release(t.bwdflag(j), 1);
  }
}

__global__ void __launch_bounds__(kDagThreads, 2) k_chol_dag(DagArgs a) {
  extern __shared__ __align__(128) double sm_dag[];
  __shared__ __align__(8) uint64_t bars[2 * NST + 1];
  __shared__ double red[kRhsCap * NB], vsol[kRhsCap * NB], rdv[NB];
  __shared__ int task[5];
  __shared__ int sh[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < NST; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bars + b)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(saddr(bars + NST + b)) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bars + 2 * NST)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Pipe p{bars, bars + NST, bars + 2 * NST, 0u, 0u};
  const int f = a.nrhs > 0 ? 1 : 0;
  for (;;) {
    if (tid == 0) {
      int t = atomicAdd(a.ticket, 1);
      task[4] = t;
      int kind = T_DONE, s = 0, i = 0, j = 0;
      if (t < a.ntask) {
        // Topological order with a look-ahead band of kLook columns: group g holds,
        // per scenario, row g+kLook's tiles (g+kLook, c) for c = max(g, 0) … g+kLook
        // (the band next to the diagonal, in column order), then the rest of
        // column g, (i, g) for i > g+kLook, then the forward-solve task g.  So the
        // tiles on and next to the diagonal — the column chain — are handed out
        // kLook columns early and have accumulated all but their last products
        // when the chain reaches them.  Then the backward-solve tasks.
        const int nt = a.nt;
        auto band_g = [&](int g) {
          const int r = g + kLook;
          return (a.factor && r >= 0 && r < nt) ? r - max(g, 0) + 1 : 0;
        };
        auto rest_g = [&](int g) { return (a.factor && g >= 0) ? max(0, nt - (g + kLook + 1)) : 0; };
        int g = -kLook;
        for (; g < nt; ++g) {
          const int nb = band_g(g), nr = rest_g(g), per = nb + nr + ((g >= 0 && f) ? 1 : 0), grp = a.S * per;
          if (t < grp) {
            s = t / per;
            const int r = t % per;
            if (r < nb) { kind = T_TILE; i = g + kLook; j = max(g, 0) + r; }
            else if (r < nb + nr) { kind = T_TILE; i = g + kLook + 1 + (r - nb); j = g; }
            else { kind = T_FWD; j = g; }
            break;
          }
          t -= grp;
        }
        if (g == nt) { kind = T_BWD; j = nt - 1 - t / a.S; s = t % a.S; }
        // a scenario that already failed at an earlier column skips its remaining tiles
        if (kind == T_TILE) {
          const int inf = *(volatile int*)(a.info + s);
          if (inf != 0 && inf <= j * NB) kind = -T_TILE;
        }
      }
      task[0] = kind; task[1] = s; task[2] = i; task[3] = j;
    }
    __syncthreads();
    const int kind = task[0], s = task[1], i = task[2], j = task[3];
    if (kind == T_DONE) break;
#ifdef PF_CHOL_TRACE
    const unsigned long long t0 = gtimer();
#endif
    TaskCtx t{&a, s, i, j, a.tiles + (size_t)s * tstride(a.nt) * TILE_D, a.flags + (size_t)s * (a.ntri + 2 * a.nt)};
    if (kind == -T_TILE) {
      if (tid == 0) st_release(t.tflag(i, j), 1);  // skipped: publish so dependants proceed
    } else if (tid >= kCons) {
      if (tid == kCons) produce(t, kind, p, sm_dag);
      else {  // keep the ring position of the other producer lanes in step (unused)
      }
    } else if (kind == T_TILE) {
      cons_tile(t, p, sm_dag, sh);
    } else if (kind == T_FWD) {
      cons_fwd(t, p, sm_dag, red, vsol, rdv);
    } else {
      cons_bwd(t, p, sm_dag, red, vsol, rdv, sh);
    }
    fence_proxy_shared();  // this task's generic SMEM writes before the next task's bulk copies
    __syncthreads();
#ifdef PF_CHOL_TRACE
    if (tid == 0 && g_chol_trace) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* e = g_chol_trace + 8 * (size_t)task[4];
      e[0] = ((unsigned long long)(kind & 0xff) << 56) | ((unsigned long long)s << 40) |
             ((unsigned long long)i << 20) | (unsigned long long)j;
      e[1] = smid; e[2] = t0; e[3] = gtimer();
      for (int m = 0; m < 4; ++m) { e[4 + m] = g_marks[m]; g_marks[m] = 0; }
    }
#endif
  }
}

__global__ void k_info_out(int n_scen, const int* __restrict__ ws, int* __restrict__ out, const int* __restrict__ sidx) {
  for (int s = threadIdx.x; s < n_scen; s += blockDim.x) out[sidx ? sidx[s] : s] = ws[s];
}

}  // namespace

size_t chol_tile_doubles(int n_u) { return tstride((n_u + NB - 1) / NB) * TILE_D; }
size_t chol_flag_ints(int n_u) {
  const size_t nt = (n_u + NB - 1) / NB;
  return nt * (nt + 1) / 2 + 2 * nt;
}
size_t chol_vec_doubles(int n_u) { return 2 * (size_t)kRhsCap * ((n_u + NB - 1) / NB) * NB; }

int chol_grid_max() {
  cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, kDagSmem);
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_dag, kDagThreads, kDagSmem);
  cudaGetLastError();
  return std::max(1, sms * std::max(per, 1));
}

int launch_chol(const DevNet& net, const Work& w, int n_scen, double* K, const double* sigma_u, double delta_w,
                double* rhs, int nrhs, int* info, int* info_ws, cudaStream_t st, int grid_max, const int* sidx,
                const double* dvec, cudaEvent_t* ev) {
  const int n = net.n_u, nt = (n + NB - 1) / NB, ntri = nt * (nt + 1) / 2;
  cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, kDagSmem);  // per device, idempotent
  int launches = 0;
  k_chol_reset<<<(int)std::min<long long>(1024, ((long long)n_scen * (ntri + 2 * nt) + 255) / 256), 256, 0, st>>>(
      nt, n_scen, w.cflag, w.cticket, info_ws, w.cticket + 1);
  ++launches;
  // the factorization runs with the first kRhsCap right-hand sides fused in; further
  // ones (rare) in solve-only runs over the finished factor
  if (ev) cudaEventRecord(ev[0], st);
  for (int r0 = 0, first = 1; first || r0 < nrhs; r0 += kRhsCap, first = 0) {
    const int nr = std::max(0, std::min(kRhsCap, nrhs - r0)), f = nr > 0 ? 1 : 0;
    if (!first) {
      k_chol_reset_solve<<<1, 256, 0, st>>>(nt, n_scen, w.cflag, w.cticket);
      ++launches;
    }
    DagArgs a;
    a.n = n; a.nt = nt; a.ntri = ntri; a.S = n_scen; a.nrhs = nr; a.factor = first; a.rhs_ld = nrhs;
    a.ntask = n_scen * ((first ? ntri : 0) + f * nt) + f * n_scen * nt;
    a.tiles = w.ctile; a.flags = w.cflag; a.ticket = w.cticket; a.info = info_ws;
    a.cy = w.cy; a.rhs = rhs ? rhs + (size_t)r0 * n : nullptr; a.crit = w.cticket + 1; a.sidx = sidx;
    a.K = K; a.sig_u = sigma_u; a.delta = delta_w; a.dvec = dvec;
    if (a.ntask > 0) {
      k_chol_dag<<<std::min(grid_max, a.ntask), kDagThreads, kDagSmem, st>>>(a);
      ++launches;
    }
  }
  if (ev) cudaEventRecord(ev[1], st);
  k_chol_unpack<<<dim3(nt, nt, n_scen), 256, 0, st>>>(n, nt, w.ctile, K, info_ws, sidx);
  ++launches;
  if (info) { k_info_out<<<1, 256, 0, st>>>(n_scen, info_ws, info, sidx); ++launches; }
  return launches;
}

}  // namespace pf
