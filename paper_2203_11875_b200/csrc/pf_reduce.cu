// pf_reduce.cu — the batched reduced-Hessian kernels (A7.1–A7.5 of SURVEY §8(a)).
//
// The paper's three steps for K̂V (with R11) over tiles of C
// directions of one scenario:
//   k_fwd  a. B = −P G_u V       (unit V: a column scatter; dense V: a row SpMM)
//          b. Z̃ = U^{-1} L^{-1} B (level-scheduled sweeps over bus blocks)
//   k_mu   c1. μ_A = Σ_r ⊙ R_r M dψ at the r buses (generator buses)
//   k_hvp  c2. [H_u; H_x] = K [V; Z] matrix-free through ψ (line-local J_ψ,
//              L_line, ∇²ψ with w̄, the r-row / p_ref terms, AᵀΣ_sA, Σ_x),
//              one team per bus gathering its incident lines (no atomics)
//   k_adj  d. Ψ̃ = L^{-T} U^{-T} H̃_x  (transposed sweeps, same level sets)
//          e. K̂V = H_u − (P G_u)ᵀ Ψ̃  (column gathers, SMEM-transposed store)
// Slabs are [n_x][C] per tile, direction fastest: a team of C lanes handles
// one row, lane j = direction j, so every slab access is one contiguous C×8 B
// run.  Sweep nonzeros are packed {value, column·C} (one 16-byte load each),
// fetched lane-parallel and broadcast by shuffles (see sweep()).
// Every column's arithmetic is independent of N, the tile and the GPU count,
// so K̂ is bit-identical across batch sizes.
#include "pf_launch.h"

#include <cstdlib>

namespace pf {

namespace {

constexpr int kThreads = 256;
constexpr int kCH = 64;        // u-columns per transposed output chunk
constexpr int kBusPerCta = 64; // buses per k_hvp CTA
#ifndef PF_DOT_W
#define PF_DOT_W 4
#endif
#ifndef PF_SWEEP_MIN_BLOCKS
#define PF_SWEEP_MIN_BLOCKS 3
#endif
constexpr int kSweepMinBlocks = PF_SWEEP_MIN_BLOCKS;  // CTAs per SM the sweep kernels are register-capped for

__device__ __forceinline__ double2 ldpk(const double2* p) { return __ldg(p); }

// A level-scheduled triangular sweep over bus blocks (1–2 rows each), driven
// by a per-level task list built on the host (pf_api.cu, one int4 per block):
//   {r0 | two << 31, start of row 0's entries, start of row 1's, cnt0 << 16 | cnt1}
// where each row's packed {value, column·C} entries are ONE contiguous range
// that includes its diagonal and the intra-block entry:
//   LOWER (L, Uᵀ; strict-lower parts, rows forward):
//     row 0 (θ): [lower part..., diag]    row 1 (v): [lower part..., (v,θ), diag]
//   UPPER (U, Lᵀ; strict-upper parts, rows backward):
//     row 1 (v): [diag, upper part...]    row 0 (θ): [diag, (θ,v), upper part...]
// The v row of a LOWER block (θ row of an UPPER block) depends on its partner
// only through the intra entry, applied once the partner is final.  A row's
// range is fetched lane-parallel (one coalesced load) and broadcast by
// shuffles; the next block's task and ranges are prefetched while the current
// block's slab loads (16 at a time, all issued before the first FMA) are in
// flight, so a block costs about one memory round trip.
struct Task { int r0, s0, s1, c0, c1; bool two; };

// The lanes of this thread's team (C consecutive lanes of the warp): teams of
// one warp follow different rows, so every shuffle names only its own team.
template <int C>
__device__ __forceinline__ unsigned team_mask() {
  if constexpr (C == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31;
    return ((1u << C) - 1u) << (lane & ~(unsigned)(C - 1));
  }
}
__device__ __forceinline__ Task unpack(int4 t) {
  Task k;
  k.r0 = t.x & 0x7fffffff; k.two = (t.x >> 31) & 1;
  k.s0 = t.y; k.s1 = t.z; k.c0 = t.w >> 16; k.c1 = t.w & 0xffff;
  return k;
}

template <int C>
__device__ __forceinline__ double2 fetch(const double2* __restrict__ pk, int s, int cnt, int i) {
  return i < cnt ? ldpk(pk + s + i) : make_double2(0.0, 0.0);
}

constexpr int kDotW = PF_DOT_W;  // slab loads per row issued before the FMAs

template <int C>
__device__ __forceinline__ double shv(unsigned mask, double2 q, int e) { return __shfl_sync(mask, q.x, e, C); }

// acc0 -= Σ_{k<n0} v0[o0+k] X[c0[o0+k]],  acc1 likewise (entries held one per
// lane in q0 / q1, all within one fetch of ≤ C entries).
template <int C>
__device__ __forceinline__ void dot2(const double* X, unsigned mask, int lane, double2 q0, int o0, int n0,
                                     double2 q1, int o1, int n1, double& acc0, double& acc1) {
  const int m = max(n0, n1);
  for (int e0 = 0; e0 < m; e0 += kDotW) {
    double x0[kDotW], x1[kDotW];
#pragma unroll
    for (int k = 0; k < kDotW; ++k) {
      const int i0 = (o0 + e0 + k) & (C - 1), i1 = (o1 + e0 + k) & (C - 1);
      const long long c0 = __double_as_longlong(__shfl_sync(mask, q0.y, i0, C));
      const long long c1 = __double_as_longlong(__shfl_sync(mask, q1.y, i1, C));
      x0[k] = e0 + k < n0 ? X[c0 + lane] : 0.0;
      x1[k] = e0 + k < n1 ? X[c1 + lane] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kDotW; ++k) {
      const int i0 = (o0 + e0 + k) & (C - 1), i1 = (o1 + e0 + k) & (C - 1);
      acc0 -= (e0 + k < n0 ? __shfl_sync(mask, q0.x, i0, C) : 0.0) * x0[k];
      acc1 -= (e0 + k < n1 ? __shfl_sync(mask, q1.x, i1, C) : 0.0) * x1[k];
    }
  }
}

// Rows longer than one fetch (separator rows of the L part): chunked, no prefetch.
template <int C>
__device__ __forceinline__ double dot_long(const double2* __restrict__ pk, const double* X, unsigned mask, int lane,
                                           int s, int n) {
  double acc = 0.0, dummy = 0.0;  // dot2 subtracts: acc = −Σ, returned as +Σ
  for (int base = 0; base < n; base += C) {
    const double2 q = fetch<C>(pk, s + base, n - base, lane);
    dot2<C>(X, mask, lane, q, 0, min(C, n - base), q, 0, 0, acc, dummy);
  }
  return -acc;
}

template <int C, bool LOWER>
__device__ __forceinline__ void sweep(const DevNet& n, const int4* __restrict__ tasks, const double2* __restrict__ pk,
                                      double* X, bool divide, int lane, int team, int nteam) {
  const int nlev = LOWER ? n.nlevL : n.nlevU;
  const int* lptr = LOWER ? n.levL_ptr : n.levU_ptr;
  const unsigned mask = team_mask<C>();
  for (int lev = 0; lev < nlev; ++lev) {
    const int b1 = __ldg(lptr + lev + 1);
    int bi = __ldg(lptr + lev) + team;
    Task nk;
    double2 nq0 = make_double2(0.0, 0.0), nq1 = nq0;
    if (bi < b1) {
      nk = unpack(__ldg(tasks + bi));
      nq0 = fetch<C>(pk, nk.s0, nk.c0, lane);
      if (nk.two) nq1 = fetch<C>(pk, nk.s1, nk.c1, lane);
    }
    for (; bi < b1; bi += nteam) {
      const Task k = nk;
      const double2 q0 = nq0, q1 = nq1;
      if (bi + nteam < b1) {  // prefetch the next block of this team
        nk = unpack(__ldg(tasks + bi + nteam));
        nq0 = fetch<C>(pk, nk.s0, nk.c0, lane);
        if (nk.two) nq1 = fetch<C>(pk, nk.s1, nk.c1, lane);
      }
      double a0 = X[k.r0 * C + lane], a1 = k.two ? X[(k.r0 + 1) * C + lane] : 0.0;
      if (LOWER) {
        const int n0 = k.c0 - 1, n1 = k.two ? k.c1 - 2 : 0;      // entries before diag / intra
        if (k.c0 <= C && k.c1 <= C) {
          dot2<C>(X, mask, lane, q0, 0, n0, q1, 0, n1, a0, a1);
        } else {
          a0 -= dot_long<C>(pk, X, mask, lane, k.s0, n0);
          if (k.two) a1 -= dot_long<C>(pk, X, mask, lane, k.s1, n1);
        }
        const double d0 = k.c0 <= C ? shv<C>(mask, q0, (k.c0 - 1) & (C - 1)) : ldpk(pk + k.s0 + k.c0 - 1).x;
        double x0 = a0;
        if (divide) x0 /= d0;
        X[k.r0 * C + lane] = x0;
        if (k.two) {
          const bool in = k.c1 <= C;
          const double intra = in ? shv<C>(mask, q1, (k.c1 - 2) & (C - 1)) : ldpk(pk + k.s1 + k.c1 - 2).x;
          const double d1 = in ? shv<C>(mask, q1, (k.c1 - 1) & (C - 1)) : ldpk(pk + k.s1 + k.c1 - 1).x;
          double x1 = a1 - intra * x0;
          if (divide) x1 /= d1;
          X[(k.r0 + 1) * C + lane] = x1;
        }
      } else {
        // upper parts are short (≤ one fetch): row 1 = [diag, U...], row 0 = [diag, intra?, U...]
        const int o0 = k.two ? 2 : 1;
        const int n0 = k.c0 - o0, n1 = k.two ? k.c1 - 1 : 0;
        if (k.c0 <= C && k.c1 <= C) {
          dot2<C>(X, mask, lane, q0, o0, n0, q1, 1, n1, a0, a1);
        } else {
          a0 -= dot_long<C>(pk, X, mask, lane, k.s0 + o0, n0);
          if (k.two) a1 -= dot_long<C>(pk, X, mask, lane, k.s1 + 1, n1);
        }
        double x1 = 0.0;
        if (k.two) {
          x1 = a1;
          if (divide) x1 /= (k.c1 <= C ? shv<C>(mask, q1, 0) : ldpk(pk + k.s1).x);
          X[(k.r0 + 1) * C + lane] = x1;
        }
        double x0 = a0;
        if (k.two) x0 -= (k.c0 <= C ? shv<C>(mask, q0, 1) : ldpk(pk + k.s0 + 1).x) * x1;
        if (divide) x0 /= (k.c0 <= C ? shv<C>(mask, q0, 0) : ldpk(pk + k.s0).x);
        X[k.r0 * C + lane] = x0;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- a, b
template <int C>
__global__ void __launch_bounds__(kThreads, kSweepMinBlocks) k_fwd(DevNet n, Work w, const double* __restrict__ V, int col0, int N) {
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % C, team = threadIdx.x / C, nteam = blockDim.x / C;
  const int j = tile * C + lane;
  const bool valid = j < N;
  const int n_x = n.n_x, n_u = n.n_u;
  double* X = w.slabZ + cta * n_x * C;
  const double* gu = w.gu + (size_t)s * n.nnz_gu;
  const double2* pk = w.pkA + (size_t)s * n.nnz_lu;
  if (V == nullptr) {  // A7.1 for unit directions: a scatter of G_u's column col0 + j
    for (int idx = threadIdx.x; idx < n_x * C; idx += blockDim.x) X[idx] = 0.0;
    __syncthreads();
    if (team == 0 && valid) {
      const int c = col0 + j;
      for (int e = __ldg(n.guc_ptr + c); e < __ldg(n.guc_ptr + c + 1); ++e)
        X[__ldg(n.guc_row + e) * C + lane] = -gu[__ldg(n.guc_src + e)];
    }
  } else {             // A7.1 for dense directions: B = −P G_u V (row SpMM)
    const double* Vs = V + ((size_t)s * N + (valid ? j : 0)) * n_u;
    for (int r = team; r < n_x; r += nteam) {
      double acc = 0.0;
      if (valid)
        for (int e = __ldg(n.gur_ptr + r); e < __ldg(n.gur_ptr + r + 1); ++e)
          acc += gu[__ldg(n.gur_src + e)] * Vs[__ldg(n.gur_col + e)];
      X[r * C + lane] = -acc;
    }
  }
  __syncthreads();
  sweep<C, true>(n, n.taskL, pk, X, false, lane, team, nteam);   // L^{-1}
  sweep<C, false>(n, n.taskU, pk, X, true, lane, team, nteam);   // U^{-1}
}

// ---------------------------------------------------------------- directions in bus space
struct Dir {
  const double* X;
  const double* Vs;
  int lane, col;  // col = col0 + j for unit directions
  bool valid;
  __device__ __forceinline__ double vdir(int c) const {
    if (!valid) return 0.0;
    return Vs ? Vs[c] : (c == col ? 1.0 : 0.0);
  }
};

template <int C>
__device__ __forceinline__ double dth_of(const DevNet& n, const Dir& d, int i) {
  const int p = __ldg(n.bus_pth + i);
  return p >= 0 ? d.X[p * C + d.lane] : 0.0;
}
template <int C>
__device__ __forceinline__ double dv_of(const DevNet& n, const Dir& d, int i) {
  const int p = __ldg(n.bus_pv + i);
  return p >= 0 ? d.X[p * C + d.lane] : d.vdir(__ldg(n.u_v + i));
}
// Direction at the far end of an incidence record {line, θ row, v row or
// −1−(u index), 1·from | 2·(gen + 1)} of the far bus (pf_api.cu builds them).
template <int C>
__device__ __forceinline__ double rec_dth(const Dir& d, int4 rec) {
  return rec.y >= 0 ? d.X[rec.y * C + d.lane] : 0.0;
}
template <int C>
__device__ __forceinline__ double rec_dv(const Dir& d, int4 rec) {
  return rec.z >= 0 ? d.X[rec.z * C + d.lane] : d.vdir(-1 - rec.z);
}

template <int C>
__device__ __forceinline__ Dir make_dir(const DevNet& n, const Work& w, const double* V, int col0, int N, int s,
                                        int tile, size_t cta, int lane) {
  Dir d;
  d.lane = lane;
  const int j = tile * C + lane;
  d.valid = j < N;
  d.col = col0 + j;
  d.X = w.slabZ + cta * n.n_x * C;
  d.Vs = (V && d.valid) ? V + ((size_t)s * N + j) * n.n_u : nullptr;
  return d;
}

// Line block of K (pf_eval.cu k_prep_line): H (3×3 sym) and J (4×3) on the
// local coordinates (v_f, v_t, Δ), 9 × 16-byte loads.
struct LBlk { double h[6], j[12]; };
__device__ __forceinline__ void load_h(const double* p, double* h) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  h[0] = a.x; h[1] = a.y; h[2] = b.x; h[3] = b.y; h[4] = c.x; h[5] = c.y;
}
__device__ __forceinline__ void load_j(const double* p, double* j) {
  const double2* q = reinterpret_cast<const double2*>(p + LB_J);
#pragma unroll
  for (int k = 0; k < 6; ++k) { const double2 v = __ldg(q + k); j[2 * k] = v.x; j[2 * k + 1] = v.y; }
}

// ---------------------------------------------------------------- c1
// μ_A at the generator buses: dG = R_r M dψ = Σ_{ends at i} J_end · d_loc plus
// the shunt part of G_ii ψ^d; μ_A = Σ_r dG (+ 2c1 dG on P_r0, folded into Σ_rP).
template <int C>
__global__ void __launch_bounds__(kThreads) k_mu(DevNet n, Work w, const double* __restrict__ V, int col0, int N) {
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.y, s = blockIdx.z;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % C, team = threadIdx.x / C, nteam = blockDim.x / C;
  const int gi = blockIdx.x * nteam + team;
  if (gi >= n.n_gb) return;
  const Dir d = make_dir<C>(n, w, V, col0, N, s, tile, cta, lane);
  const int n_b = n.n_b;
  const double* lb = w.lblk + (size_t)s * n.n_l * LB_N;
  const double* bs = w.bs + (size_t)s * BS_N * n_b;
  const int i = __ldg(n.gbus + gi);
  const double dvi = dv_of<C>(n, d, i), dthi = dth_of<C>(n, d, i);
  double dP = 0.0, dQ = 0.0;
  for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
    const int4 rec = __ldg(n.inc_rec + e);
    const int l = rec.x;
    const bool from = rec.w & 1;
    const double dvo = rec_dv<C>(d, rec), dtho = rec_dth<C>(d, rec);
    const double dvf = from ? dvi : dvo, dvt = from ? dvo : dvi;
    const double dD = from ? dthi - dtho : dtho - dthi;
    double J[12];
    load_j(lb + (size_t)l * LB_N, J);
    // rows (s_p, s_q) of this end
    dP += from ? J[0] * dvf + J[1] * dvt + J[2] * dD : J[6] * dvf + J[7] * dvt + J[8] * dD;
    dQ += from ? J[3] * dvf + J[4] * dvt + J[5] * dD : J[9] * dvf + J[10] * dvt + J[11] * dD;
  }
  const double vi = bs[BS_V * n_b + i];
  dP += 2.0 * __ldg(n.gsh + i) * vi * dvi;
  dQ -= 2.0 * __ldg(n.bsh + i) * vi * dvi;
  double* MU = w.mu + cta * n.n_g * 2 * C;
  const int g = __ldg(n.bus_gen + i);
  MU[(2 * g) * C + lane] = bs[BS_SRP * n_b + i] * dP;
  MU[(2 * g + 1) * C + lane] = bs[BS_SRQ * n_b + i] * dQ;
}

// ---------------------------------------------------------------- c2
// [H_u; H_x] = K [V; Z]: per bus, Σ over incident lines of the line block
// (H d_loc + Jᵀ μ_A(ends)) restricted to the bus's own (v, θ), plus the bus
// terms 2w̄^d dv (ψ^d curvature), the shunt part of Mᵀμ_A, and Σ_x.
template <int C>
__global__ void __launch_bounds__(kThreads) k_hvp(DevNet n, Work w, const double* __restrict__ V, int col0, int N) {
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.y, s = blockIdx.z;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % C, team = threadIdx.x / C, nteam = blockDim.x / C;
  const Dir d = make_dir<C>(n, w, V, col0, N, s, tile, cta, lane);
  const int n_b = n.n_b;
  const double* lb = w.lblk + (size_t)s * n.n_l * LB_N;
  const double* bs = w.bs + (size_t)s * BS_N * n_b;
  const double* MU = w.mu + cta * n.n_g * 2 * C;
  double* Y = w.slabW + cta * n.n_x * C;
  double* Hs = w.hu + cta * n.n_u * C;
  const int k1 = min(n_b, (int)(blockIdx.x + 1) * kBusPerCta);
  // buses in elimination order: a chunk's own θ/v rows are contiguous slab rows
  for (int kb = blockIdx.x * kBusPerCta + team; kb < k1; kb += nteam) {
    const int i = __ldg(n.hvp_bus + kb);
    const double dvi = dv_of<C>(n, d, i), dthi = dth_of<C>(n, d, i);
    const int gi_own = __ldg(n.bus_gen + i);
    const double mPi = gi_own >= 0 ? MU[(2 * gi_own) * C + lane] : 0.0;
    const double mQi = gi_own >= 0 ? MU[(2 * gi_own + 1) * C + lane] : 0.0;
    double hv = 0.0, hth = 0.0;
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int4 rec = __ldg(n.inc_rec + e);
      const int l = rec.x;
      const bool from = rec.w & 1;
      const double dvo = rec_dv<C>(d, rec), dtho = rec_dth<C>(d, rec);
      const double dvf = from ? dvi : dvo, dvt = from ? dvo : dvi;
      const double dD = from ? dthi - dtho : dtho - dthi;
      const double* p = lb + (size_t)l * LB_N;
      double h[6];
      load_h(p, h);
      const double hvv = from ? h[0] * dvf + h[1] * dvt + h[2] * dD : h[1] * dvf + h[3] * dvt + h[4] * dD;
      double hD = h[2] * dvf + h[4] * dvt + h[5] * dD;
      double hvo = hvv;
      const int go = (rec.w >> 1) - 1;
      if (gi_own >= 0 || go >= 0) {  // Jᵀ μ_A: only lines touching an r bus
        double J[12];
        load_j(p, J);
        const double mPo = go >= 0 ? MU[(2 * go) * C + lane] : 0.0;
        const double mQo = go >= 0 ? MU[(2 * go + 1) * C + lane] : 0.0;
        const double mpf = from ? mPi : mPo, mqf = from ? mQi : mQo;
        const double mpt = from ? mPo : mPi, mqt = from ? mQo : mQi;
        hvo += from ? J[0] * mpf + J[3] * mqf + J[6] * mpt + J[9] * mqt
                    : J[1] * mpf + J[4] * mqf + J[7] * mpt + J[10] * mqt;
        hD += J[2] * mpf + J[5] * mqf + J[8] * mpt + J[11] * mqt;
      }
      hv += hvo;
      hth += from ? hD : -hD;
    }
    const double vi = bs[BS_V * n_b + i];
    hv += bs[BS_WD2 * n_b + i] * dvi + 2.0 * vi * (__ldg(n.gsh + i) * mPi - __ldg(n.bsh + i) * mQi);
    hv += bs[BS_SXV * n_b + i] * dvi;
    hth += bs[BS_SXT * n_b + i] * dthi;
    const int pt = __ldg(n.bus_pth + i), pv = __ldg(n.bus_pv + i);
    if (pt >= 0) Y[pt * C + lane] = hth;
    if (pv >= 0) Y[pv * C + lane] = hv;
    else Hs[__ldg(n.u_v + i) * C + lane] = hv;
  }
  if (blockIdx.x == 0)  // objective curvature on explicit p_g
    for (int g = team; g < n.n_g; g += nteam) {
      const int up = __ldg(n.u_p + g);
      if (up >= 0) Hs[up * C + lane] = 2.0 * __ldg(n.c_quad + g) * d.vdir(up);
    }
}

// ---------------------------------------------------------------- d, e
template <int C>
__global__ void __launch_bounds__(kThreads, kSweepMinBlocks) k_adj(DevNet n, Work w, int N, double* __restrict__ KV) {
  __shared__ double T[C][kCH + 1];
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % C, team = threadIdx.x / C, nteam = blockDim.x / C;
  const int n_x = n.n_x, n_u = n.n_u;
  double* Y = w.slabW + cta * n_x * C;
  const double* Hs = w.hu + cta * n_u * C;
  const double* gu = w.gu + (size_t)s * n.nnz_gu;
  const double2* pk = w.pkT + (size_t)s * n.nnz_lu;
  sweep<C, true>(n, n.taskL, pk, Y, true, lane, team, nteam);    // U^{-T}
  sweep<C, false>(n, n.taskU, pk, Y, false, lane, team, nteam);  // L^{-T}
  for (int c0 = 0; c0 < n_u; c0 += kCH) {
    for (int cc = team; cc < kCH && c0 + cc < n_u; cc += nteam) {
      const int c = c0 + cc;
      double acc = Hs[c * C + lane];
      for (int e = __ldg(n.guc_ptr + c); e < __ldg(n.guc_ptr + c + 1); ++e)
        acc -= gu[__ldg(n.guc_src + e)] * Y[__ldg(n.guc_row + e) * C + lane];
      T[lane][cc] = acc;
    }
    __syncthreads();
    const int w_c = min(kCH, n_u - c0);
    for (int idx = threadIdx.x; idx < C * kCH; idx += blockDim.x) {
      const int jl = idx / kCH, cc = idx % kCH;
      const int jj = tile * C + jl;
      if (jj < N && cc < w_c) KV[((size_t)s * N + jj) * n_u + c0 + cc] = T[jl][cc];
    }
    __syncthreads();
  }
}

template <int C>
void launch_all(const DevNet& n, const Work& w, int n_scen, const double* V, int col0, int N, double* KV,
                cudaStream_t st, cudaEvent_t* ev) {
  const int ntile = (N + C - 1) / C;
  const int teams = kThreads / C;
  if (ev) cudaEventRecord(ev[0], st);
  k_fwd<C><<<dim3(ntile, n_scen), kThreads, 0, st>>>(n, w, V, col0, N);
  if (ev) cudaEventRecord(ev[1], st);
  k_mu<C><<<dim3((n.n_gb + teams - 1) / teams, ntile, n_scen), kThreads, 0, st>>>(n, w, V, col0, N);
  if (ev) cudaEventRecord(ev[2], st);
  k_hvp<C><<<dim3((n.n_b + kBusPerCta - 1) / kBusPerCta, ntile, n_scen), kThreads, 0, st>>>(n, w, V, col0, N);
  if (ev) cudaEventRecord(ev[3], st);
  k_adj<C><<<dim3(ntile, n_scen), kThreads, 0, st>>>(n, w, N, KV);
  if (ev) cudaEventRecord(ev[4], st);
}

}  // namespace

int pick_tile_cols(int n_x, int total_cols) {
  if (const char* e = getenv("PF_TILE_COLS")) {  // experiments: force 8 / 16 / 32
    const int c = atoi(e);
    if (c == 8 || c == 16 || c == 32) return c;
  }
  // Enough CTAs to fill 148 SMs twice, wide tiles when the work allows.
  if (total_cols >= 32 * 296) return 32;
  if (total_cols >= 16 * 296) return 16;
  return 8;
}

int launch_reduce(const DevNet& n, const Work& w, int C, int n_scen, const double* V, int col0,
                  int N, double* KV, cudaStream_t st, cudaEvent_t* ev) {
  switch (C) {
    case 32: launch_all<32>(n, w, n_scen, V, col0, N, KV, st, ev); break;
    case 16: launch_all<16>(n, w, n_scen, V, col0, N, KV, st, ev); break;
    default: launch_all<8>(n, w, n_scen, V, col0, N, KV, st, ev); break;
  }
  return 4;
}

}  // namespace pf
