// pf_reduce.cu — the batched reduced-Hessian kernels (A7.1–A7.5 of SURVEY §8(a)).
//
// The paper's three steps for K̂V (with R11) over tiles of C
// directions of one scenario:
//   k_fwd  a. B = −P G_u V       (unit V: a column scatter; dense V: a row SpMM)
//          b. Z̃ = U^{-1} L^{-1} B (level-scheduled sweeps over bus blocks)
//   k_mu   c1. μ_A = Σ_r ⊙ R_r M dψ at the r buses (generator buses)
//   k_hvp  c2. [H_u; H_x] = K [V; Z] matrix-free: per bus, the incident lines'
//              precomputed K blocks (H d_loc + Jᵀ μ_A) plus the bus terms
//   k_adj  d. Ψ̃ = L^{-T} U^{-T} H̃_x  (transposed sweeps, same level sets)
//          e. K̂V = H_u − (P G_u)ᵀ Ψ̃  (column gathers, SMEM-transposed store)
// Slabs are [n_x][C] per tile, direction fastest.  A team of W = min(C, 32)
// lanes handles one row; lane l owns the CPL = C / W directions l, l+W, …, so a
// slab row is read as CPL contiguous W×8-byte runs, and every memory round
// trip of the latency-bound sweeps carries CPL directions per lane.
// Every column's arithmetic is independent of N, the tile and the GPU count,
// so K̂ is bit-identical across batch sizes.
#include "pf_launch.h"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace pf {

namespace {

constexpr int kThreads = 256;
constexpr int kCH = 64;        // u-columns per transposed output chunk
#ifndef PF_DOT_W
#define PF_DOT_W 4
#endif
#ifndef PF_SWEEP_MIN_BLOCKS
#define PF_SWEEP_MIN_BLOCKS 3
#endif
constexpr int kSweepMinBlocks = PF_SWEEP_MIN_BLOCKS;  // CTAs per SM the sweep kernels are register-capped for
constexpr int kDotW = PF_DOT_W;                       // entries per row whose slab loads are issued together

template <int C> struct Geo {
  static constexpr int W = C < 32 ? C : 32;  // team width (lanes)
  static constexpr int CPL = C / W;          // directions per lane
  static constexpr int DW = CPL > 1 ? (kDotW + 1) / 2 : kDotW;  // entries per load batch (register budget)
};

__device__ __forceinline__ double2 ldpk(const double2* p) { return __ldg(p); }

// The lanes of this thread's team (W consecutive lanes of the warp): teams of
// one warp follow different rows, so every shuffle names only its own team.
template <int W>
__device__ __forceinline__ unsigned team_mask() {
  if constexpr (W == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31;
    return ((1u << W) - 1u) << (lane & ~(unsigned)(W - 1));
  }
}

// ---------------------------------------------------------------- sweeps
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
// block's slab loads (kDotW entries × 2 rows × CPL directions, all issued
// before the first FMA) are in flight, so a block costs about one round trip.
struct Task { int r0, s0, s1, c0, c1; bool two; };
__device__ __forceinline__ Task unpack(int4 t) {
  Task k;
  k.r0 = t.x & 0x7fffffff; k.two = (t.x >> 31) & 1;
  k.s0 = t.y; k.s1 = t.z; k.c0 = t.w >> 16; k.c1 = t.w & 0xffff;
  return k;
}

__device__ __forceinline__ double2 fetch(const double2* __restrict__ pk, int s, int cnt, int i) {
  return i < cnt ? ldpk(pk + s + i) : make_double2(0.0, 0.0);
}

template <int W>
__device__ __forceinline__ double shv(unsigned mask, double2 q, int e) { return __shfl_sync(mask, q.x, e, W); }

// acc0[j] -= Σ_{k<n0} v0[o0+k] X[c0[o0+k] + lane + W j], acc1 likewise; the
// entries are held one per lane in q0 / q1 (all within one fetch of ≤ W).
// With a reach bitmap bm (SMEM, one bit per slab row), rows outside the reach
// read as 0 (their slab rows were never written).
__device__ __forceinline__ bool in_reach(const unsigned* bm, int colC, int log2C) {
  const int r = colC >> log2C;
  return (bm[r >> 5] >> (r & 31)) & 1u;
}

// Lane l of a team owns the CPL adjacent directions l·CPL … l·CPL + CPL − 1, so a
// gathered row piece is one 16-byte load for CPL = 2.
template <int CPL>
__device__ __forceinline__ void ld_dirs(const double* p, bool ok, double* x) {
  if constexpr (CPL == 2) {
    const double2 v = ok ? *reinterpret_cast<const double2*>(p) : make_double2(0.0, 0.0);
    x[0] = v.x; x[1] = v.y;
  } else {
#pragma unroll
    for (int j = 0; j < CPL; ++j) x[j] = ok ? p[j] : 0.0;
  }
}

template <int C>
__device__ __forceinline__ void dot2(const double* X, unsigned mask, int lane, double2 q0, int o0, int n0,
                                     double2 q1, int o1, int n1, double* acc0, double* acc1,
                                     const unsigned* bm = nullptr) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL, DW = Geo<C>::DW;
  constexpr int L2C = C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
  const int m = max(n0, n1);
  for (int e0 = 0; e0 < m; e0 += DW) {
    double x0[DW][CPL], x1[DW][CPL];
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const int i0 = (o0 + e0 + k) & (W - 1), i1 = (o1 + e0 + k) & (W - 1);
      const int c0 = __shfl_sync(mask, __double2loint(q0.y), i0, W);  // column · C (< 2^31)
      const int c1 = __shfl_sync(mask, __double2loint(q1.y), i1, W);
      const bool ok0 = e0 + k < n0 && (!bm || in_reach(bm, c0, L2C));
      const bool ok1 = e0 + k < n1 && (!bm || in_reach(bm, c1, L2C));
      ld_dirs<CPL>(X + c0 + lane * CPL, ok0, x0[k]);
      ld_dirs<CPL>(X + c1 + lane * CPL, ok1, x1[k]);
    }
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const int i0 = (o0 + e0 + k) & (W - 1), i1 = (o1 + e0 + k) & (W - 1);
      const double v0 = e0 + k < n0 ? __shfl_sync(mask, q0.x, i0, W) : 0.0;
      const double v1 = e0 + k < n1 ? __shfl_sync(mask, q1.x, i1, W) : 0.0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        acc0[j] -= v0 * x0[k][j];
        acc1[j] -= v1 * x1[k][j];
      }
    }
  }
}

// As dot2, with the block's entries in SMEM (e0[i] = entry i of row 0, read as a
// broadcast): no shuffles, and the prefetched entries hold no registers, so a
// whole row's gathers (up to DS per batch) are in flight at once.
#ifndef PF_DOT_S
#define PF_DOT_S 2
#endif
template <int C>
__device__ __forceinline__ void dot2s(const double* X, int lane, const double2* e0, int n0, const double2* e1, int n1,
                                      double* acc0, double* acc1, const unsigned* bm = nullptr) {
  constexpr int CPL = Geo<C>::CPL, DS = PF_DOT_S;
  constexpr int L2C = C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
  const int m = max(n0, n1);
  for (int b = 0; b < m; b += DS) {
    double x0[DS][CPL], x1[DS][CPL];
#pragma unroll
    for (int k = 0; k < DS; ++k) {
      const int c0 = b + k < n0 ? __double2loint(e0[b + k].y) : 0;  // column · C (< 2^31)
      const int c1 = b + k < n1 ? __double2loint(e1[b + k].y) : 0;
      const bool ok0 = b + k < n0 && (!bm || in_reach(bm, c0, L2C));
      const bool ok1 = b + k < n1 && (!bm || in_reach(bm, c1, L2C));
      ld_dirs<CPL>(X + c0 + lane * CPL, ok0, x0[k]);
      ld_dirs<CPL>(X + c1 + lane * CPL, ok1, x1[k]);
    }
#pragma unroll
    for (int k = 0; k < DS; ++k) {
      const double v0 = b + k < n0 ? e0[b + k].x : 0.0;
      const double v1 = b + k < n1 ? e1[b + k].x : 0.0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        acc0[j] -= v0 * x0[k][j];
        acc1[j] -= v1 * x1[k][j];
      }
    }
  }
}

__device__ __forceinline__ void cp_ent(double2* dst, const double2* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

// Rows longer than one fetch (separator rows of the L part): acc[j] -= Σ in
// chunks of W entries, no prefetch.
template <int C>
__device__ __forceinline__ void dot_long(const double2* __restrict__ pk, const double* X, unsigned mask, int lane,
                                         int s, int n, double* acc, const unsigned* bm = nullptr) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL;
  double dummy[CPL];
  for (int base = 0; base < n; base += W) {
    const double2 q = fetch(pk, s + base, n - base, lane);
    dot2<C>(X, mask, lane, q, 0, min(W, n - base), q, 0, 0, acc, dummy, bm);
  }
}

// Initial row values of a sweep: the slab itself, or (first forward sweep) the
// right-hand side B = −P G_u V computed on the fly from G_u's row, so the slab
// needs no zero-fill pass.
struct FromSlab {};
// U sweep after a reach-restricted L sweep: rows outside the reach start at 0
struct FromSlabReach { const unsigned* bm; };
// L sweep after the RHS scatter: rows marked in bm start from the slab, the rest at 0
struct FromSlabMarked { const unsigned* bm; };
template <int C>
struct FromRhs {
  const int* gur_ptr; const int* gur_col; const int* gur_src; const double* gu;
  const double* Vs;  // dense V row of this lane's first direction (the next ones follow at stride n_u), or null = unit
  const double* X4;  // optional extra right-hand side of direction 0 (step recovery, Newton): B −= P X4
  const int* x4map;  //   … X4 entry of permuted row r: X4[x4map[r]]
  int base, nvalid, n_u, lane;  // base = col0 + tile*C: the u column of direction 0 of the tile
  __device__ __forceinline__ void operator()(int r, double* a) const {
    constexpr int CPL = Geo<C>::CPL;
#pragma unroll
    for (int j = 0; j < CPL; ++j) a[j] = 0.0;
    if (X4 && lane == 0) a[0] = -X4[__ldg(x4map + r)];
    for (int e = __ldg(gur_ptr + r); e < __ldg(gur_ptr + r + 1); ++e) {
      const int c = __ldg(gur_col + e);
      if (!Vs && (c < base || c >= base + nvalid)) continue;  // unit directions: only the tile's columns
      const double g = gu[__ldg(gur_src + e)];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int jl = lane * CPL + j;
        if (jl < nvalid) a[j] -= g * (Vs ? Vs[(size_t)j * n_u + c] : (c == base + jl ? 1.0 : 0.0));
      }
    }
  }
};

// One team runs the blocks tasks[first], tasks[first + stride], … < end in
// order (the blocks of one level, or the team's bottom subtrees in postorder).
template <int C, bool LOWER, class Init>
__device__ __forceinline__ void run_seq(const int4* __restrict__ tasks, int first, int end, int stride,
                                        const double2* __restrict__ pk, double* X, bool divide, int lane,
                                        double2* ent, const Init& init, const unsigned* bm) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL;
  const unsigned mask = team_mask<W>();
  auto fits = [](const Task& k) { return k.c0 <= W && k.c1 <= W; };
  auto fill = [&](const Task& k, double2* e) {  // lane-parallel copy of the block's entry ranges
    if (lane < k.c0) cp_ent(e + lane, pk + k.s0 + lane);
    if (k.two && lane < k.c1) cp_ent(e + W + lane, pk + k.s1 + lane);
  };
  int bi = first, buf = 0;
  Task k, nk;
  if (bi < end) {
    k = unpack(__ldg(tasks + bi));
    if (fits(k)) fill(k, ent);
    cp_commit();
    if (bi + stride < end) nk = unpack(__ldg(tasks + bi + stride));
  }
  for (; bi < end; bi += stride) {
    const bool hn = bi + stride < end;
    if (hn && fits(nk)) fill(nk, ent + (buf ^ 1) * 2 * W);  // next block's entries in flight
    cp_commit();
    Task nnk = nk;
    if (bi + 2 * stride < end) nnk = unpack(__ldg(tasks + bi + 2 * stride));
    double* x0p = X + (size_t)k.r0 * C + lane * CPL;
    double* x1p = x0p + C;
    double a0[CPL], a1[CPL];
    if constexpr (std::is_same<Init, FromSlab>::value) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) { a0[j] = x0p[j]; a1[j] = k.two ? x1p[j] : 0.0; }
    } else if constexpr (std::is_same<Init, FromSlabReach>::value || std::is_same<Init, FromSlabMarked>::value) {
      const bool in0 = (init.bm[k.r0 >> 5] >> (k.r0 & 31)) & 1u;
      const bool in1 = k.two && ((init.bm[(k.r0 + 1) >> 5] >> ((k.r0 + 1) & 31)) & 1u);
#pragma unroll
      for (int j = 0; j < CPL; ++j) { a0[j] = in0 ? x0p[j] : 0.0; a1[j] = in1 ? x1p[j] : 0.0; }
    } else {
      init(k.r0, a0);
      if (k.two) {
        init(k.r0 + 1, a1);
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j) a1[j] = 0.0;
      }
    }
    cp_wait<1>();  // this block's entries have landed (this lane's copies) …
    __syncwarp(mask);  // … and every lane's
    const double2* e0 = ent + buf * 2 * W;
    const double2* e1 = e0 + W;
    const bool f = fits(k);
    if (LOWER) {
      const int n0 = k.c0 - 1, n1 = k.two ? k.c1 - 2 : 0;      // entries before diag / intra
      if (f) {
        dot2s<C>(X, lane, e0, n0, e1, n1, a0, a1, bm);
      } else {
        dot_long<C>(pk, X, mask, lane, k.s0, n0, a0, bm);
        if (k.two) dot_long<C>(pk, X, mask, lane, k.s1, n1, a1, bm);
      }
      const double d0 = f ? e0[k.c0 - 1].x : ldpk(pk + k.s0 + k.c0 - 1).x;
      double intra = 0.0, d1 = 1.0;
      if (k.two) {
        intra = f ? e1[k.c1 - 2].x : ldpk(pk + k.s1 + k.c1 - 2).x;
        d1 = f ? e1[k.c1 - 1].x : ldpk(pk + k.s1 + k.c1 - 1).x;
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        double x0 = a0[j];
        if (divide) x0 *= d0;
        x0p[j] = x0;
        if (k.two) {
          double x1 = a1[j] - intra * x0;
          if (divide) x1 *= d1;
          x1p[j] = x1;
        }
      }
    } else {
      // row 1 = [diag, U...], row 0 = [diag, intra?, U...]
      const int o0 = k.two ? 2 : 1;
      const int n0 = k.c0 - o0, n1 = k.two ? k.c1 - 1 : 0;
      if (f) {
        dot2s<C>(X, lane, e0 + o0, n0, e1 + 1, n1, a0, a1);
      } else {
        dot_long<C>(pk, X, mask, lane, k.s0 + o0, n0, a0);
        if (k.two) dot_long<C>(pk, X, mask, lane, k.s1 + 1, n1, a1);
      }
      const double d0 = f ? e0[0].x : ldpk(pk + k.s0).x;
      double intra = 0.0, d1 = 1.0;
      if (k.two) {
        intra = f ? e0[1].x : ldpk(pk + k.s0 + 1).x;
        d1 = f ? e1[0].x : ldpk(pk + k.s1).x;
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        double x1 = 0.0;
        if (k.two) {
          x1 = a1[j];
          if (divide) x1 *= d1;
          x1p[j] = x1;
        }
        double x0 = a0[j] - intra * x1;
        if (divide) x0 *= d0;
        x0p[j] = x0;
      }
    }
    __syncwarp(mask);  // every lane is done with this buffer before it is refilled
    buf ^= 1;
    k = nk;
    nk = nnk;
  }
  cp_wait<0>();
}

// A level-scheduled triangular sweep.  With a phase-1 list (p1, p1ptr) the
// bottom levels < lev0 are run first without barriers, each team walking its
// own bottom subtrees in postorder (every row a LOWER row gathers is a
// descendant, so a subtree is self-contained and its rows are re-read while
// still in L2); the levels ≥ lev0 then run level by level.
template <int C, bool LOWER, class Init = FromSlab>
__device__ __forceinline__ void sweep(const int4* __restrict__ tasks, const int* __restrict__ lptr, int nlev,
                                      const double2* __restrict__ pk, double* X, bool divide, int lane, int team,
                                      int nteam, double2* ent, Init init = Init(), const unsigned* bm = nullptr,
                                      const int4* __restrict__ p1 = nullptr, const int* __restrict__ p1ptr = nullptr,
                                      int lev0 = 0) {
  // LOWER: bottom subtrees (children first), then the levels ≥ lev0.  UPPER: the
  // given (top) levels, then the bottom subtrees (parents first).
  if (LOWER && p1) {
    run_seq<C, LOWER>(p1, __ldg(p1ptr + team), __ldg(p1ptr + team + 1), 1, pk, X, divide, lane, ent, init, bm);
    __syncthreads();
  }
  for (int lev = (LOWER && p1) ? lev0 : 0; lev < nlev; ++lev) {
    run_seq<C, LOWER>(tasks, __ldg(lptr + lev) + team, __ldg(lptr + lev + 1), nteam, pk, X, divide, lane, ent, init, bm);
    __syncthreads();
  }
  if (!LOWER && p1) {
    run_seq<C, LOWER>(p1, __ldg(p1ptr + team), __ldg(p1ptr + team + 1), 1, pk, X, divide, lane, ent, init, bm);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- directions in bus space
// Lane ℓ of a team owns the tile's columns ℓ·CPL … ℓ·CPL+CPL−1 (as in the sweeps),
// so a slab row's directions are one 16-byte access per lane pair of columns.
template <int C>
struct Dir {
  const double* X;   // Z̃ slab of the tile
  const double* Vs;  // dense directions: V[s][tile*C + k][·], column k at Vs + k n_u
  int lane, col, nvalid, n_u;  // col = col0 + tile*C (unit directions); nvalid = directions in the tile
  __device__ __forceinline__ double vdir(int c, int j) const {
    const int k = lane * Geo<C>::CPL + j;
    if (k >= nvalid) return 0.0;
    return Vs ? Vs[(size_t)k * n_u + c] : (c == col + k ? 1.0 : 0.0);
  }
};

template <int C>
__device__ __forceinline__ Dir<C> make_dir(const DevNet& n, const Work& w, const double* V, int col0, int N, int s,
                                           int tile, size_t cta, int lane) {
  Dir<C> d;
  d.lane = lane;
  d.col = col0 + tile * C;
  d.nvalid = min(C, N - tile * C);
  d.n_u = n.n_u;
  d.X = w.slabZ + cta * n.n_x * C;
  d.Vs = V ? V + ((size_t)s * N + tile * C) * n.n_u : nullptr;
  return d;
}

// this lane's CPL columns of row r of a C-wide slab (load / store)
template <int C>
__device__ __forceinline__ void row_ld(const double* S, int r, int lane, double* o) {
  constexpr int CPL = Geo<C>::CPL;
  const double* p = S + (size_t)r * C + lane * CPL;
  if constexpr (CPL == 1) {
    o[0] = *p;
  } else {
#pragma unroll
    for (int q = 0; q < CPL / 2; ++q) {
      const double2 v = reinterpret_cast<const double2*>(p)[q];
      o[2 * q] = v.x; o[2 * q + 1] = v.y;
    }
  }
}
template <int C>
__device__ __forceinline__ void row_st(double* S, int r, int lane, const double* o) {
  constexpr int CPL = Geo<C>::CPL;
  double* p = S + (size_t)r * C + lane * CPL;
  if constexpr (CPL == 1) {
    *p = o[0];
  } else {
#pragma unroll
    for (int q = 0; q < CPL / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(o[2 * q], o[2 * q + 1]);
  }
}

// ---------------------------------------------------------------- a, b
template <int C>
__global__ void __launch_bounds__(kThreads, kSweepMinBlocks) k_fwd(DevNet n, Work w, const double* __restrict__ V, int col0,
                                                                   int N, int rt, const double* __restrict__ X4 = nullptr,
                                                                   const int* __restrict__ x4map = nullptr, int x4ld = 0) {
  constexpr int W = Geo<C>::W;
  extern __shared__ unsigned bm_sm[];  // reach bitmap of this tile (rt ≥ 0)
  __shared__ __align__(16) double2 ent_sm[kThreads / Geo<C>::W][2][2][Geo<C>::W];  // per-team entry buffers
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  const int nvalid = min(C, N - tile * C);
  const int n_x = n.n_x, n_u = n.n_u;
  double* X = w.slabZ + cta * n_x * C;
  const double* gu = w.gu + (size_t)s * n.nnz_gu;
  const double2* pk = w.pkA + (size_t)s * n.nnz_lu;
  double2* ent = &ent_sm[team][0][0][0];
  // A7.1 fused into the first sweep: B = −P G_u V row by row (unit V: G_u's column col0 + j)
  FromRhs<C> rhs;
  rhs.gur_ptr = n.gur_ptr; rhs.gur_col = n.gur_col; rhs.gur_src = n.gur_src; rhs.gu = gu;
  rhs.Vs = V ? V + ((size_t)s * N + tile * C + lane * Geo<C>::CPL) * n_u : nullptr;
  rhs.base = col0 + tile * C; rhs.nvalid = nvalid; rhs.n_u = n_u; rhs.lane = lane;
  rhs.X4 = X4 ? X4 + (size_t)s * x4ld : nullptr; rhs.x4map = x4map;
  if (rt >= 0) {
    // sparse RHS: only the tile's reach (tree paths of its columns' G_u rows) is nonzero
    const unsigned* bmg = n.rowbm + (size_t)(rt + tile) * n.bmw;
    unsigned* rhs_sm = bm_sm + n.bmw;  // rows of B with a nonzero in this tile
    for (int i = threadIdx.x; i < n.bmw; i += blockDim.x) { bm_sm[i] = __ldg(bmg + i); rhs_sm[i] = 0u; }
    __syncthreads();
    // B(r, j) = −G_u(r, base + j) scattered from the tile's G_u columns (off the sweep's
    // latency chain): mark and zero the rows, then drop the entries in
    const int base = col0 + tile * C;
    const int e0 = __ldg(n.guc_ptr + base), e1 = __ldg(n.guc_ptr + base + nvalid);
    for (int e = e0 + team; e < e1; e += nteam) {
      const int r = __ldg(n.guc_row + e);
      if (lane == 0) atomicOr(rhs_sm + (r >> 5), 1u << (r & 31));
      double z[Geo<C>::CPL] = {};
      row_st<C>(X, r, lane, z);
    }
    __syncthreads();
    for (int c = team; c < nvalid; c += nteam)
      for (int e = __ldg(n.guc_ptr + base + c) + lane; e < __ldg(n.guc_ptr + base + c + 1); e += W)
        X[(size_t)__ldg(n.guc_row + e) * C + c] = -gu[__ldg(n.guc_src + e)];
    __syncthreads();
    sweep<C, true>(n.taskLr, n.levLr_ptr + (size_t)(rt + tile) * (n.nlevL + 1), n.nlevL, pk, X, false, lane, team,
                   nteam, ent, FromSlabMarked{rhs_sm}, bm_sm);                                   // L^{-1} B
    sweep<C, false>(n.u_top, n.u_top_ptr, n.nlevU, pk, X, true, lane, team, nteam, ent, FromSlabReach{bm_sm}, nullptr,
                    n.u_bot, n.u_bot_ptr);                                                 // U^{-1}
  } else {
    sweep<C, true>(n.taskL, n.levL_ptr, n.nlevL, pk, X, false, lane, team, nteam, ent, rhs, nullptr, n.p1_task,
                   n.p1_ptr, n.p1_lev0);                                                  // L^{-1} B
    sweep<C, false>(n.u_top, n.u_top_ptr, n.nlevU, pk, X, true, lane, team, nteam, ent, FromSlab(), nullptr, n.u_bot,
                    n.u_bot_ptr);                                                          // U^{-1}
  }
}

// ---------------------------------------------------------------- c1
// μ_A at the generator buses: dG = R_r M dψ = A_r d (the rows P_g, Q_g of J_bus on the bus's
// neighbourhood), μ_A = Σ_r dG (+ 2c₁ dG on P_r0, folded into Σ_rP) — k_blk<C, true> below.

// ---------------------------------------------------------------- c2
// [H_u; H_x] = K [V; Z] as a 2×2 bus-block SpMM: for bus i,
//   (h_θ, h_v)_i = Σ_{j ∈ N(i) ∪ {i}} B_ij (dθ_j, dv_j) + JT_ij (μ^P_j, μ^Q_j)   (JT only at generator buses j)
// with the blocks precomputed per scenario (k_prep_hblk: the line blocks of K, Σ_x, the ψ^d
// curvature and A_rᵀ).  A CTA takes one chunk of consecutive buses of the elimination-forest
// postorder and one direction tile: the chunk's distinct slab rows (own and neighbour buses) are
// pulled into SMEM by cp.async.bulk row copies issued up front (many bytes in flight, no
// registers held), then each team walks its buses reading d from SMEM.
constexpr int kHvpRowCap64 = 80;  // staged rows per chunk at C = 64 (40 KB + the chunk's blocks: 4 CTAs per SM)

__device__ __forceinline__ unsigned sm_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// MU = false: k_hvp (block set n.hb, values w.hbval) writes H_x / H_u rows;
// MU = true:  k_mu  (block set n.mb, values w.mbval) writes μ_A = Σ_r ⊙ dG_r rows at the
//             generator buses (Σ_rP includes the p_ref curvature 2c₁, R8).
template <int C, bool MU>
__global__ void __launch_bounds__(kThreads, 4) k_blk(DevNet n, Work w, const double* __restrict__ V, int col0, int N) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL;
  const BlkSet& B = MU ? n.mb : n.hb;
  // SMEM: [st_max rows][C] staged d / μ rows | [blk_max][8] block values | [blk_max] block meta | [ck_max] output meta
  extern __shared__ __align__(128) double stg[];
  __shared__ __align__(8) uint64_t bar;
  const int ntile = (N + C - 1) / C;
  const int ck = blockIdx.x, tile = blockIdx.y, s = blockIdx.z;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  const double* X = w.slabZ + cta * n.n_x * C;
  double* MU_ = w.mu + cta * n.n_g * 2 * C;
  const int r0 = __ldg(B.st_ptr + ck), nr = __ldg(B.st_ptr + ck + 1) - r0;
  const int p0 = __ldg(B.ck_ptr + ck), p1 = __ldg(B.ck_ptr + ck + 1);
  const int e0 = __ldg(B.ptr + p0), ne = __ldg(B.ptr + p1) - e0;
  double* vals = stg + (size_t)B.st_max * C;                           // [blk_max][8]
  int4* meta = reinterpret_cast<int4*>(vals + (size_t)B.blk_max * 8);  // [blk_max]
  int4* bmeta = meta + B.blk_max;                                      // [ck_max]
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_addr(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    auto bulk = [&](void* dst, const void* src, unsigned bytes) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sm_addr(dst)), "l"(src), "r"(bytes), "r"(sm_addr(&bar)) : "memory");
    };
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(&bar)),
                   "r"((unsigned)(nr * C * 8 + ne * (64 + 16) + (p1 - p0) * 16)) : "memory");
      bulk(vals, (MU ? w.mbval : w.hbval) + ((size_t)s * B.nblk + e0) * 8, ne * 64);
      bulk(meta, B.meta + e0, ne * 16);
      bulk(bmeta, B.out + p0, (p1 - p0) * 16);
    }
    for (int k = threadIdx.x; k < nr; k += 32) {
      const int row = __ldg(B.st_row + r0 + k);
      bulk(stg + (size_t)k * C, row < n.n_x ? X + (size_t)row * C : MU_ + (size_t)(row - n.n_x) * C, C * 8);
    }
  }
  const Dir<C> d = make_dir<C>(n, w, V, col0, N, s, tile, cta, lane);
  double* Y = w.slabW + cta * n.n_x * C;
  double* Hs = w.hu + cta * n.n_u * C;
  const double* bsv = w.bs + (size_t)s * BS_N * n.n_b;
  {
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sm_addr(&bar)) : "memory");
  }
  const double2* vv = reinterpret_cast<const double2*>(vals);
  for (int p = team; p < p1 - p0; p += nteam) {
    const int4 me = bmeta[p];
    double ath[CPL], av[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) { ath[j] = 0.0; av[j] = 0.0; }
    const int eb = __ldg(B.ptr + p0 + p) - e0, ee = __ldg(B.ptr + p0 + p + 1) - e0;
    double th_i[CPL];  // dθ of the bus itself (its block comes first)
    for (int e = eb; e < ee; ++e) {
      const int4 m = meta[e];
      const double2 b0 = vv[4 * e], b1 = vv[4 * e + 1];
      double dth[CPL], dv[CPL];
      if (m.x >= 0) row_ld<C>(stg, m.x, lane, dth);
      else
#pragma unroll
        for (int j = 0; j < CPL; ++j) dth[j] = 0.0;
      if (m.y >= 0) row_ld<C>(stg, m.y, lane, dv);
      else
#pragma unroll
        for (int j = 0; j < CPL; ++j) dv[j] = d.vdir(-1 - m.y, j);
      if (e == eb) {
#pragma unroll
        for (int j = 0; j < CPL; ++j) th_i[j] = dth[j];  // the diagonal θ column is Σ_x (k_hvp) or 0 (k_mu)
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j) dth[j] -= th_i[j];  // θ columns act on angle differences
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {  // explicit FMAs: the same rounding for every tile width (T3)
        ath[j] = fma(b0.y, dv[j], fma(b0.x, dth[j], ath[j]));
        av[j] = fma(b1.y, dv[j], fma(b1.x, dth[j], av[j]));
      }
      if (!MU && m.z >= 0) {  // A_rᵀ μ_A: generator bus j (μ^P, μ^Q rows staged at m.z, m.z + 1)
        const double2 j0 = vv[4 * e + 2], j1 = vv[4 * e + 3];
        double mp[CPL], mq[CPL];
        row_ld<C>(stg, m.z, lane, mp);
        row_ld<C>(stg, m.z + 1, lane, mq);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          ath[j] = fma(j0.y, mq[j], fma(j0.x, mp[j], ath[j]));
          av[j] = fma(j1.y, mq[j], fma(j1.x, mp[j], av[j]));
        }
      }
    }
    if (MU) {  // me = {bus, gen}: μ^P = Σ_rP dP, μ^Q = Σ_rQ dQ
      const double srp = bsv[BS_SRP * n.n_b + me.x], srq = bsv[BS_SRQ * n.n_b + me.x];
#pragma unroll
      for (int j = 0; j < CPL; ++j) { ath[j] *= srp; av[j] *= srq; }
      row_st<C>(MU_, 2 * me.y, lane, ath);
      row_st<C>(MU_, 2 * me.y + 1, lane, av);
    } else {   // me = {bus, θ row, v row or −1−u, gen}
      if (me.y >= 0) row_st<C>(Y, me.y, lane, ath);
      if (me.z >= 0) row_st<C>(Y, me.z, lane, av);
      else row_st<C>(Hs, -1 - me.z, lane, av);
    }
  }
  if (!MU && blockIdx.x == 0)  // objective curvature on explicit p_g
    for (int g = team; g < n.n_g; g += nteam) {
      const int up = __ldg(n.u_p + g);
      if (up >= 0) {
        double o[CPL];
#pragma unroll
        for (int j = 0; j < CPL; ++j) o[j] = 2.0 * __ldg(n.c_quad + g) * d.vdir(up, j);
        row_st<C>(Hs, up, lane, o);
      }
    }
  (void)W;
}

// ---------------------------------------------------------------- d, e
template <int C>
__global__ void __launch_bounds__(kThreads, kSweepMinBlocks) k_adj(DevNet n, Work w, int N, bool full = false) {
  constexpr int W = Geo<C>::W;
  __shared__ __align__(16) double2 sm_adj[(kThreads / W) * 4 * W];  // the sweeps' per-team entry buffers
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  double* Y = w.slabW + cta * n.n_x * C;
  const double2* pk = w.pkT + (size_t)s * n.nnz_lu;
  double2* ent = sm_adj + (size_t)team * 4 * W;
  sweep<C, true>(n.taskL, n.levL_ptr, n.nlevL, pk, Y, true, lane, team, nteam, ent, FromSlab(), nullptr, n.p1_task,
                 n.p1_ptr, n.p1_lev0);                                                  // U^{-T}
  // L^{-T}: only the ancestors of G_u's rows (the projection reads Ψ there), or every row
  // when the whole Ψ is an output (adjoint step / multipliers)
  if (full)
    sweep<C, false>(n.u_top, n.u_top_ptr, n.nlevU, pk, Y, false, lane, team, nteam, ent, FromSlab(), nullptr, n.u_bot,
                    n.u_bot_ptr);
  else
    sweep<C, false>(n.ua_top, n.ua_top_ptr, n.nlevU, pk, Y, false, lane, team, nteam, ent, FromSlab(), nullptr, n.ua_bot,
                    n.ua_bot_ptr);
}

// G_u of each scenario in column (CSC) order, packed {value, row·C} for the projection
__global__ void k_pack_gu(DevNet n, Work w, int n_scen) {
  const long long total = (long long)n_scen * n.nnz_gu;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.nnz_gu), e = (int)(t % n.nnz_gu);
    const double v = w.gu[(size_t)s * n.nnz_gu + __ldg(n.guc_src + e)];
    w.pkG[t] = make_double2(v, __longlong_as_double((long long)__ldg(n.guc_row + e) * n.C));
  }
}

// e. K̂V = H_u − (P G_u)ᵀ Ψ̃ for a chunk of kCH columns of one tile: a column's
// packed G_u entries are fetched lane-parallel (the next column's while this one
// is gathered), its Ψ̃ rows gathered kPG at a time; the chunk is transposed in
// SMEM so every direction's run of kCH outputs is stored contiguously.
template <int C>
__global__ void __launch_bounds__(kThreads) k_proj(DevNet n, Work w, int N, double* __restrict__ KV) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL, kPG = 4;
  __shared__ double T[C][kCH + 1];
  const int ntile = (N + C - 1) / C;
  const int c0 = blockIdx.x * kCH, tile = blockIdx.y, s = blockIdx.z;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  const unsigned mask = team_mask<W>();
  const int n_u = n.n_u;
  const double* Y = w.slabW + cta * n.n_x * C;
  const double* Hs = w.hu + cta * n_u * C;
  const double2* pg = w.pkG + (size_t)s * n.nnz_gu;
  const int cend = min(kCH, n_u - c0);
  int cc = team, e0n = 0, nen = 0;
  double2 qn = make_double2(0.0, 0.0);
  if (cc < cend) {
    e0n = __ldg(n.guc_ptr + c0 + cc); nen = __ldg(n.guc_ptr + c0 + cc + 1) - e0n;
    if (lane < nen) qn = __ldg(pg + e0n + lane);
  }
  for (; cc < cend; cc += nteam) {
    const int c = c0 + cc, e0 = e0n, ne = nen;
    const double2 q = qn;
    if (cc + nteam < cend) {
      e0n = __ldg(n.guc_ptr + c + nteam); nen = __ldg(n.guc_ptr + c + nteam + 1) - e0n;
      qn = lane < nen ? __ldg(pg + e0n + lane) : make_double2(0.0, 0.0);
    }
    double acc[CPL];
    row_ld<C>(Hs, c, lane, acc);
    for (int b = 0; b < ne; b += kPG) {
      double gv[kPG], y[kPG][CPL];
#pragma unroll
      for (int t = 0; t < kPG; ++t) {
        const int ix = (b + t) & (W - 1);
        double2 qe;
        if (ne <= W) {
          qe.x = __shfl_sync(mask, q.x, ix, W);
          qe.y = __shfl_sync(mask, q.y, ix, W);
        } else {
          qe = b + t < ne ? __ldg(pg + e0 + b + t) : make_double2(0.0, 0.0);
        }
        const bool on = b + t < ne;
        gv[t] = on ? qe.x : 0.0;
        const int rowC = __double2loint(qe.y);
        if (on) row_ld<C>(Y + rowC, 0, lane, y[t]);
        else
#pragma unroll
          for (int j = 0; j < CPL; ++j) y[t][j] = 0.0;
      }
#pragma unroll
      for (int t = 0; t < kPG; ++t)
#pragma unroll
        for (int j = 0; j < CPL; ++j) acc[j] -= gv[t] * y[t][j];
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) T[lane * CPL + j][cc] = acc[j];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < C * kCH; idx += blockDim.x) {
    const int jl = idx / kCH, k = idx % kCH;
    const int jj = tile * C + jl;
    if (jj < N && k < cend) KV[((size_t)s * N + jj) * n_u + c0 + k] = T[jl][k];
  }
}

// ---------------------------------------------------------------- NEXT-1 / NEXT-2 single-direction passes
// One direction per scenario: the tile of scenario s is CTA s (ntile = 1) and the
// direction is column 0 of its slabs.  DESIGN.md §"Step recovery" derives the passes:
// with q = [r₁; r₂] + Aᵀ(Σ_s r₅ + r₃) and d = [V; Z], Z = −G_x⁻¹(G_u V + r₄), the HVP
// pipeline runs on H := −(K d + q):
//   condensed rhs   (V = 0):   b = H_u − G_uᵀG_x⁻ᵀH_x  (= −(r̂₁ + Â_uᵀΣ_s r̂₃ + Â_uᵀ r̂₂), R10);
//   recovery (V = p_u):        p_x = Z, p_λ = G_x⁻ᵀH_x, p_s = A[p_u; p_x] + r₅, p_y = Σ_s p_s + r₃;
//   reduced gradient:          H := ∇_z(f + yᵀ[r; h]) = Aᵀỹ + ∂f/∂p_g, λ = −G_x⁻ᵀH_x, ∇f_r = H_u − G_uᵀG_x⁻ᵀH_x.
enum { KV_RHS = 0, KV_GRAD = 1 };

template <int C>
__global__ void k_kkt_vec(DevNet n, Work w, int n_scen, int mode, const double* __restrict__ r,
                          const double* __restrict__ sig_s, const double* __restrict__ y,
                          const double* __restrict__ p_g) {
  const int n_u = n.n_u, n_x = n.n_x, m = n.m, nz = n_u + n_x;
  const size_t ld = 2 * (size_t)n_x + n_u + 2 * (size_t)m;
  const long long total = (long long)n_scen * nz;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / nz), z = (int)(t % nz);
    const double* A = w.aval + (size_t)s * n.nnz_a;
    const double* rs = r ? r + s * ld : nullptr;
    double q = 0.0;
    for (int e = __ldg(n.a_cptr + z); e < __ldg(n.a_cptr + z + 1); ++e) {
      const int k = __ldg(n.a_crow + e);
      double om;
      if (mode == KV_RHS) {
        om = rs[n_u + n_x + k];                                                   // r₃
        if (sig_s) om += sig_s[(size_t)s * m + k] * rs[n_u + n_x + m + n_x + k];  // Σ_s r₅
      } else {
        // ỹ: y, and on row P_r0 (r row 0) the implicit p_ref's (2c₁p_ref + c₂) (R8), which
        // k_prep_bus1 folded into μ̃^P_r0 = y_0 + (2c₁p_ref + c₂) (λ has no P_r0 row)
        om = k == 0 ? w.bs[(size_t)s * BS_N * n.n_b + BS_MUP * n.n_b + n.r0] : y[(size_t)s * m + k];
      }
      q += A[__ldg(n.a_cpos + e)] * om;
    }
    double* H = z < n_u ? w.hu + (size_t)s * n_u * C + (size_t)z * C
                        : w.slabW + (size_t)s * n_x * C + (size_t)__ldg(n.iperm + z - n_u) * C;
    if (mode == KV_RHS) {
      q += rs[z];  // [r₁; r₂]
      *H = -(*H + q);
    } else {
      if (z < n_u) {
        const int g = __ldg(n.u_gen + z);
        if (g >= 0) q += 2.0 * __ldg(n.c_quad + g) * p_g[(size_t)s * n.n_g + g] + __ldg(n.c_lin + g);
      }
      *H = q;
    }
  }
}

// Step recovery output, ordered (p_u, p_x, p_s, p_λ, p_y) like eq. kktmatrix:normal's blocks.
template <int C>
__global__ void k_step_out(DevNet n, Work w, int n_scen, const double* __restrict__ r, const double* __restrict__ sig_s,
                           const double* __restrict__ p_u, double* __restrict__ p) {
  const int n_u = n.n_u, n_x = n.n_x, m = n.m;
  const int ld = 2 * n_x + n_u + 2 * m;
  const long long total = (long long)n_scen * ld;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / ld);
    int k = (int)(t % ld);
    const double* Z = w.slabZ + (size_t)s * n_x * C;
    const double* Y = w.slabW + (size_t)s * n_x * C;
    const double* pu = p_u + (size_t)s * n_u;
    const double* rs = r + (size_t)s * ld;
    double* ps = p + (size_t)s * ld;
    if (k < n_u) { ps[k] = pu[k]; continue; }
    k -= n_u;
    if (k < n_x) { ps[n_u + k] = Z[(size_t)__ldg(n.iperm + k) * C]; continue; }
    k -= n_x;
    if (k < m) {  // p_s = A [p_u; p_x] + r₅ (row 5 of K_aug), p_y = Σ_s p_s + r₃ (row 3)
      double a = rs[n_u + n_x + m + n_x + k];
      const double* A = w.aval + (size_t)s * n.nnz_a;
      for (int e = __ldg(n.a_ptr + k); e < __ldg(n.a_ptr + k + 1); ++e) {
        const int z = __ldg(n.a_idx + e);
        a += A[e] * (z < n_u ? pu[z] : Z[(size_t)__ldg(n.iperm + z - n_u) * C]);
      }
      ps[n_u + n_x + k] = a;
      ps[n_u + n_x + m + n_x + k] = (sig_s ? sig_s[(size_t)s * m + k] : 0.0) * a + rs[n_u + n_x + k];
      continue;
    }
    k -= m;
    if (k < n_x) { ps[n_u + n_x + m + k] = Y[(size_t)__ldg(n.iperm + k) * C]; continue; }
  }
}

// λ = −Ψ (the adjoint step of Algorithm 2: λ = −G_x⁻ᵀ∇_xℒ), x order
template <int C>
__global__ void k_lam_out(DevNet n, Work w, int n_scen, double* __restrict__ lam) {
  const long long total = (long long)n_scen * n.n_x;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_x), x = (int)(t % n.n_x);
    lam[t] = -w.slabW[(size_t)s * n.n_x * C + (size_t)__ldg(n.iperm + x) * C];
  }
}

// Newton: x += Z (Z = −G_x⁻¹ g) for the scenarios still iterating
template <int C>
__global__ void k_pf_update(DevNet n, Work w, int n_scen, double* __restrict__ v, double* __restrict__ th) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    if (!w.active[s]) continue;
    const double* Z = w.slabZ + (size_t)s * n.n_x * C;
    const int pt = __ldg(n.bus_pth + i), pv = __ldg(n.bus_pv + i);
    if (pt >= 0) th[t] += Z[(size_t)pt * C];
    if (pv >= 0) v[t] += Z[(size_t)pv * C];
  }
}

inline int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>(148LL * 16, (n + kThreads - 1) / kThreads)); }

template <int C, bool MU>
size_t blk_smem(const DevNet& n) {
  const BlkSet& B = MU ? n.mb : n.hb;
  const size_t b = (size_t)B.st_max * C * sizeof(double) + (size_t)B.blk_max * 80 + (size_t)B.ck_max * 16;
  // per device and function, so set on every launch (a host-side call, graph-capture safe)
  cudaFuncSetAttribute(k_blk<C, MU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
  return b;
}

template <int C>
void one_dir_fwd_hvp(const DevNet& n, const Work& w, int n_scen, const double* V, const double* X4, const int* map,
                     int x4ld, bool hvp, cudaStream_t st) {
  k_fwd<C><<<dim3(1, n_scen), kThreads, 0, st>>>(n, w, V, 0, 1, -1, X4, map, x4ld);
  if (!hvp) return;
  k_blk<C, true><<<dim3(n.mb.nchunk, 1, n_scen), kThreads, blk_smem<C, true>(n), st>>>(n, w, V, 0, 1);
  k_blk<C, false><<<dim3(n.hb.nchunk, 1, n_scen), kThreads, blk_smem<C, false>(n), st>>>(n, w, V, 0, 1);
}

template <int C>
int step_all(int what, const DevNet& n, const Work& w, int n_scen, const double* r, const double* sig_s,
             const double* y, const double* p_g, const double* p_u, double* out, double* out2, cudaStream_t st) {
  const int ld = 2 * n.n_x + n.n_u + 2 * n.m;
  const int nz = n.n_u + n.n_x;
  int launches = 0;
  if (what == 0 || what == 2) {  // the projection needs G_u packed by columns
    k_pack_gu<<<(int)std::min<long long>(4096, ((long long)n_scen * n.nnz_gu + kThreads - 1) / kThreads), kThreads, 0,
                st>>>(n, w, n_scen);
    ++launches;
  }
  if (what == 0 || what == 1) {  // condensed rhs / recovery: forward pass with r₄, K·d
    one_dir_fwd_hvp<C>(n, w, n_scen, what == 0 ? w.zero : p_u, r + n.n_u + n.n_x + n.m, n.perm, ld, true, st);
    k_kkt_vec<C><<<grid_for((long long)n_scen * nz), kThreads, 0, st>>>(n, w, n_scen, KV_RHS, r, sig_s, nullptr, nullptr);
    k_adj<C><<<dim3(1, n_scen), kThreads, 0, st>>>(n, w, 1, what == 1);
    launches += 6;
  } else {  // reduced gradient
    k_kkt_vec<C><<<grid_for((long long)n_scen * nz), kThreads, 0, st>>>(n, w, n_scen, KV_GRAD, nullptr, nullptr, y, p_g);
    k_adj<C><<<dim3(1, n_scen), kThreads, 0, st>>>(n, w, 1, true);
    launches += 2;
  }
  if (what == 0 || what == 2) {
    k_proj<C><<<dim3((n.n_u + kCH - 1) / kCH, 1, n_scen), kThreads, 0, st>>>(n, w, 1, out);
    ++launches;
  }
  if (what == 1) {
    k_step_out<C><<<grid_for((long long)n_scen * ld), kThreads, 0, st>>>(n, w, n_scen, r, sig_s, p_u, out);
    ++launches;
  }
  if (what == 2 && out2) {
    k_lam_out<C><<<grid_for((long long)n_scen * n.n_x), kThreads, 0, st>>>(n, w, n_scen, out2);
    ++launches;
  }
  return launches;
}

template <int C>
int newton_step(const DevNet& n, const Work& w, int n_scen, double* v, double* th, cudaStream_t st) {
  one_dir_fwd_hvp<C>(n, w, n_scen, w.zero, w.gbuf, n.row_g, 2 * n.n_b, false, st);  // Z = −G_x⁻¹ g
  k_pf_update<C><<<grid_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen, v, th);
  return 2;
}

template <int C>
void launch_all(const DevNet& n, const Work& w, int n_scen, const double* V, int col0, int N, double* KV,
                cudaStream_t st, cudaEvent_t* ev) {
  const int ntile = (N + C - 1) / C;
  k_pack_gu<<<(int)std::min<long long>(4096, ((long long)n_scen * n.nnz_gu + kThreads - 1) / kThreads), kThreads, 0,
              st>>>(n, w, n_scen);
  if (ev) cudaEventRecord(ev[0], st);
  const int rt = (V == nullptr && col0 % C == 0) ? col0 / C : -1;  // canonical tile of the call's first tile
  k_fwd<C><<<dim3(ntile, n_scen), kThreads, rt >= 0 ? 2 * n.bmw * sizeof(unsigned) : 0, st>>>(n, w, V, col0, N, rt);
  if (ev) cudaEventRecord(ev[1], st);
  k_blk<C, true><<<dim3(n.mb.nchunk, ntile, n_scen), kThreads, blk_smem<C, true>(n), st>>>(n, w, V, col0, N);
  if (ev) cudaEventRecord(ev[2], st);
  k_blk<C, false><<<dim3(n.hb.nchunk, ntile, n_scen), kThreads, blk_smem<C, false>(n), st>>>(n, w, V, col0, N);
  if (ev) cudaEventRecord(ev[3], st);
  k_adj<C><<<dim3(ntile, n_scen), kThreads, 0, st>>>(n, w, N);
  if (ev) cudaEventRecord(ev[4], st);
  k_proj<C><<<dim3((n.n_u + kCH - 1) / kCH, ntile, n_scen), kThreads, 0, st>>>(n, w, N, KV);
  if (ev) cudaEventRecord(ev[7], st);
}

}  // namespace

int hvp_stage_rows(int C) {
  // 48 KB of staged rows per CTA at C = 64 (4 CTAs per SM); narrower tiles stage more rows of
  // fewer bytes (capped at the same byte budget, at most 4 × the buses of a chunk)
  return std::min(256, kHvpRowCap64 * 64 / C);
}

int pick_tile_cols(int n_x, int total_cols) {
  (void)n_x;
  // Wide tiles carry more directions per memory round trip of the latency-
  // bound sweeps; narrow ones keep ≥ 2 CTAs per SM when the work is small.
  if (total_cols >= 64 * 296) return 64;
  if (total_cols >= 32 * 296) return 32;
  if (total_cols >= 16 * 296) return 16;
  return 8;
}

// ‖g‖∞ over the x rows of G (w.gbuf) per scenario
__global__ void k_pf_resid(DevNet n, Work w, int n_scen) {
  __shared__ double red[kThreads / 32];
  const int s = blockIdx.x;
  double mx = 0.0;
  for (int r = threadIdx.x; r < n.n_x; r += blockDim.x) {
    const double g = w.gbuf[(size_t)s * 2 * n.n_b + __ldg(n.row_g + r)];
    mx = (g != g) ? g : fmax(mx, fabs(g));  // NaN propagates
  }
  for (int o = 16; o > 0; o >>= 1) { const double t = __shfl_xor_sync(0xffffffffu, mx, o); mx = (t != t) ? t : fmax(mx, t); }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) a = (red[k] != red[k]) ? red[k] : fmax(a, red[k]);
    w.res[s] = a;
  }
}

int launch_step(int what, const DevNet& n, const Work& w, int C, int n_scen, const double* r, const double* sig_s,
                const double* y, const double* p_g, const double* p_u, double* out, double* out2, cudaStream_t st) {
  switch (C) {
    case 64: return step_all<64>(what, n, w, n_scen, r, sig_s, y, p_g, p_u, out, out2, st);
    case 32: return step_all<32>(what, n, w, n_scen, r, sig_s, y, p_g, p_u, out, out2, st);
    case 16: return step_all<16>(what, n, w, n_scen, r, sig_s, y, p_g, p_u, out, out2, st);
    default: return step_all<8>(what, n, w, n_scen, r, sig_s, y, p_g, p_u, out, out2, st);
  }
}

int launch_pf_resid(const DevNet& n, const Work& w, int n_scen, cudaStream_t st) {
  k_pf_resid<<<n_scen, kThreads, 0, st>>>(n, w, n_scen);
  return 1;
}

int launch_newton_step(const DevNet& n, const Work& w, int C, int n_scen, double* v, double* th, cudaStream_t st) {
  switch (C) {
    case 64: return newton_step<64>(n, w, n_scen, v, th, st);
    case 32: return newton_step<32>(n, w, n_scen, v, th, st);
    case 16: return newton_step<16>(n, w, n_scen, v, th, st);
    default: return newton_step<8>(n, w, n_scen, v, th, st);
  }
}

int launch_reduce(const DevNet& n, const Work& w, int C, int n_scen, const double* V, int col0,
                  int N, double* KV, cudaStream_t st, cudaEvent_t* ev) {
  switch (C) {
    case 64: launch_all<64>(n, w, n_scen, V, col0, N, KV, st, ev); break;
    case 32: launch_all<32>(n, w, n_scen, V, col0, N, KV, st, ev); break;
    case 16: launch_all<16>(n, w, n_scen, V, col0, N, KV, st, ev); break;
    default: launch_all<8>(n, w, n_scen, V, col0, N, KV, st, ev); break;
  }
  return 6;
}

}  // namespace pf
