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
#ifndef PF_BLK_SPIN_NS
#define PF_BLK_SPIN_NS 64
#endif
#ifndef PF_BLK_PF_DIST
#define PF_BLK_PF_DIST 296
#endif
#ifndef PF_INIT_PF
#define PF_INIT_PF 1  // sweeps from the slab: L2 prefetch of the initial rows PF_INIT_DIST blocks ahead
#endif
#ifndef PF_PROJ_PF
#define PF_PROJ_PF 1
#endif
#ifndef PF_SEG_PF
#define PF_SEG_PF 1
#endif
#ifndef PF_INIT_DIST
#define PF_INIT_DIST 3
#endif
#ifndef PF_SWEEP_MIN_BLOCKS
#define PF_SWEEP_MIN_BLOCKS 3
#endif
constexpr int kSweepMinBlocks = PF_SWEEP_MIN_BLOCKS;  // CTAs per SM the sweep kernels are register-capped for

template <int C> struct Geo {
  static constexpr int W = C < 32 ? C : 32;  // team width (lanes)
  static constexpr int CPL = C / W;          // directions per lane
};

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
// A level-scheduled triangular sweep over bus blocks (1–2 rows each), driven by
// per-level task lists built on the host (pf_api.cu): task {r0 | two << 31, s, m, 0}
// names the block's segment of a sweep stream (w.swA for L / U, w.swT for Uᵀ / Lᵀ):
//   [row A gathers, m][row B gathers, m (two-row blocks)][{d_A, intra}, {d_B, 0}]
// of packed {value, column·C} gathers.  Row A is solved first (LOWER — the L and Uᵀ
// sweeps — the θ row r0; UPPER — U and Lᵀ — the v row r0 + 1); row B depends on it
// only through the intra entry.  m is even and short rows are padded with zero-valued
// entries that read a row the block gathers anyway, so the inner loop carries no
// bounds predicates: per step it issues the slab loads of two entries of each row,
// then their FMAs, about six instructions per entry.  A segment is copied
// lane-parallel into the team's SMEM buffer one block ahead (cp.async); the rare
// segments longer than the buffer are read from global memory.
struct Task { int r0, s, m; bool two; };
__device__ __forceinline__ Task unpack(int4 t) {
  Task k;
  k.r0 = t.x & 0x7fffffff; k.two = (t.x >> 31) & 1; k.s = t.y; k.m = t.z;
  return k;
}
template <int W> struct Seg { static constexpr int CAP = 2 * W + 2; };  // entries of a buffered segment

// With a reach bitmap bm (SMEM, one bit per slab row), rows outside the reach
// read as 0 (their slab rows were never written).
__device__ __forceinline__ bool in_reach(const unsigned* bm, unsigned colC, int log2C) {
  const unsigned r = colC >> log2C;
  return (bm[r >> 5] >> (r & 31)) & 1u;
}

__device__ __forceinline__ void cp_ent(double2* dst, const double2* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

// base + c doubles as one IMAD.WIDE.U32 (the compiler otherwise rebuilds a 64-bit
// index from lane·CPL + c and scales it: four instructions per gathered entry)
__device__ __forceinline__ const double* off8(const double* base, unsigned c) {
  const double* r;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(r) : "r"(c), "l"(base));
  return r;
}

// Lane l of a team owns the CPL adjacent directions l·CPL … l·CPL + CPL − 1, so a
// gathered row piece is one 16-byte load for CPL = 2.
template <int C, bool REACH>
__device__ __forceinline__ void gather(const double* Xl, double2 q, const unsigned* bm, double* x) {
  constexpr int CPL = Geo<C>::CPL;
  constexpr int L2C = C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
  const unsigned c = (unsigned)__double2loint(q.y);  // column · C (< 2^31)
  if (REACH && !in_reach(bm, c, L2C)) {
#pragma unroll
    for (int j = 0; j < CPL; ++j) x[j] = 0.0;
    return;
  }
  const double* p = off8(Xl, c);
  if constexpr (CPL == 2) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    x[0] = v.x; x[1] = v.y;
  } else {
    x[0] = *p;
  }
}

// Segment entry i: its column·C (the low word of .y) and its value, read separately so
// a gather in flight holds only its data registers.  G: the segment is in global memory.
template <bool G>
__device__ __forceinline__ unsigned ent_col(const double2* e, int i) {
  const int* p = reinterpret_cast<const int*>(e) + 4 * i + 2;
  return (unsigned)(G ? __ldg(p) : *p);
}
template <bool G>
__device__ __forceinline__ double ent_val(const double2* e, int i) {
  const double* p = reinterpret_cast<const double*>(e) + 2 * i;
  return G ? __ldg(p) : *p;
}

template <int C, bool REACH>
__device__ __forceinline__ void gather_c(const double* Xl, unsigned c, const unsigned* bm, double* x) {
  gather<C, REACH>(Xl, make_double2(0.0, __hiloint2double(0, (int)c)), bm, x);
}

// accA[j] −= Σ_{i<m} v_i · X[column_i + lane·CPL + j] over the entries e[0, m) in order, and
// for two-row blocks accB likewise over the values of e[m, 2m), whose columns are those of
// e[0, m) (m even).  Four entries per step: all their slab loads are issued before the first
// FMA (one memory round trip per step).
template <int C, bool REACH, bool G>
__device__ __forceinline__ void dot_seg(const double2* e, int m, bool two, const double* Xl, const unsigned* bm,
                                        double* accA, double* accB) {
  constexpr int CPL = Geo<C>::CPL;
  int i = 0;
  if (two) {
    // both rows list the same columns (pf_api.cu segment): one gather feeds both rows
#pragma unroll 1
    for (; i + 4 <= m; i += 4) {
      double x[4][CPL];
#pragma unroll
      for (int k = 0; k < 4; ++k) gather_c<C, REACH>(Xl, ent_col<G>(e, i + k), bm, x[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double va = ent_val<G>(e, i + k), vb = ent_val<G>(e, m + i + k);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          accA[j] -= va * x[k][j];
          accB[j] -= vb * x[k][j];
        }
      }
    }
    if (i < m) {  // m is even: one pair left
      double x[2][CPL];
#pragma unroll
      for (int k = 0; k < 2; ++k) gather_c<C, REACH>(Xl, ent_col<G>(e, i + k), bm, x[k]);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double va = ent_val<G>(e, i + k), vb = ent_val<G>(e, m + i + k);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          accA[j] -= va * x[k][j];
          accB[j] -= vb * x[k][j];
        }
      }
    }
  } else {
#pragma unroll 1
    for (; i < m; i += 2) {
      double xa[2][CPL];
#pragma unroll
      for (int k = 0; k < 2; ++k) gather_c<C, REACH>(Xl, ent_col<G>(e, i + k), bm, xa[k]);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double va = ent_val<G>(e, i + k);
#pragma unroll
        for (int j = 0; j < CPL; ++j) accA[j] -= va * xa[k][j];
      }
    }
  }
}

template <int CPL>
__device__ __forceinline__ void st_dirs(double* p, const double* x) {
  if constexpr (CPL == 2) *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
  else *p = x[0];
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
template <int C, bool LOWER, bool REACH, class Init>
__device__ __forceinline__ void run_seq(const int4* __restrict__ tasks, int first, int end, int stride,
                                        const double2* __restrict__ sv, double* X, bool divide, int lane,
                                        double2* ent, const Init& init, const unsigned* bm) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL, CAP = Seg<W>::CAP;
  const unsigned mask = team_mask<W>();
  auto len = [](const Task& k) { return k.m * (1 + k.two) + 2; };
  auto fill = [&](const Task& k, double2* e) {  // lane-parallel copy of the block's segment
    const int n = len(k);
    if (n <= CAP)
      for (int i = lane; i < n; i += W) cp_ent(e + i, sv + k.s + i);
  };
  const double* Xl = X + lane * CPL;
  int bi = first, buf = 0;
  Task k, nk;
  if (bi < end) {
    k = unpack(__ldg(tasks + bi));
    fill(k, ent);
    cp_commit();
    if (bi + stride < end) nk = unpack(__ldg(tasks + bi + stride));
  }
  for (; bi < end; bi += stride) {
    if (bi + stride < end) fill(nk, ent + (buf ^ 1) * CAP);  // next block's segment in flight
    cp_commit();
    Task nnk = nk;
    if (bi + 2 * stride < end) nnk = unpack(__ldg(tasks + bi + 2 * stride));
#if PF_INIT_PF
    // sweeps that start from the slab (k_adj: H_x written by k_hvp, mostly in DRAM): the initial
    // rows of the block PF_INIT_DIST ahead — off the dependency chain — are prefetched into L2
    // once its task has arrived, at the end of this block (k_adj 3.17 → 2.80 ms); the other
    // sweeps start from rows their previous sweep just wrote (L2-hot) and gain nothing
    const bool pf3 = std::is_same<Init, FromSlab>::value && bi + PF_INIT_DIST * stride < end;
    // k_fwd's sweeps (not from the slab): the segment of the block PF_INIT_DIST ahead instead
    // (k_fwd 1.89 → 1.86 ms; in k_adj it costs more than it saves)
    const bool pfs = PF_SEG_PF && !std::is_same<Init, FromSlab>::value && bi + PF_INIT_DIST * stride < end;
    const int4 t3 = (pf3 || pfs) ? __ldg(tasks + bi + PF_INIT_DIST * stride) : make_int4(0, 0, 0, 0);
#endif
    const int rA = k.r0 + (!LOWER && k.two), rB = k.r0 + (LOWER ? 1 : 0);
    double* xa = X + (size_t)rA * C + lane * CPL;
    double* xb = X + (size_t)rB * C + lane * CPL;
    double aA[CPL], aB[CPL];
    if constexpr (std::is_same<Init, FromSlab>::value) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) { aA[j] = xa[j]; aB[j] = k.two ? xb[j] : 0.0; }
    } else if constexpr (std::is_same<Init, FromSlabReach>::value || std::is_same<Init, FromSlabMarked>::value) {
      const bool inA = (init.bm[rA >> 5] >> (rA & 31)) & 1u;
      const bool inB = k.two && ((init.bm[rB >> 5] >> (rB & 31)) & 1u);
#pragma unroll
      for (int j = 0; j < CPL; ++j) { aA[j] = inA ? xa[j] : 0.0; aB[j] = inB ? xb[j] : 0.0; }
    } else {
      init(rA, aA);
      if (k.two) {
        init(rB, aB);
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j) aB[j] = 0.0;
      }
    }
    cp_wait<1>();      // this block's segment has landed (this lane's copies) …
    __syncwarp(mask);  // … and every lane's
    const int n = len(k);
    double2 sc0, sc1;  // {d_A, intra}, {d_B, 0}
    if (n <= CAP) {
      const double2* es = ent + buf * CAP;
      dot_seg<C, REACH, false>(es, k.m, k.two, Xl, bm, aA, aB);
      sc0 = es[n - 2]; sc1 = es[n - 1];
    } else {
      const double2* eg = sv + k.s;
      dot_seg<C, REACH, true>(eg, k.m, k.two, Xl, bm, aA, aB);
      sc0 = __ldg(eg + n - 2); sc1 = __ldg(eg + n - 1);
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      if (divide) aA[j] *= sc0.x;
      aB[j] -= sc0.y * aA[j];
      if (divide) aB[j] *= sc1.x;
    }
    st_dirs<CPL>(xa, aA);
    if (k.two) st_dirs<CPL>(xb, aB);
#if PF_INIT_PF
    if (pf3) {
      constexpr int NL = C * 8 / 128 > 0 ? C * 8 / 128 : 1;  // 128-byte lines of a slab row
      const Task k3 = unpack(t3);
      const int r = (lane < NL) ? k3.r0 + (!LOWER && k3.two) : k3.r0 + (LOWER ? 1 : 0);
      if (lane < NL || (k3.two && lane < 2 * NL)) {
        const char* pr = reinterpret_cast<const char*>(X + (size_t)r * C) + (lane % NL) * 128;
        if (PF_INIT_PF == 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(pr));
        else asm volatile("prefetch.global.L2 [%0];" ::"l"(pr));
      }
    }
    if (pfs) {  // … and that block's segment (the stream lines the cp.async copy will read)
      const Task k3 = unpack(t3);
      const char* b = reinterpret_cast<const char*>(sv + k3.s);
      const char* e = reinterpret_cast<const char*>(sv + k3.s + len(k3));
      const char* pl = reinterpret_cast<const char*>(reinterpret_cast<size_t>(b) & ~(size_t)127) + lane * 128;
      if (pl < e) asm volatile("prefetch.global.L2 [%0];" ::"l"(pl));
    }
#endif
    __syncwarp(mask);  // every lane is done with this buffer before it is refilled
    buf ^= 1;
    k = nk;
    nk = nnk;
  }
  cp_wait<0>();
}

#ifdef PF_SWEEP_TRACE
__device__ unsigned long long* g_sw_trace;  // tools/sweep_trace.py: [sweep slot][512] globaltimer stamps of CTA (0, 0)
__device__ __forceinline__ void sw_stamp(int tr, int ev) {
  if (tr >= 0 && g_sw_trace && blockIdx.x == 0 && blockIdx.y == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sw_trace[tr * 512 + ev] = t;
  }
}
#define SW_STAMP(ev) sw_stamp(tr, ev)
#else
#define SW_STAMP(ev) (void)0
#endif

template <int C, bool LOWER, bool REACH = false, class Init = FromSlab>
__device__ __forceinline__ void sweep(const int4* __restrict__ tasks, const int* __restrict__ lptr, int nlev,
                                      const double2* __restrict__ pk, double* X, bool divide, int lane, int team,
                                      int nteam, double2* ent, Init init = Init(), const unsigned* bm = nullptr,
                                      const int4* __restrict__ p1 = nullptr, const int* __restrict__ p1ptr = nullptr,
                                      int lev0 = 0, int tr = -1) {
  (void)tr;
  if (threadIdx.x == 0) SW_STAMP(0);
  // LOWER: bottom subtrees (children first), then the levels ≥ lev0.  UPPER: the
  // given (top) levels, then the bottom subtrees (parents first).
  if (LOWER && p1) {
    run_seq<C, LOWER, REACH>(p1, __ldg(p1ptr + team), __ldg(p1ptr + team + 1), 1, pk, X, divide, lane, ent, init, bm);
    if (lane == 0) SW_STAMP(1 + team);
    __syncthreads();
  }
  for (int lev = (LOWER && p1) ? lev0 : 0; lev < nlev; ++lev) {
    run_seq<C, LOWER, REACH>(tasks, __ldg(lptr + lev) + team, __ldg(lptr + lev + 1), nteam, pk, X, divide, lane, ent, init, bm);
    __syncthreads();
    if (threadIdx.x == 0) SW_STAMP(64 + lev);
  }
  if (!LOWER && p1) {
    run_seq<C, LOWER, REACH>(p1, __ldg(p1ptr + team), __ldg(p1ptr + team + 1), 1, pk, X, divide, lane, ent, init, bm);
    if (lane == 0) SW_STAMP(1 + team);
    __syncthreads();
  }
  if (threadIdx.x == 0) SW_STAMP(511);
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
// RT: unit directions from canonical tile rt (sparse right-hand sides, reach-restricted L sweep);
// otherwise dense V (or V = 0 with the extra right-hand side X4) and full sweeps.
template <int C, bool RT>
__global__ void __launch_bounds__(kThreads, kSweepMinBlocks) k_fwd(DevNet n, Work w, const double* __restrict__ V, int col0,
                                                                   int N, int rt, const double* __restrict__ X4 = nullptr,
                                                                   const int* __restrict__ x4map = nullptr, int x4ld = 0) {
  constexpr int W = Geo<C>::W;
  extern __shared__ unsigned bm_sm[];  // reach bitmap of this tile (rt ≥ 0)
  __shared__ __align__(16) double2 ent_sm[kThreads / Geo<C>::W][2][Seg<Geo<C>::W>::CAP];  // per-team segment buffers
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  const int nvalid = min(C, N - tile * C);
  const int n_x = n.n_x, n_u = n.n_u;
  double* X = w.slabZ + cta * n_x * C;
  const double* gu = w.gu + (size_t)s * n.nnz_gu;
  const double2* pk = w.swA + (size_t)s * n.nsw;
  double2* ent = &ent_sm[team][0][0];
  if constexpr (RT) {
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
    sweep<C, true, true>(n.taskLr, n.levLr_ptr + (size_t)(rt + tile) * (n.nlevL + 1), n.nlevL, pk, X, false, lane, team,
                         nteam, ent, FromSlabMarked{rhs_sm}, bm_sm, n.p1r_task,
                         n.p1r_ptr + (size_t)(rt + tile) * (nteam + 1), n.p1_lev0, 0);                                   // L^{-1} B
    sweep<C, false>(n.u_top, n.u_top_ptr, n.nlevU, pk, X, true, lane, team, nteam, ent, FromSlabReach{bm_sm}, nullptr,
                    n.u_bot, n.u_bot_ptr, 0, 1);                                                 // U^{-1}
  } else {
    // A7.1 fused into the first sweep: B = −P G_u V row by row (unit V: G_u's column col0 + j)
    FromRhs<C> rhs;
    rhs.gur_ptr = n.gur_ptr; rhs.gur_col = n.gur_col; rhs.gur_src = n.gur_src; rhs.gu = gu;
    rhs.Vs = V ? V + ((size_t)s * N + tile * C + lane * Geo<C>::CPL) * n_u : nullptr;
    rhs.base = col0 + tile * C; rhs.nvalid = nvalid; rhs.n_u = n_u; rhs.lane = lane;
    rhs.X4 = X4 ? X4 + (size_t)s * x4ld : nullptr; rhs.x4map = x4map;
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
#if PF_BLK_PF_DIST > 0
  else if (threadIdx.x < 64) {
    // L2 prefetch of the rows a CTA about one resident wave later will stage (no SMEM held):
    // more DRAM bytes in flight than the staged chunks alone allow
    const long long lin = ((long long)s * ntile + tile) * gridDim.x + ck + PF_BLK_PF_DIST;
    if (lin < (long long)gridDim.x * ntile * gridDim.z) {
      const int ck2 = (int)(lin % gridDim.x);
      const long long c2 = lin / gridDim.x;  // s2 * ntile + tile2
      const double* X2 = w.slabZ + (size_t)c2 * n.n_x * C;
      const double* M2 = w.mu + (size_t)c2 * n.n_g * 2 * C;
      const int q0 = __ldg(B.st_ptr + ck2), nq = __ldg(B.st_ptr + ck2 + 1) - q0;
      for (int k = threadIdx.x - 32; k < nq; k += 32) {
        const int row = __ldg(B.st_row + q0 + k);
        const double* src = row < n.n_x ? X2 + (size_t)row * C : M2 + (size_t)(row - n.n_x) * C;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((unsigned)(C * 8)) : "memory");
      }
    }
  }
#endif
  const Dir<C> d = make_dir<C>(n, w, V, col0, N, s, tile, cta, lane);
  double* Y = w.slabW + cta * n.n_x * C;
  double* Hs = w.hu + cta * n.n_u * C;
  const double* bsv = w.bs + (size_t)s * BS_N * n.n_b;
  {
    // back off between polls: the co-resident CTAs' computing warps keep the issue slots
    unsigned done = 0;
    for (;;) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sm_addr(&bar)) : "memory");
      if (done) break;
      __nanosleep(PF_BLK_SPIN_NS);
    }
  }
  const double2* vv = reinterpret_cast<const double2*>(vals);
  const double* myrow = stg + lane * CPL;  // this lane's columns of staged row 0
  for (int p = team; p < p1 - p0; p += nteam) {
    const int4 me = bmeta[p];
    double ath[CPL], av[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) { ath[j] = 0.0; av[j] = 0.0; }
    const int eb = __ldg(B.ptr + p0 + p) - e0, ee = __ldg(B.ptr + p0 + p + 1) - e0;
    auto rld = [&](int slot, double* o) {
      if constexpr (CPL == 2) {
        const double2 v = *reinterpret_cast<const double2*>(myrow + (size_t)slot * C);
        o[0] = v.x; o[1] = v.y;
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j) o[j] = myrow[(size_t)slot * C + j];
      }
    };
    auto jt = [&](int e, const int4& m) {  // A_rᵀ μ_A: generator bus j (μ^P, μ^Q rows staged at m.z, m.z + 1)
      if (!MU && m.z >= 0) {
        const double2 j0 = vv[4 * e + 2], j1 = vv[4 * e + 3];
        double mp[CPL], mq[CPL];
        rld(m.z, mp);
        rld(m.z + 1, mq);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          ath[j] = fma(j0.y, mq[j], fma(j0.x, mp[j], ath[j]));
          av[j] = fma(j1.y, mq[j], fma(j1.x, mp[j], av[j]));
        }
      }
    };
    double th_i[CPL];  // dθ of the bus itself: its own block comes first, its θ column is Σ_x (k_hvp) or 0 (k_mu)
    {
      const int4 m = meta[eb];
      const double2 b0 = vv[4 * eb], b1 = vv[4 * eb + 1];
      double dv[CPL];
      if (m.x >= 0) rld(m.x, th_i);
      else
#pragma unroll
        for (int j = 0; j < CPL; ++j) th_i[j] = 0.0;
      if (m.y >= 0) rld(m.y, dv);
      else
#pragma unroll
        for (int j = 0; j < CPL; ++j) dv[j] = d.vdir(-1 - m.y, j);
#pragma unroll
      for (int j = 0; j < CPL; ++j) {  // explicit FMAs: the same rounding for every tile width (T3)
        ath[j] = fma(b0.y, dv[j], fma(b0.x, th_i[j], ath[j]));
        av[j] = fma(b1.y, dv[j], fma(b1.x, th_i[j], av[j]));
      }
      jt(eb, m);
    }
    for (int e = eb + 1; e < ee; ++e) {  // neighbours: θ columns act on angle differences dθ_j − dθ_i
      const int4 m = meta[e];
      const double2 b0 = vv[4 * e], b1 = vv[4 * e + 1];
      double dth[CPL], dv[CPL];
      if (m.x >= 0) {
        rld(m.x, dth);
#pragma unroll
        for (int j = 0; j < CPL; ++j) dth[j] -= th_i[j];
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j) dth[j] = 0.0 - th_i[j];
      }
      if (m.y >= 0) rld(m.y, dv);
      else
#pragma unroll
        for (int j = 0; j < CPL; ++j) dv[j] = d.vdir(-1 - m.y, j);
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        ath[j] = fma(b0.y, dv[j], fma(b0.x, dth[j], ath[j]));
        av[j] = fma(b1.y, dv[j], fma(b1.x, dth[j], av[j]));
      }
      jt(e, m);
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
  __shared__ __align__(16) double2 sm_adj[(kThreads / W) * 2 * Seg<W>::CAP];  // the sweeps' per-team segment buffers
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % W, team = threadIdx.x / W, nteam = blockDim.x / W;
  double* Y = w.slabW + cta * n.n_x * C;
  const double2* pk = w.swT + (size_t)s * n.nsw;
  double2* ent = sm_adj + (size_t)team * 2 * Seg<W>::CAP;
  sweep<C, true>(n.taskL, n.levL_ptr, n.nlevL, pk, Y, true, lane, team, nteam, ent, FromSlab(), nullptr, n.p1_task,
                 n.p1_ptr, n.p1_lev0, 2);                                                 // U^{-T}
  // L^{-T}: only the ancestors of G_u's rows (the projection reads Ψ there), or every row
  // when the whole Ψ is an output (adjoint step / multipliers)
  if (full)
    sweep<C, false>(n.u_top, n.u_top_ptr, n.nlevU, pk, Y, false, lane, team, nteam, ent, FromSlab(), nullptr, n.u_bot,
                    n.u_bot_ptr);
  else
    sweep<C, false>(n.ua_top, n.ua_top_ptr, n.nlevU, pk, Y, false, lane, team, nteam, ent, FromSlab(), nullptr, n.ua_bot,
                    n.ua_bot_ptr, 0, 3);
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
// SMEM (T) so every direction's run of kCH outputs is stored contiguously.
template <int C>
__device__ __forceinline__ void proj_chunk(const DevNet& n, const Work& w, int N, double* __restrict__ KV, int c0,
                                           int tile, int s, size_t cta, double (*T)[kCH + 1]) {
  constexpr int W = Geo<C>::W, CPL = Geo<C>::CPL, kPG = 4;
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
#if PF_PROJ_PF
      // the next column's Ψ rows and H_u row into L2 while this column is gathered (k_adj and
      // k_hvp wrote them; they come from DRAM)
      constexpr int NL = C * 8 / 128 > 0 ? C * 8 / 128 : 1;
      if (lane < nen && lane < W)
        for (int l = 0; l < NL; ++l)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(Y + __double2loint(qn.y)) + l * 128));
      if (lane < NL)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(Hs + (size_t)(c + nteam) * C) + lane * 128));
#endif
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
  __syncthreads();  // T is reused by the next chunk
}

template <int C>
__global__ void __launch_bounds__(kThreads) k_proj(DevNet n, Work w, int N, double* __restrict__ KV) {
  __shared__ double T[C][kCH + 1];
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.y, s = blockIdx.z;
  proj_chunk<C>(n, w, N, KV, blockIdx.x * kCH, tile, s, (size_t)s * ntile + tile, T);
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

// ---------------------------------------------------------------- single-direction solves in SMEM
// The NEXT passes (condensed rhs, step recovery, reduced gradient, Newton) solve with ONE
// direction per scenario: the tile layout above would run each sweep's ~1,150 blocks per team
// as a chain of global-memory round trips on one CTA.  Here the whole permuted vector (n_x
// doubles) lives in SMEM and every level of the full level schedule (taskL / taskU) runs
// across the CTA's 1024 threads: a block is taken by a team of TW lanes (TW from the
// level's width: one warp per block on the narrow top levels, one lane per block on the
// wide bottom ones), the lanes split its segment's gathers (read from the same sweep
// streams as the tiled sweeps; columns are SMEM indices) and reduce by shuffles, and lane 0
// finishes the block (row A, then row B through the intra entry).  One __syncthreads per level.
constexpr int kTri1Threads = 1024;

template <int TW>
__device__ __forceinline__ void tri1_level(const int4* __restrict__ tasks, int b0, int b1,
                                           const double2* __restrict__ sv, double* xs, bool divide, bool lower,
                                           int shift) {
  const int lane = threadIdx.x & (TW - 1), team = threadIdx.x / TW, nteam = kTri1Threads / TW;
  const unsigned mask = TW == 32 ? 0xffffffffu : (((1u << TW) - 1u) << ((threadIdx.x & 31) & ~(TW - 1)));
  for (int bi = b0 + team; bi < b1; bi += nteam) {
    const Task k = unpack(__ldg(tasks + bi));
    const double2* e = sv + k.s;
    const int n = k.m * (1 + k.two) + 2;
    double2 sc0 = make_double2(0.0, 0.0), sc1 = sc0;
    if (lane == 0) { sc0 = __ldg(e + n - 2); sc1 = __ldg(e + n - 1); }  // in flight with the gathers
    double sA = 0.0, sB = 0.0;
    if (k.two) {
#pragma unroll 2
      for (int i = lane; i < k.m; i += TW) {
        const double2 qa = __ldg(e + i), qb = __ldg(e + k.m + i);
        sA = fma(qa.x, xs[(unsigned)__double2loint(qa.y) >> shift], sA);
        sB = fma(qb.x, xs[(unsigned)__double2loint(qb.y) >> shift], sB);
      }
    } else {
#pragma unroll 4
      for (int i = lane; i < k.m; i += TW) {
        const double2 qa = __ldg(e + i);
        sA = fma(qa.x, xs[(unsigned)__double2loint(qa.y) >> shift], sA);
      }
    }
#pragma unroll
    for (int o = TW / 2; o > 0; o >>= 1) {
      sA += __shfl_xor_sync(mask, sA, o, TW);
      sB += __shfl_xor_sync(mask, sB, o, TW);
    }
    if (lane == 0) {
      const int rA = k.r0 + (!lower && k.two), rB = k.r0 + (lower ? 1 : 0);
      double a = xs[rA] - sA;
      if (divide) a *= sc0.x;
      xs[rA] = a;
      if (k.two) {
        double b = xs[rB] - sB - sc0.y * a;
        if (divide) b *= sc1.x;
        xs[rB] = b;
      }
    }
  }
}

__device__ __forceinline__ void tri1_sweep(const int4* __restrict__ tasks, const int* __restrict__ lptr, int nlev,
                                           const double2* __restrict__ sv, double* xs, bool divide, bool lower,
                                           int shift) {
  for (int lev = 0; lev < nlev; ++lev) {
    const int b0 = __ldg(lptr + lev), b1 = __ldg(lptr + lev + 1), nb = b1 - b0;
    // the next level's tasks and segments do not depend on x: thread t loads task t of the next
    // level now and, once this level is done, prefetches its segment into L1, so the next level
    // starts from L1 instead of two dependent L2 round trips
    int4 nxt = make_int4(0, 0, -1, 0);
    if (lev + 1 < nlev) {
      const int c0 = __ldg(lptr + lev + 1);
      if (c0 + (int)threadIdx.x < __ldg(lptr + lev + 2)) nxt = __ldg(tasks + c0 + threadIdx.x);
    }
    if (nb * 32 <= kTri1Threads) tri1_level<32>(tasks, b0, b1, sv, xs, divide, lower, shift);
    else if (nb * 8 <= kTri1Threads) tri1_level<8>(tasks, b0, b1, sv, xs, divide, lower, shift);
    else if (nb * 2 <= kTri1Threads) tri1_level<2>(tasks, b0, b1, sv, xs, divide, lower, shift);
    else tri1_level<1>(tasks, b0, b1, sv, xs, divide, lower, shift);
    if (nxt.z >= 0) {
      const Task k = unpack(nxt);
      const char* p = reinterpret_cast<const char*>(sv + k.s);
      const int bytes = (k.m * (1 + k.two) + 2) * 16;
      for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + o));
    }
    __syncthreads();
  }
}

// mode 0 (forward): Z = −G_x⁻¹ P (G_u V + X4) → slabZ column 0 (the right-hand side as FromRhs
// builds it); mode 1 (adjoint): Ψ = G_x⁻ᵀ (slabW column 0) in place, Lᵀ over every row (full)
// or over the ancestors of G_u's rows.  One CTA per scenario.
template <int C>
__global__ void __launch_bounds__(kTri1Threads) k_tri1(DevNet n, Work w, int mode, bool full,
                                                         const double* __restrict__ V,
                                                         const double* __restrict__ X4,
                                                         const int* __restrict__ x4map, int x4ld) {
  extern __shared__ double xs[];
  constexpr int shift = C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
  const int s = blockIdx.x, n_x = n.n_x;
  if (mode == 0) {
    double* X = w.slabZ + (size_t)s * n_x * C;
    const double* gu = w.gu + (size_t)s * n.nnz_gu;
    const double* Vs = V + (size_t)s * n.n_u;
    const double* X4s = X4 ? X4 + (size_t)s * x4ld : nullptr;
    for (int r = threadIdx.x; r < n_x; r += blockDim.x) {
      double a = X4s ? -X4s[__ldg(x4map + r)] : 0.0;
      for (int e = __ldg(n.gur_ptr + r); e < __ldg(n.gur_ptr + r + 1); ++e)
        a -= gu[__ldg(n.gur_src + e)] * Vs[__ldg(n.gur_col + e)];
      xs[r] = a;
    }
    __syncthreads();
    const double2* pk = w.swA + (size_t)s * n.nsw;
    tri1_sweep(n.taskL, n.levL_ptr, n.nlevL, pk, xs, false, true, shift);   // L⁻¹
    tri1_sweep(n.taskU, n.levU_ptr, n.nlevU, pk, xs, true, false, shift);   // U⁻¹
    for (int r = threadIdx.x; r < n_x; r += blockDim.x) X[(size_t)r * C] = xs[r];
  } else {
    double* Y = w.slabW + (size_t)s * n_x * C;
    for (int r = threadIdx.x; r < n_x; r += blockDim.x) xs[r] = Y[(size_t)r * C];
    __syncthreads();
    const double2* pk = w.swT + (size_t)s * n.nsw;
    tri1_sweep(n.taskL, n.levL_ptr, n.nlevL, pk, xs, true, true, shift);    // U⁻ᵀ
    if (full) tri1_sweep(n.taskU, n.levU_ptr, n.nlevU, pk, xs, false, false, shift);   // L⁻ᵀ
    else tri1_sweep(n.taskUa, n.levUa_ptr, n.nlevU, pk, xs, false, false, shift);
    for (int r = threadIdx.x; r < n_x; r += blockDim.x) Y[(size_t)r * C] = xs[r];
  }
}

// whether the vector fits the SMEM of one CTA (else the tiled sweeps run the pass)
inline bool tri1_fits(const DevNet& n) { return (size_t)n.n_x * sizeof(double) <= 200 * 1024; }

template <int C>
void tri1_launch(const DevNet& n, const Work& w, int n_scen, int mode, bool full, const double* V, const double* X4,
                 const int* map, int x4ld, cudaStream_t st) {
  const int smem = (int)((size_t)n.n_x * sizeof(double));
  cudaFuncSetAttribute(k_tri1<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  // per device: every launch
  k_tri1<C><<<n_scen, kTri1Threads, smem, st>>>(n, w, mode, full, V, X4, map, x4ld);
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
  if (tri1_fits(n)) tri1_launch<C>(n, w, n_scen, 0, true, V, X4, map, x4ld, st);
  else k_fwd<C, false><<<dim3(1, n_scen), kThreads, 0, st>>>(n, w, V, 0, 1, -1, X4, map, x4ld);
  if (!hvp) return;
  k_blk<C, true><<<dim3(n.mb.nchunk, 1, n_scen), kThreads, blk_smem<C, true>(n), st>>>(n, w, V, 0, 1);
  k_blk<C, false><<<dim3(n.hb.nchunk, 1, n_scen), kThreads, blk_smem<C, false>(n), st>>>(n, w, V, 0, 1);
}

template <int C>
void one_dir_adj(const DevNet& n, const Work& w, int n_scen, bool full, cudaStream_t st) {
  if (tri1_fits(n)) tri1_launch<C>(n, w, n_scen, 1, full, nullptr, nullptr, nullptr, 0, st);
  else k_adj<C><<<dim3(1, n_scen), kThreads, 0, st>>>(n, w, 1, full);
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
    one_dir_adj<C>(n, w, n_scen, what == 1, st);
    launches += 6;
  } else {  // reduced gradient
    k_kkt_vec<C><<<grid_for((long long)n_scen * nz), kThreads, 0, st>>>(n, w, n_scen, KV_GRAD, nullptr, nullptr, y, p_g);
    one_dir_adj<C>(n, w, n_scen, true, st);
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
                cudaStream_t st, cudaEvent_t* ev, cudaEvent_t after_fwd) {
  const int ntile = (N + C - 1) / C;
  k_pack_gu<<<(int)std::min<long long>(4096, ((long long)n_scen * n.nnz_gu + kThreads - 1) / kThreads), kThreads, 0,
              st>>>(n, w, n_scen);
  if (ev) cudaEventRecord(ev[0], st);
  const int rt = (V == nullptr && col0 % C == 0) ? col0 / C : -1;  // canonical tile of the call's first tile
#ifdef PF_SWEEP_CARVEOUT  // experiment: SMEM carve-out of the sweep kernels (L1 size)
  cudaFuncSetAttribute(k_fwd<C, true>, cudaFuncAttributePreferredSharedMemoryCarveout, PF_SWEEP_CARVEOUT);
  cudaFuncSetAttribute(k_fwd<C, false>, cudaFuncAttributePreferredSharedMemoryCarveout, PF_SWEEP_CARVEOUT);
  cudaFuncSetAttribute(k_adj<C>, cudaFuncAttributePreferredSharedMemoryCarveout, PF_SWEEP_CARVEOUT);
#endif
  if (rt >= 0) k_fwd<C, true><<<dim3(ntile, n_scen), kThreads, 2 * n.bmw * sizeof(unsigned), st>>>(n, w, V, col0, N, rt);
  else k_fwd<C, false><<<dim3(ntile, n_scen), kThreads, 0, st>>>(n, w, V, col0, N, rt);
  if (ev) cudaEventRecord(ev[1], st);
  if (after_fwd) cudaStreamWaitEvent(st, after_fwd, 0);
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

#ifdef PF_SWEEP_TRACE
void set_sweep_trace(unsigned long long* p) { cudaMemcpyToSymbol(g_sw_trace, &p, sizeof(p)); }
#endif

int launch_reduce(const DevNet& n, const Work& w, int C, int n_scen, const double* V, int col0,
                  int N, double* KV, cudaStream_t st, cudaEvent_t* ev, cudaEvent_t after_fwd) {
  switch (C) {
    case 64: launch_all<64>(n, w, n_scen, V, col0, N, KV, st, ev, after_fwd); break;
    case 32: launch_all<32>(n, w, n_scen, V, col0, N, KV, st, ev, after_fwd); break;
    case 16: launch_all<16>(n, w, n_scen, V, col0, N, KV, st, ev, after_fwd); break;
    default: launch_all<8>(n, w, n_scen, V, col0, N, KV, st, ev, after_fwd); break;
  }
  return 6;
}

}  // namespace pf
