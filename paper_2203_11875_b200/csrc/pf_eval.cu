// pf_eval.cu — ψ-basis evaluation (A2/A3), ψ-chain Jacobians (A4), the
// level-scheduled numeric LU refactorization of G_x (A5) and the per-scenario
// ψ weights of the Hessian-vector product (A6).  sm_100a, FP64.
//
// Readings: R1 conj in s_f, R2/R3 L_line blocks, R4 M entries,
// R5 ψ orientation Δ = θ_f − θ_t, R8 implicit p_ref, R18 static pivots.
#include "pf_launch.h"

#include <algorithm>
#include <climits>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace pf {

namespace {

constexpr int kThreads = 256;

inline int blocks_for(long long n, int t = kThreads) {
  long long b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > 148LL * 64) b = 148LL * 64;
  return (int)b;
}

struct LineCoef { double gff, bff, gft, bft, gtf, btf, gtt, btt; };

__device__ __forceinline__ LineCoef load_coef(const DevNet& n, int l) {
  LineCoef c;
  c.gff = __ldg(n.coef + 0 * n.n_l + l); c.bff = __ldg(n.coef + 1 * n.n_l + l);
  c.gft = __ldg(n.coef + 2 * n.n_l + l); c.bft = __ldg(n.coef + 3 * n.n_l + l);
  c.gtf = __ldg(n.coef + 4 * n.n_l + l); c.btf = __ldg(n.coef + 5 * n.n_l + l);
  c.gtt = __ldg(n.coef + 6 * n.n_l + l); c.btt = __ldg(n.coef + 7 * n.n_l + l);
  return c;
}

// ψ^c = v_f v_t cos Δ, ψ^s = v_f v_t sin Δ (R5), and the line-local
// L_line products (eq. base:powerlines P:L128–154 with R1–R3).
struct Flows { double c, s, pc, ps, spf, sqf, spt, sqt; };

__device__ __forceinline__ Flows line_flows(const LineCoef& k, double vf, double vt, double thf, double tht) {
  Flows o;
  sincos(thf - tht, &o.s, &o.c);
  const double vv = vf * vt;
  o.pc = vv * o.c;
  o.ps = vv * o.s;
  o.spf = k.gft * o.pc + k.bft * o.ps + k.gff * vf * vf;
  o.sqf = -k.bft * o.pc + k.gft * o.ps - k.bff * vf * vf;
  o.spt = k.gtf * o.pc - k.btf * o.ps + k.gtt * vt * vt;
  o.sqt = -k.btf * o.pc - k.gtf * o.ps - k.btt * vt * vt;
  return o;
}

// ---------------------------------------------------------------- A2/A3
__global__ void k_line_eval(DevNet n, Work w, int n_scen, const double* __restrict__ v,
                            const double* __restrict__ th, double* __restrict__ H,
                            double* __restrict__ s_out) {
  const long long total = (long long)n_scen * n.n_l;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_l), l = (int)(t % n.n_l);
    const int f = __ldg(n.lf + l), to = __ldg(n.lt + l);
    const double* vs = v + (size_t)s * n.n_b;
    const double* ts = th + (size_t)s * n.n_b;
    Flows o = line_flows(load_coef(n, l), vs[f], vs[to], ts[f], ts[to]);
    double* sf = w.sflow + (size_t)s * 4 * n.n_l;
    sf[l] = o.spf; sf[n.n_l + l] = o.sqf; sf[2 * n.n_l + l] = o.spt; sf[3 * n.n_l + l] = o.sqt;
    if (s_out) {
      double* so = s_out + (size_t)s * 4 * n.n_l;
      so[l] = o.spf; so[n.n_l + l] = o.sqf; so[2 * n.n_l + l] = o.spt; so[3 * n.n_l + l] = o.sqt;
    }
    if (H) {  // eq. linelimitsvec
      double* hs = H + (size_t)s * 2 * n.n_l;
      hs[l] = o.spf * o.spf + o.sqf * o.sqf;
      hs[n.n_l + l] = o.spt * o.spt + o.sqt * o.sqt;
    }
  }
}

// G = Mψ + [p_d − C_g p_g ; q_d − C_g q_g] (eq. base:powerflow P:L109–125).
// Row P_i of M gathers the line ends incident to i (R4) plus G_ii ψ^d_i;
// G_ii's Y_ff / Y_tt parts already sit in s_p^f / s_p^t, the shunt remains.
__global__ void k_bus_eval(DevNet n, Work w, int n_scen, const double* __restrict__ v,
                           const double* __restrict__ p_g, const double* __restrict__ q_g,
                           const double* __restrict__ p_d, const double* __restrict__ q_d,
                           double* __restrict__ G) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    const double* sf = w.sflow + (size_t)s * 4 * n.n_l;
    double P = 0.0, Q = 0.0;
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int l = __ldg(n.inc_line + e);
      const bool from = __ldg(n.lf + l) == i;
      P += from ? sf[l] : sf[2 * n.n_l + l];
      Q += from ? sf[n.n_l + l] : sf[3 * n.n_l + l];
    }
    const double vi = v[(size_t)s * n.n_b + i];
    P += __ldg(n.gsh + i) * vi * vi;
    Q -= __ldg(n.bsh + i) * vi * vi;
    const int g = __ldg(n.bus_gen + i);
    if (g >= 0) { P -= p_g[(size_t)s * n.n_g + g]; Q -= q_g[(size_t)s * n.n_g + g]; }
    P += p_d ? p_d[(size_t)s * n.n_b + i] : __ldg(n.p_d0 + i);
    Q += q_d ? q_d[(size_t)s * n.n_b + i] : __ldg(n.q_d0 + i);
    G[(size_t)s * 2 * n.n_b + i] = P;
    G[(size_t)s * 2 * n.n_b + n.n_b + i] = Q;
  }
}

// ---------------------------------------------------------------- A4
__global__ void k_line_state(DevNet n, Work w, int n_scen, const double* __restrict__ v,
                             const double* __restrict__ th) {
  const long long total = (long long)n_scen * n.n_l;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_l), l = (int)(t % n.n_l);
    const int f = __ldg(n.lf + l), to = __ldg(n.lt + l);
    const double vf = v[(size_t)s * n.n_b + f], vt = v[(size_t)s * n.n_b + to];
    Flows o = line_flows(load_coef(n, l), vf, vt, th[(size_t)s * n.n_b + f], th[(size_t)s * n.n_b + to]);
    double* ls = w.ls + (size_t)s * LS_N * n.n_l;
    ls[LS_VF * n.n_l + l] = vf; ls[LS_VT * n.n_l + l] = vt;
    ls[LS_C * n.n_l + l] = o.c; ls[LS_S * n.n_l + l] = o.s;
    ls[LS_SPF * n.n_l + l] = o.spf; ls[LS_SQF * n.n_l + l] = o.sqf;
    ls[LS_SPT * n.n_l + l] = o.spt; ls[LS_SQT * n.n_l + l] = o.sqt;
  }
}

// ∂(s_p, s_q) of one line end w.r.t. the local variables (v_f, v_t, θ_f, θ_t):
// J_ψ rows ∂ψ^c = (v_t c, v_f c, −ψ^s, ψ^s), ∂ψ^s = (v_t s, v_f s, ψ^c, −ψ^c),
// composed with the L_line coefficients.
struct EndGrad { double p[4], q[4]; };

__device__ __forceinline__ EndGrad end_grad(const LineCoef& k, double vf, double vt, double c, double s, bool from) {
  const double pc = vf * vt * c, ps = vf * vt * s;
  const double dc[4] = {vt * c, vf * c, -ps, ps};
  const double ds[4] = {vt * s, vf * s, pc, -pc};
  EndGrad g;
  if (from) {
#pragma unroll
    for (int a = 0; a < 4; ++a) { g.p[a] = k.gft * dc[a] + k.bft * ds[a]; g.q[a] = -k.bft * dc[a] + k.gft * ds[a]; }
    g.p[0] += 2.0 * k.gff * vf; g.q[0] -= 2.0 * k.bff * vf;
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) { g.p[a] = k.gtf * dc[a] - k.btf * ds[a]; g.q[a] = -k.btf * dc[a] - k.gtf * ds[a]; }
    g.p[1] += 2.0 * k.gtt * vt; g.q[1] -= 2.0 * k.btt * vt;
  }
  return g;
}

// J_bus rows P_i, Q_i: one thread per (scenario, bus), ascending incident
// lines (parallel lines accumulate into the same entries, deterministically).
__global__ void k_jbus(DevNet n, Work w, int n_scen) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    double* jb = w.jb + (size_t)s * n.nnz_jb;
    const double* ls = w.ls + (size_t)s * LS_N * n.n_l;
    double* rp = jb + __ldg(n.jb_ptr + i);
    double* rq = jb + __ldg(n.jb_ptr + n.n_b + i);
    const int len = __ldg(n.jb_ptr + i + 1) - __ldg(n.jb_ptr + i);
    for (int a = 0; a < len; ++a) { rp[a] = 0.0; rq[a] = 0.0; }
    double pv = 0, pth = 0, qv = 0, qth = 0;
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int l = __ldg(n.inc_line + e);
      const bool from = __ldg(n.lf + l) == i;
      EndGrad g = end_grad(load_coef(n, l), ls[LS_VF * n.n_l + l], ls[LS_VT * n.n_l + l],
                           ls[LS_C * n.n_l + l], ls[LS_S * n.n_l + l], from);
      const int own_v = from ? 0 : 1, oth_v = from ? 1 : 0, own_t = from ? 2 : 3, oth_t = from ? 3 : 2;
      pv += g.p[own_v]; qv += g.q[own_v]; pth += g.p[own_t]; qth += g.q[own_t];
      const int ov = __ldg(n.inc_off_v + e), ot = __ldg(n.inc_off_th + e);
      rp[ov] += g.p[oth_v]; rq[ov] += g.q[oth_v];
      if (ot >= 0) { rp[ot] += g.p[oth_t]; rq[ot] += g.q[oth_t]; }
    }
    const int sv = __ldg(n.jb_self_v + i), st = __ldg(n.jb_self_th + i);
    // shunt part of G_ii ψ^d_i (R4): ∂/∂v_i of g_sh v_i², −b_sh v_i²
    const double vb = w.bs[(size_t)s * BS_N * n.n_b + BS_V * n.n_b + i];
    pv += 2.0 * __ldg(n.gsh + i) * vb;
    qv -= 2.0 * __ldg(n.bsh + i) * vb;
    rp[sv] += pv; rq[sv] += qv;
    if (st >= 0) { rp[st] += pth; rq[st] += qth; }
  }
}

__global__ void k_bus_v(DevNet n, Work w, int n_scen, const double* __restrict__ v) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    w.bs[(size_t)s * BS_N * n.n_b + BS_V * n.n_b + i] = v[(size_t)s * n.n_b + i];
  }
}

// Gathers J_bus values into the G_x / G_u / A patterns; h rows of A from the
// line ends: ∇H = 2(s_p ∇s_p + s_q ∇s_q).
__global__ void k_gather(DevNet n, Work w, int n_scen, double* __restrict__ Gx,
                         double* __restrict__ Gu, double* __restrict__ A) {
  const int per = n.nnz_gx + n.nnz_gu + n.nnz_a;
  const long long total = (long long)n_scen * per;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / per);
    int k = (int)(t % per);
    const double* jb = w.jb + (size_t)s * n.nnz_jb;
    if (k < n.nnz_gx) {
      if (Gx) Gx[(size_t)s * n.nnz_gx + k] = jb[__ldg(n.gx_src + k)];
      continue;
    }
    k -= n.nnz_gx;
    if (k < n.nnz_gu) {
      const int src = __ldg(n.gu_src + k);
      const double val = src >= 0 ? jb[src] : -1.0;  // −C_g p_g entry (eq. powerflowvec)
      w.gu[(size_t)s * n.nnz_gu + k] = val;
      if (Gu) Gu[(size_t)s * n.nnz_gu + k] = val;
      continue;
    }
    k -= n.nnz_gu;
    double* Aw = w.aval + (size_t)s * n.nnz_a;  // kept for the step recovery / reduced gradient
    const int src = __ldg(n.a_src + k);
    if (src >= 0) {
      Aw[k] = jb[src];
      if (A) A[(size_t)s * n.nnz_a + k] = jb[src];
      continue;
    }
    // h row owning position k: binary search in a_ptr over rows [n_r, m)
    int lo = n.n_r, hi = n.m - 1;
    while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (__ldg(n.a_ptr + mid) <= k) lo = mid; else hi = mid - 1; }
    const int h = lo - n.n_r, base = __ldg(n.a_ptr + lo);
    const int l = __ldg(n.h_line + h), e = __ldg(n.h_end + h);
    const double* ls = w.ls + (size_t)s * LS_N * n.n_l;
    EndGrad g = end_grad(load_coef(n, l), ls[LS_VF * n.n_l + l], ls[LS_VT * n.n_l + l],
                         ls[LS_C * n.n_l + l], ls[LS_S * n.n_l + l], e == 0);
    const double sp = e == 0 ? ls[LS_SPF * n.n_l + l] : ls[LS_SPT * n.n_l + l];
    const double sq = e == 0 ? ls[LS_SQF * n.n_l + l] : ls[LS_SQT * n.n_l + l];
    for (int a = 0; a < 4; ++a)
      if (__ldg(n.ah_off + 4 * h + a) == k - base) {
        const double val = 2.0 * (sp * g.p[a] + sq * g.q[a]);
        Aw[k] = val;
        if (A) A[(size_t)s * n.nnz_a + k] = val;
      }
  }
}

// ---------------------------------------------------------------- A5
// Numeric LU of P G_x Pᵀ with the fixed symbolic pattern and static pivots
// (R18): up-looking IKJ rows, one warp per bus block (the row kept in a SMEM
// workspace, the pivot rows' U parts and update targets prefetched one step
// ahead), the blocks of one level spread over all warps of the scenario's
// thread-block CLUSTER; a cluster barrier (≈0.2 µs, no grid-wide sync)
// separates levels.  One cluster per scenario, so scenarios run independently.
// Values written by other SMs of the cluster are read with ld.global.cg (L2).
constexpr int kLuThreads = 512;
constexpr int kLuStageMin = 8;    // rows with at least this many pivots stage their working set
constexpr int kLuMaxPiv = 128;    // … and at most this many
constexpr int kLuStageCap = 768;  // update entries staged per warp
constexpr int kLuStageWarps = 6;  // warps of a CTA with a staging area

// A warp's staging area for one long LU row: per pivot a its 1/u_kk and the
// offset of its update list; the lists' values (pivot U row) and targets.
struct LuStage {
  double* pin;  // [kLuMaxPiv]
  double* val;  // [kLuStageCap]
  int* off;     // [kLuMaxPiv + 1]
  int* dst;     // [kLuStageCap]
};
constexpr size_t kLuStageBytes = (size_t)kLuMaxPiv * 8 + kLuStageCap * 8 + (kLuMaxPiv + 2) * 4 + kLuStageCap * 4;

// Lane-parallel gather of row (base, dl)'s IKJ working set.  The row's update lists are one
// contiguous run of upd_dst / upd_src (entries e = base … base + dl − 1 in order), so the
// pivot offsets come straight from upd_ptr and every update entry is an independent pair of
// loads (its target offset, and the U value at upd_src; __ldcg: written by other SMs of the
// cluster), 4 in flight per lane.  False (nothing staged) when the lists exceed the area.
__device__ bool stage_row(const DevNet& n, const double* lu, const double* invd, int base, int dl, int lane,
                          const LuStage& st) {
  const int q0 = __ldg(n.upd_ptr + base), total = __ldg(n.upd_ptr + base + dl) - q0;
  if (total > kLuStageCap) return false;
  for (int a = lane; a <= dl; a += 32) {
    st.off[a] = __ldg(n.upd_ptr + base + a) - q0;
    if (a < dl) st.pin[a] = __ldcg(invd + __ldg(n.lu_idx + base + a));
  }
  for (int i0 = 0; i0 < total; i0 += 128) {
    double v[4];
    int dd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = i0 + 32 * q + lane;
      if (idx < total) {
        v[q] = __ldcg(lu + __ldg(n.upd_src + q0 + idx));
        dd[q] = __ldg(n.upd_dst + q0 + idx);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = i0 + 32 * q + lane;
      if (idx < total) { st.val[idx] = v[q]; st.dst[idx] = dd[q]; }
    }
  }
  __syncwarp();
  return true;
}

#ifdef PF_LU_TRACE
__device__ unsigned long long* g_lu_trace;  // tools/lu_trace.py: globaltimer after each level (cluster 0)
#define LU_PH(lev, ph)                                                                              \
  do {                                                                                              \
    if (blockIdx.x == 0 && warp == 0 && lane == 0 && g_lu_trace) {                                  \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      g_lu_trace[1024 + 8 * (lev) + (ph)] = t_;                                                     \
    }                                                                                               \
  } while (0)
#else
#define LU_PH(lev, ph) (void)0
#endif

// The dense front of one scenario's LU (levels ≥ fr_lev, after their cluster.sync).
// (a) Every front row applies its pivots outside the front — rows of lower levels, final —
//     in ascending order (a front pivot never precedes a non-front one it updates: U(k', k) ≠ 0
//     makes k depend on k', so a front k' forces k into the front), one warp per row over the
//     cluster.  (b) CTA 0 gathers the front Schur complement S (F × F, F ≤ kFrontMax) into SMEM
//     and eliminates it densely in pivot order — l = s_ik · (1 / s_kk), s_ij −= l s_kj, the same
//     operations the row-wise IKJ applies — with two CTA barriers per pivot instead of one
//     cluster barrier per level; the pattern entries go back to lu, 1 / u_rr to invd, and the
//     R18 pivot test to info.
__device__ void lu_front(const DevNet& n, double* lu, double* invd, const double* rowmax, int* info, double* smem,
                         int sub, int CS, cg::cluster_group& cluster) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5, F = n.fr_n;
  double* ws = smem + warp * n.lu_maxlen;
  for (int f = warp * CS + sub; f < F; f += CS * nwarp) {
    const int r = __ldg(n.fr_row + f), base = __ldg(n.lu_ptr + r), len = __ldg(n.lu_ptr + r + 1) - base;
    const int dl = __ldg(n.lu_diag + r) - base;
    for (int a = lane; a < len; a += 32) ws[a] = __ldcg(lu + base + a);
    __syncwarp();
    for (int a = 0; a < dl; ++a) {
      const int e = base + a, k = __ldg(n.lu_idx + e);
      if (__ldg(n.fr_pos + k) >= 0) continue;  // a front pivot: the dense phase
      const double l = ws[a] * __ldcg(invd + k);
      const int q0 = __ldg(n.upd_ptr + e), cnt = __ldg(n.upd_ptr + e + 1) - q0, u0 = __ldg(n.lu_diag + k) + 1;
      for (int t = lane; t < cnt; t += 32) ws[__ldg(n.upd_dst + q0 + t)] -= l * __ldcg(lu + u0 + t);
      __syncwarp();
      if (lane == 0) ws[a] = l;
      __syncwarp();
    }
    for (int a = lane; a < len; a += 32) __stcg(lu + base + a, ws[a]);
    __syncwarp();
  }
  cluster.sync();
  if (sub == 0) {
    const int LDS = F + 1;
    double* S = smem;  // [F][F + 1]
    for (int x = threadIdx.x; x < F * LDS; x += blockDim.x) S[x] = 0.0;
    __syncthreads();
    for (int f = warp; f < F; f += nwarp) {
      const int r = __ldg(n.fr_row + f), base = __ldg(n.lu_ptr + r), len = __ldg(n.lu_ptr + r + 1) - base;
      for (int a = lane; a < len; a += 32) {
        const int fc = __ldg(n.fr_pos + __ldg(n.lu_idx + base + a));
        if (fc >= 0) S[f * LDS + fc] = __ldcg(lu + base + a);
      }
    }
    __syncthreads();
    for (int k = 0; k < F; ++k) {
      const double piv = 1.0 / S[k * LDS + k];
      for (int i = k + 1 + threadIdx.x; i < F; i += blockDim.x) S[i * LDS + k] *= piv;
      __syncthreads();
      for (int i = k + 1 + warp; i < F; i += nwarp) {  // warp per row, lanes along it
        const double l = S[i * LDS + k];
        for (int j = k + 1 + lane; j < F; j += 32) S[i * LDS + j] -= l * S[k * LDS + j];
      }
      __syncthreads();
    }
    for (int f = warp; f < F; f += nwarp) {
      const int r = __ldg(n.fr_row + f), base = __ldg(n.lu_ptr + r), len = __ldg(n.lu_ptr + r + 1) - base;
      for (int a = lane; a < len; a += 32) {
        const int fc = __ldg(n.fr_pos + __ldg(n.lu_idx + base + a));
        if (fc >= 0) __stcg(lu + base + a, S[f * LDS + fc]);
      }
      if (lane == 0) {
        const double d = S[f * LDS + f];
        __stcg(invd + r, 1.0 / d);
        if (!(fabs(d) >= 1e-12 * rowmax[r]) || !isfinite(d) || d == 0.0) atomicMin(info, r + 1);
      }
    }
  }
  cluster.sync();
}

__global__ void __launch_bounds__(kLuThreads) k_lu(DevNet n, Work w, int CS) {
  cg::cluster_group cluster = cg::this_cluster();
  const int s = blockIdx.x / CS, sub = (int)cluster.block_rank();
  double* lu = w.lu + (size_t)s * n.nnz_lu;
  double* rowmax = w.rowmax + (size_t)s * n.n_x;
  const double* jb = w.jb + (size_t)s * n.nnz_jb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int gthread = sub * blockDim.x + threadIdx.x, nthread = CS * blockDim.x;
  // blocks go to the cluster's CTAs round-robin (below), so a narrow level puts at
  // most a few rows on each CTA, on its low warps, which own the staging areas
  if (gthread == 0) w.info[s] = INT_MAX;
  for (int r = gthread; r < n.n_x; r += nthread) {
    double mx = 0.0;
    for (int e = __ldg(n.lu_ptr + r); e < __ldg(n.lu_ptr + r + 1); ++e) {
      const int src = __ldg(n.lu_src + e);
      const double val = src >= 0 ? jb[src] : 0.0;
      __stcg(lu + e, val);
      mx = fmax(mx, fabs(val));
    }
    rowmax[r] = mx;
  }
  cluster.sync();
#ifdef PF_LU_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_lu_trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_lu_trace[0] = t;
  }
#endif
  extern __shared__ double lu_ws[];
  double* ws = lu_ws + warp * n.lu_maxlen;  // the warp's dense row workspace
  unsigned char* stb = reinterpret_cast<unsigned char*>(lu_ws + (size_t)nwarp * n.lu_maxlen) +
                       (size_t)min(warp, kLuStageWarps - 1) * kLuStageBytes;
  LuStage st;
  st.pin = reinterpret_cast<double*>(stb);
  st.val = st.pin + kLuMaxPiv;
  st.off = reinterpret_cast<int*>(st.val + kLuStageCap);
  st.dst = st.off + kLuMaxPiv + 2;
  double* invd = w.invd + (size_t)s * n.n_x;
  // Blocks go to warp PAIRS: the θ row of a bus block on the even warp, its v row on
  // the odd one.  The v row depends on the θ row only through its last pivot (the
  // intra-block entry), so both chains run at once; the v row applies that pivot
  // from the θ row's workspace after a pair barrier.
  const int pw = warp >> 1, hv = warp & 1;
  const int gpair = pw * CS + sub, ngpair = CS * (nwarp >> 1);
  // one bus block (its θ row on the pair's even warp, its v row on the odd one)
  auto do_block = [&](const int p, const int lev) {
    const int rb = __ldg(n.blk_ptr + p), nrow = __ldg(n.blk_ptr + p + 1) - rb;
    const int r = rb + hv;
    int base = 0, len = 0, dl = 0;
    bool defer = false;
    if (hv < nrow) {
      base = __ldg(n.lu_ptr + r); len = __ldg(n.lu_ptr + r + 1) - base;
      dl = __ldg(n.lu_diag + r) - base;
      defer = hv == 1 && dl > 0 && __ldg(n.lu_idx + base + dl - 1) == rb;
      if (hv == 1 && !defer) asm volatile("bar.sync %0, 64;" ::"r"(1 + pw) : "memory");  // no intra entry: wait
      LU_PH(lev, 0);
      for (int a = lane; a < len; a += 32) ws[a] = __ldcg(lu + base + a);
      __syncwarp();
      LU_PH(lev, 1);
      const int np = defer ? dl - 1 : dl;  // pivots of this pass
        if (warp < kLuStageWarps && np >= kLuStageMin && np <= kLuMaxPiv && stage_row(n, lu, invd, base, np, lane, st)) {
          LU_PH(lev, 2);
          // long (separator) row: its whole IKJ working set is in SMEM, the chain runs there
          for (int a = 0; a < np; ++a) {
            const double l = ws[a] * st.pin[a];
            const int o = st.off[a], cnt = st.off[a + 1] - o;
            for (int t = lane; t < cnt; t += 32) ws[st.dst[o + t]] -= l * st.val[o + t];
            __syncwarp();  // the next pivot's entry may just have been updated
            if (lane == 0) ws[a] = l;  // (entry a is not read again by the chain)
          }
          __syncwarp();
        } else {
          // IKJ over the row's L entries; the U row of the next pivot and the
          // update targets are prefetched into registers while this one runs.
          double pu[4], pin = 0.0;
          int pd[4], pq0 = 0, pcnt = 0, pu0 = 0;
          auto fetch = [&](int a) {
            const int e = base + a, k = __ldg(n.lu_idx + e);
            pu0 = __ldg(n.lu_diag + k) + 1;
            pq0 = __ldg(n.upd_ptr + e);
            pcnt = __ldg(n.upd_ptr + e + 1) - pq0;
            pin = __ldcg(invd + k);
  #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int t = lane + 32 * j;
              pu[j] = t < pcnt ? __ldcg(lu + pu0 + t) : 0.0;
              pd[j] = t < pcnt ? __ldg(n.upd_dst + pq0 + t) : 0;
            }
          };
          if (np > 0) fetch(0);
          for (int a = 0; a < np; ++a) {
            const double cu[4] = {pu[0], pu[1], pu[2], pu[3]};
            const int cd[4] = {pd[0], pd[1], pd[2], pd[3]};
            const double cin = pin;
            const int q0 = pq0, cnt = pcnt, u0 = pu0;
            if (a + 1 < np) fetch(a + 1);
            const double l = ws[a] * cin;
  #pragma unroll
            for (int j = 0; j < 4; ++j)
              if (lane + 32 * j < cnt) ws[cd[j]] -= l * cu[j];
            for (int t = lane + 128; t < cnt; t += 32) ws[__ldg(n.upd_dst + q0 + t)] -= l * __ldcg(lu + u0 + t);
            __syncwarp();
            if (lane == 0) ws[a] = l;
          }
        }
    }
    if (nrow == 2 && (hv == 0 || defer)) asm volatile("bar.sync %0, 64;" ::"r"(1 + pw) : "memory");
    if (defer) {  // the θ row's pivot, from its workspace
      const double* ws0 = lu_ws + (size_t)(warp - 1) * n.lu_maxlen;
      const int base0 = __ldg(n.lu_ptr + rb), dl0 = __ldg(n.lu_diag + rb) - base0;
      const int e = base + dl - 1, q0 = __ldg(n.upd_ptr + e), cnt = __ldg(n.upd_ptr + e + 1) - q0;
      const int o0 = dl0 + 1;  // U part of the θ row in ws0
      const double l = ws[dl - 1] * (1.0 / ws0[dl0]);
      for (int t = lane; t < cnt; t += 32) ws[__ldg(n.upd_dst + q0 + t)] -= l * ws0[o0 + t];
      __syncwarp();
      if (lane == 0) ws[dl - 1] = l;
    }
    if (hv < nrow) {
      __syncwarp();
      LU_PH(lev, 3);
      for (int a = lane; a < len; a += 32) __stcg(lu + base + a, ws[a]);
      if (lane == 0) {
        const double d = ws[dl];
        __stcg(invd + r, 1.0 / d);
        if (!(fabs(d) >= 1e-12 * rowmax[r]) || !isfinite(d) || d == 0.0) atomicMin(w.info + s, r + 1);
      }
      __syncwarp();
    }
    // ws0 free for the next block; and both rows stored before the pair's next block (in the
    // bottom subtrees that block may be this one's parent)
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pw) : "memory");
    LU_PH(lev, 4);
  };
  // Bottom levels (< lu_lev0): each warp pair walks its subtrees of the block elimination
  // forest in postorder (a block needs only its descendants, done earlier by the same pair),
  // with no cluster barrier; the schedule is built for lu_nteam pairs (pf_api.cu).
  for (int t = gpair; t < n.lu_nteam; t += ngpair)
    for (int q = __ldg(n.lu_p1_ptr + t); q < __ldg(n.lu_p1_ptr + t + 1); ++q) do_block(__ldg(n.lu_p1_blk + q), 0);
  cluster.sync();
  for (int lev = n.lu_lev0; lev < n.fr_lev; ++lev) {
    const int b0 = __ldg(n.levL_ptr + lev), b1 = __ldg(n.levL_ptr + lev + 1);
    for (int bi = b0 + gpair; bi < b1; bi += ngpair) do_block(__ldg(n.lu_lev_blk + bi), lev);
    LU_PH(lev, 5);
    cluster.sync();
#ifdef PF_LU_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_lu_trace) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_lu_trace[lev + 1] = t;
    }
#endif
  }
  if (n.fr_n > 0) lu_front(n, lu, invd, rowmax, w.info + s, lu_ws, sub, CS, cluster);
  // sweep streams (pf_api.cu segment layout): a diagonal entry (its own transpose position)
  // is packed as 1/u_rr, so the sweeps that divide multiply instead
  double2* swA = w.swA + (size_t)s * n.nsw;
  double2* swT = w.swT + (size_t)s * n.nsw;
  auto vA = [&](int e) { const double x = __ldcg(lu + e); return __ldg(n.lu_tpos + e) == e ? 1.0 / x : x; };
  auto vT = [&](int e) {
    const int tp = __ldg(n.lu_tpos + e);
    return tp == e ? 1.0 / __ldcg(lu + e) : __ldcg(lu + tp);
  };
  for (int q = gthread; q < n.nsw; q += nthread) {
    const int2 src = __ldg(n.sw_src + q);
    double2 a, t;
    if (src.y == -1 || src.y == -2) {  // gather / pad: {value or 0, column·C}
      const double c = __longlong_as_double((long long)__ldg(n.lu_idx + src.x) * n.C);
      a = make_double2(src.y == -1 ? vA(src.x) : 0.0, c);
      t = make_double2(src.y == -1 ? vT(src.x) : 0.0, c);
    } else {                           // block scalars
      a = make_double2(src.x >= 0 ? vA(src.x) : 0.0, src.y >= 0 ? vA(src.y) : 0.0);
      t = make_double2(src.x >= 0 ? vT(src.x) : 0.0, src.y >= 0 ? vT(src.y) : 0.0);
    }
    swA[q] = a;
    swT[q] = t;
  }
}

__global__ void k_lu_info(int n_scen, int* __restrict__ info, int* __restrict__ info_out) {
  for (int s = threadIdx.x; s < n_scen; s += blockDim.x) {
    const int v = info[s] == INT_MAX ? 0 : info[s];
    info[s] = v;
    if (info_out) info_out[s] = v;
  }
}

// ---------------------------------------------------------------- A6
// μ̃ (bus multipliers of ∇²p_i, ∇²q_i): λ on g rows, y_r on r rows and
// (2c1 p_ref + c2)_{g_r} on P_r0 (R8); Σ of the r rows (with the p_ref
// curvature 2c1_{g_r} folded into P_r0) and Σ_x of each bus variable.
__global__ void k_prep_bus1(DevNet n, Work w, int n_scen, const double* __restrict__ p_d,
                            const double* __restrict__ lam, const double* __restrict__ y,
                            const double* __restrict__ sig_s, const double* __restrict__ sig_x) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    const double* L = lam + (size_t)s * n.n_x;
    const double* Y = y + (size_t)s * n.m;
    double* bs = w.bs + (size_t)s * BS_N * n.n_b;
    const int xt = __ldg(n.x_th + i), xv = __ldg(n.x_v + i), rp = __ldg(n.bus_rP + i), rq = __ldg(n.bus_rQ + i);
    double muP = (xt >= 0 ? L[xt] : 0.0) + (rp >= 0 ? Y[rp] : 0.0);
    double muQ = (xv >= 0 ? L[xv] : 0.0) + (rq >= 0 ? Y[rq] : 0.0);
    double srp = (rp >= 0 && sig_s) ? sig_s[(size_t)s * n.m + rp] : 0.0;
    if (i == n.r0) {
      const double* ls = w.ls + (size_t)s * LS_N * n.n_l;
      double P = 0.0;
      for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
        const int l = __ldg(n.inc_line + e);
        P += __ldg(n.lf + l) == i ? ls[LS_SPF * n.n_l + l] : ls[LS_SPT * n.n_l + l];
      }
      const double vi = bs[BS_V * n.n_b + i];
      P += __ldg(n.gsh + i) * vi * vi;
      const double pref = P + (p_d ? p_d[(size_t)s * n.n_b + i] : __ldg(n.p_d0 + i));
      const double c1 = __ldg(n.c_quad + n.g_r), c2 = __ldg(n.c_lin + n.g_r);
      muP += 2.0 * c1 * pref + c2;
      srp += 2.0 * c1;
    }
    bs[BS_MUP * n.n_b + i] = muP;
    bs[BS_MUQ * n.n_b + i] = muQ;
    bs[BS_SRP * n.n_b + i] = srp;
    bs[BS_SRQ * n.n_b + i] = (rq >= 0 && sig_s) ? sig_s[(size_t)s * n.m + rq] : 0.0;
    bs[BS_SXT * n.n_b + i] = (xt >= 0 && sig_x) ? sig_x[(size_t)s * n.n_x + xt] : 0.0;
    bs[BS_SXV * n.n_b + i] = (xv >= 0 && sig_x) ? sig_x[(size_t)s * n.n_x + xv] : 0.0;
  }
}

// w̄ = Mᵀμ̃ + L_lineᵀ(2ŷ ⊙ s) per line (A6): with the end "efforts"
// E = μ̃ + 2ŷ s, w̄^c = g_ft E_fp − b_ft E_fq + g_tf E_tp − b_tf E_tq,
// w̄^s = b_ft E_fp + g_ft E_fq − b_tf E_tp − g_tf E_tq; the v² columns give
// the per-end diagonal parts d_f, d_t of w̄^d.
__global__ void k_prep_line(DevNet n, Work w, int n_scen, const double* __restrict__ y,
                            const double* __restrict__ sig_s) {
  const long long total = (long long)n_scen * n.n_l;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_l), l = (int)(t % n.n_l);
    double* ls = w.ls + (size_t)s * LS_N * n.n_l;
    const double* bs = w.bs + (size_t)s * BS_N * n.n_b;
    const int f = __ldg(n.lf + l), to = __ldg(n.lt + l);
    const int hf = __ldg(n.line_hf + l), ht = __ldg(n.line_ht + l);
    const double* Y = y + (size_t)s * n.m;
    const double y2f = hf >= 0 ? 2.0 * Y[n.n_r + hf] : 0.0;
    const double y2t = ht >= 0 ? 2.0 * Y[n.n_r + ht] : 0.0;
    const double sgf = (hf >= 0 && sig_s) ? sig_s[(size_t)s * n.m + n.n_r + hf] : 0.0;
    const double sgt = (ht >= 0 && sig_s) ? sig_s[(size_t)s * n.m + n.n_r + ht] : 0.0;
    const LineCoef k = load_coef(n, l);
    const double Efp = bs[BS_MUP * n.n_b + f] + y2f * ls[LS_SPF * n.n_l + l];
    const double Efq = bs[BS_MUQ * n.n_b + f] + y2f * ls[LS_SQF * n.n_l + l];
    const double Etp = bs[BS_MUP * n.n_b + to] + y2t * ls[LS_SPT * n.n_l + l];
    const double Etq = bs[BS_MUQ * n.n_b + to] + y2t * ls[LS_SQT * n.n_l + l];
    ls[LS_WC * n.n_l + l] = k.gft * Efp - k.bft * Efq + k.gtf * Etp - k.btf * Etq;
    ls[LS_WS * n.n_l + l] = k.bft * Efp + k.gft * Efq - k.btf * Etp - k.gtf * Etq;
    ls[LS_DF * n.n_l + l] = k.gff * Efp - k.bff * Efq;
    ls[LS_DT * n.n_l + l] = k.gtt * Etp - k.btt * Etq;
    ls[LS_Y2F * n.n_l + l] = y2f; ls[LS_Y2T * n.n_l + l] = y2t;
    ls[LS_SGF * n.n_l + l] = sgf; ls[LS_SGT * n.n_l + l] = sgt;

    // Line-local blocks of K in the coordinates (v_f, v_t, Δ = θ_f − θ_t):
    //   J (4×3) = ∂(s_p^f, s_q^f, s_p^t, s_q^t) = L_line J_ψ (+ the v² columns),
    //   H (3×3) = w̄^c ∇²ψ^c + w̄^s ∇²ψ^s                       (second order, A6)
    //           + Σ_ends 2ŷ (∇s_p∇s_pᵀ + ∇s_q∇s_qᵀ)            (y_h Gauss–Newton)
    //           + Σ_ends Σ_h ∇H ∇Hᵀ, ∇H = 2(s_p∇s_p + s_q∇s_q)   (AᵀΣ_sA on h rows).
    // K·d restricted to the line is then H d_loc + Jᵀ μ_A(ends): linear in d,
    // so it is precomputed once per scenario instead of once per direction.
    {
      const double vf = ls[LS_VF * n.n_l + l], vt = ls[LS_VT * n.n_l + l];
      const double c = ls[LS_C * n.n_l + l], sn = ls[LS_S * n.n_l + l];
      const double pc = vf * vt * c, ps = vf * vt * sn;
      const double dc[3] = {vt * c, vf * c, -ps}, ds[3] = {vt * sn, vf * sn, pc};
      double J[4][3];
      for (int a = 0; a < 3; ++a) {
        J[0][a] = k.gft * dc[a] + k.bft * ds[a];
        J[1][a] = -k.bft * dc[a] + k.gft * ds[a];
        J[2][a] = k.gtf * dc[a] - k.btf * ds[a];
        J[3][a] = -k.btf * dc[a] - k.gtf * ds[a];
      }
      J[0][0] += 2.0 * k.gff * vf; J[1][0] -= 2.0 * k.bff * vf;
      J[2][1] += 2.0 * k.gtt * vt; J[3][1] -= 2.0 * k.btt * vt;
      const double wc = ls[LS_WC * n.n_l + l], ws = ls[LS_WS * n.n_l + l];
      // ∇²ψ^c = [[0, c, −v_t s], [c, 0, −v_f s], [−v_t s, −v_f s, −ψ^c]],
      // ∇²ψ^s = [[0, s, v_t c], [s, 0, v_f c], [v_t c, v_f c, −ψ^s]]
      double H[3][3] = {{0.0, wc * c + ws * sn, -wc * vt * sn + ws * vt * c},
                        {0.0, 0.0, -wc * vf * sn + ws * vf * c},
                        {0.0, 0.0, -wc * pc - ws * ps}};
      const double spv[2] = {ls[LS_SPF * n.n_l + l], ls[LS_SPT * n.n_l + l]};
      const double sqv[2] = {ls[LS_SQF * n.n_l + l], ls[LS_SQT * n.n_l + l]};
      const double y2[2] = {y2f, y2t}, sg[2] = {sgf, sgt};
      for (int e = 0; e < 2; ++e) {
        const double* Jp = J[2 * e];
        const double* Jq = J[2 * e + 1];
        double gH[3];
        for (int a = 0; a < 3; ++a) gH[a] = 2.0 * (spv[e] * Jp[a] + sqv[e] * Jq[a]);
        for (int a = 0; a < 3; ++a)
          for (int b = a; b < 3; ++b) H[a][b] += y2[e] * (Jp[a] * Jp[b] + Jq[a] * Jq[b]) + sg[e] * gH[a] * gH[b];
      }
      double* o = w.lblk + ((size_t)s * n.n_l + l) * LB_N;
      o[LB_H00] = H[0][0]; o[LB_H01] = H[0][1]; o[LB_H02] = H[0][2];
      o[LB_H11] = H[1][1]; o[LB_H12] = H[1][2]; o[LB_H22] = H[2][2];
      for (int r = 0; r < 4; ++r)
        for (int a = 0; a < 3; ++a) o[LB_J + 3 * r + a] = J[r][a];
    }
  }
}

// w̄^d_i = Σ_{ends at i} d_end + g_sh μ̃^P_i − b_sh μ̃^Q_i (R4 diagonal); stores 2 w̄^d.
__global__ void k_prep_bus2(DevNet n, Work w, int n_scen) {
  const long long total = (long long)n_scen * n.n_b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.n_b), i = (int)(t % n.n_b);
    const double* ls = w.ls + (size_t)s * LS_N * n.n_l;
    double* bs = w.bs + (size_t)s * BS_N * n.n_b;
    double wd = __ldg(n.gsh + i) * bs[BS_MUP * n.n_b + i] - __ldg(n.bsh + i) * bs[BS_MUQ * n.n_b + i];
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int l = __ldg(n.inc_line + e);
      wd += __ldg(n.lf + l) == i ? ls[LS_DF * n.n_l + l] : ls[LS_DT * n.n_l + l];
    }
    bs[BS_WD2 * n.n_b + i] = 2.0 * wd;
  }
}

// K's 2×2 bus blocks for k_hvp (A6): B_ij on (θ, v) of buses i, j from the line
// blocks H (3×3 on (v_f, v_t, Δ), Δ = θ_f − θ_t) of the lines between them —
//   B_ff = [[H22, H02], [H02, H00]],   B_ft = [[−H22, H12], [−H02, H01]],
//   B_tt = [[H22, −H12], [−H12, H11]], B_tf = B_ftᵀ —
// plus, on the diagonal, Σ_x and the ψ^d curvature 2w̄^d; and JT_ij =
// ∂(P_j, Q_j)/∂(θ_i, v_i)ᵀ from J_bus when j is a generator bus (the A_rᵀ μ_A part).
// The θ columns of B sum to zero over j (every line term depends on Δ only), so
// k_hvp applies them to angle DIFFERENCES, (h_θ, h_v)_i += B_ij[:, θ] (dθ_j − dθ_i),
// as the line form does (no cancellation for smooth directions such as state
// steps); the diagonal block then keeps only Σ_x on its θ column.
__global__ void k_prep_hblk(DevNet n, Work w, int n_scen) {
  const long long total = (long long)n_scen * n.hb.nblk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.hb.nblk), e = (int)(t % n.hb.nblk);
    const int i = __ldg(n.hb.self + e), j = __ldg(n.hb.nbr + e);
    const double* lb = w.lblk + (size_t)s * n.n_l * LB_N;
    double b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
    for (int q = __ldg(n.inc_ptr + i); q < __ldg(n.inc_ptr + i + 1); ++q) {
      const int l = __ldg(n.inc_line + q);
      const bool from = __ldg(n.lf + l) == i;
      const int o = from ? __ldg(n.lt + l) : __ldg(n.lf + l);
      if (j != i && o != j) continue;
      const double* H = lb + (size_t)l * LB_N;
      const double h00 = H[LB_H00], h01 = H[LB_H01], h02 = H[LB_H02], h11 = H[LB_H11], h12 = H[LB_H12],
                   h22 = H[LB_H22];
      if (j == i) {  // θ column: carried by the off-diagonal blocks' differences
        if (from) { b01 += h02; b11 += h00; }
        else { b01 -= h12; b11 += h11; }
      } else {
        if (from) { b00 -= h22; b01 += h12; b10 -= h02; b11 += h01; }
        else { b00 -= h22; b01 -= h02; b10 += h12; b11 += h01; }
      }
    }
    if (j == i) {
      const double* bs = w.bs + (size_t)s * BS_N * n.n_b;
      b00 += bs[BS_SXT * n.n_b + i];
      b11 += bs[BS_WD2 * n.n_b + i] + bs[BS_SXV * n.n_b + i];
    }
    double jt[4] = {0.0, 0.0, 0.0, 0.0};
    const int2 off = __ldg(n.hb.jt + e);
    if (__ldg(n.bus_gen + j) >= 0) {
      const double* jb = w.jb + (size_t)s * n.nnz_jb;
      const int rp = __ldg(n.jb_ptr + j), rq = __ldg(n.jb_ptr + n.n_b + j);
      if (off.x >= 0) { jt[0] = jb[rp + off.x]; jt[1] = jb[rq + off.x]; }
      if (off.y >= 0) { jt[2] = jb[rp + off.y]; jt[3] = jb[rq + off.y]; }
    }
    double2* o = reinterpret_cast<double2*>(w.hbval + ((size_t)s * n.hb.nblk + e) * 8);
    o[0] = make_double2(b00, b01); o[1] = make_double2(b10, b11);
    o[2] = make_double2(jt[0], jt[1]); o[3] = make_double2(jt[2], jt[3]);
  }
}

// The generator-bus blocks of k_mu (A7.3 first half): dG_g = A_r,g · d as 2×2 blocks
// M_gj = ∂(P_g, Q_g)/∂(θ_j, v_j) from the line Jacobians J (4×3 on (v_f, v_t, Δ)) —
// θ columns applied to angle differences (dθ_j − dθ_g) like k_hvp's, so the diagonal
// block carries only the v column (own line ends + the shunt 2 g_sh v_g, −2 b_sh v_g).
__global__ void k_prep_mblk(DevNet n, Work w, int n_scen) {
  const long long total = (long long)n_scen * n.mb.nblk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / n.mb.nblk), e = (int)(t % n.mb.nblk);
    const int g = __ldg(n.mb.self + e), j = __ldg(n.mb.nbr + e);
    const double* lb = w.lblk + (size_t)s * n.n_l * LB_N;
    double pt = 0.0, pv = 0.0, qt = 0.0, qv = 0.0;
    for (int q = __ldg(n.inc_ptr + g); q < __ldg(n.inc_ptr + g + 1); ++q) {
      const int l = __ldg(n.inc_line + q);
      const bool from = __ldg(n.lf + l) == g;
      const int o = from ? __ldg(n.lt + l) : __ldg(n.lf + l);
      if (j != g && o != j) continue;
      const double* J = lb + (size_t)l * LB_N + LB_J;   // rows (s_p^f, s_q^f, s_p^t, s_q^t), cols (v_f, v_t, Δ)
      const double* Jp = J + (from ? 0 : 6);
      const double* Jq = J + (from ? 3 : 9);
      if (j == g) { pv += Jp[from ? 0 : 1]; qv += Jq[from ? 0 : 1]; }
      else {        // Δ = θ_f − θ_t: ∂/∂θ_j = −∂/∂Δ at the from end, +∂/∂Δ at the to end
        pt += from ? -Jp[2] : Jp[2]; qt += from ? -Jq[2] : Jq[2];
        pv += Jp[from ? 1 : 0]; qv += Jq[from ? 1 : 0];
      }
    }
    if (j == g) {
      const double vg = w.bs[(size_t)s * BS_N * n.n_b + BS_V * n.n_b + g];
      pv += 2.0 * __ldg(n.gsh + g) * vg;
      qv -= 2.0 * __ldg(n.bsh + g) * vg;
    }
    double2* out = reinterpret_cast<double2*>(w.mbval + ((size_t)s * n.mb.nblk + e) * 8);
    out[0] = make_double2(pt, pv); out[1] = make_double2(qt, qv);
  }
}

}  // namespace

#ifdef PF_LU_TRACE
void set_lu_trace(unsigned long long* p) { cudaMemcpyToSymbol(g_lu_trace, &p, sizeof(p)); }
#endif

int launch_eval(const DevNet& n, const Work& w, int n_scen, const double* v, const double* th,
                const double* p_g, const double* q_g, const double* p_d, const double* q_d,
                double* G, double* H, double* s_flow, cudaStream_t st) {
  k_line_eval<<<blocks_for((long long)n_scen * n.n_l), kThreads, 0, st>>>(n, w, n_scen, v, th, H, s_flow);
  k_bus_eval<<<blocks_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen, v, p_g, q_g, p_d, q_d, G);
  return 2;
}

static size_t lu_smem(const DevNet& n) {
  const size_t rows = (size_t)(kLuThreads / 32) * n.lu_maxlen * sizeof(double) + kLuStageWarps * kLuStageBytes;
  return std::max(rows, (size_t)n.fr_n * (n.fr_n + 1) * sizeof(double));  // the front reuses the area
}

size_t lu_smem_bytes(const DevNet& n) { return lu_smem(n); }

int lu_cluster_size(const DevNet& n) {
  // 16-CTA clusters (non-portable) when the part supports them, else 8, 4, …
  const size_t smem = lu_smem(n);
  cudaFuncSetAttribute(k_lu, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int CS = 0;
  for (int cs : {16, 8, 4, 2, 1}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(kLuThreads); cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (void*)k_lu, &cfg) == cudaSuccess && nc > 0) { CS = cs; break; }
  }
  cudaGetLastError();
  return CS ? CS : 1;
}

int launch_jacobian(const DevNet& n, const Work& w, int n_scen, const double* v, const double* th,
                    double* Gx, double* Gu, double* A, int* info, cudaStream_t st, int lu_cs, cudaEvent_t* ev) {
  k_line_state<<<blocks_for((long long)n_scen * n.n_l), kThreads, 0, st>>>(n, w, n_scen, v, th);
  k_bus_v<<<blocks_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen, v);
  k_jbus<<<blocks_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen);
  k_gather<<<blocks_for((long long)n_scen * (n.nnz_gx + n.nnz_gu + n.nnz_a)), kThreads, 0, st>>>(n, w, n_scen, Gx, Gu, A);
  const size_t smem = lu_smem(n);
  const int CS = lu_cs;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(n_scen * CS); cfg.blockDim = dim3(kLuThreads); cfg.dynamicSmemBytes = smem;
  cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;
  if (ev) cudaEventRecord(ev[0], st);
  cudaLaunchKernelEx(&cfg, k_lu, n, w, CS);
  if (ev) cudaEventRecord(ev[1], st);
  k_lu_info<<<1, 256, 0, st>>>(n_scen, w.info, info);
  return 6;
}

int launch_prep(const DevNet& n, const Work& w, int n_scen, const double* p_d, const double* lam,
                const double* y, const double* sigma_s, const double* sigma_x, cudaStream_t st) {
  k_prep_bus1<<<blocks_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen, p_d, lam, y, sigma_s, sigma_x);
  k_prep_line<<<blocks_for((long long)n_scen * n.n_l), kThreads, 0, st>>>(n, w, n_scen, y, sigma_s);
  k_prep_bus2<<<blocks_for((long long)n_scen * n.n_b), kThreads, 0, st>>>(n, w, n_scen);
  k_prep_hblk<<<blocks_for((long long)n_scen * n.hb.nblk), kThreads, 0, st>>>(n, w, n_scen);
  k_prep_mblk<<<blocks_for((long long)n_scen * n.mb.nblk), kThreads, 0, st>>>(n, w, n_scen);
  return 5;
}

}  // namespace pf
