// pf_reduce.cu — the batched reduced-Hessian kernel (A7.1–A7.5 of SURVEY §8(a)).
//
// One CTA owns a tile of C Hessian-vector directions of one scenario and runs
// the paper's three steps (with R11) end to end, without
// leaving the kernel:
//   a. B = −P G_u V            (unit V: a column scatter; dense V: a row SpMM)
//   b. Z̃ = U^{-1} L^{-1} B     (level-scheduled sweeps, bus blocks of 1–2 rows)
//   c. [H_u; H_x] = K [V; Z]   (matrix-free through ψ: line-local J_ψ, L_line,
//                              ∇²ψ with w̄, plus the r-row / p_ref terms,
//                              AᵀΣ_sA, Σ_x; deterministic bus gathers)
//   d. Ψ̃ = L^{-T} U^{-T} H̃_x  (transposed sweeps on the same level sets)
//   e. K̂V = H_u − (P G_u)ᵀ Ψ̃  (column gathers, transposed through SMEM so the
//                              [N][n_u] output is written coalesced)
// Slabs are [n_x][C] (direction fastest): a team of C lanes handles one row,
// lane j = direction j, so every slab access is one contiguous C×8-byte run.
// Columns are independent: each column's arithmetic is the same for any N,
// any tile, any GPU count (bit-identical K̂ across batch sizes).
#include "pf_launch.h"

namespace pf {

namespace {

constexpr int kRedThreads = 256;
constexpr int kCH = 64;  // u-columns per transposed output chunk

template <int C>
__device__ __forceinline__ void sweep_L(const DevNet& n, const double* __restrict__ lu, double* X, int lane, int team, int nteam) {
  for (int lev = 0; lev < n.nlevL; ++lev) {
    const int b1 = __ldg(n.levL_ptr + lev + 1);
    for (int bi = __ldg(n.levL_ptr + lev) + team; bi < b1; bi += nteam) {
      const int p = __ldg(n.levL_blk + bi);
      const int r1 = __ldg(n.blk_ptr + p + 1);
      for (int r = __ldg(n.blk_ptr + p); r < r1; ++r) {
        double acc = X[r * C + lane];
        const int e1 = __ldg(n.lu_diag + r);
        for (int e = __ldg(n.lu_ptr + r); e < e1; ++e) acc -= __ldg(lu + e) * X[__ldg(n.lu_idx + e) * C + lane];
        X[r * C + lane] = acc;
      }
    }
    __syncthreads();
  }
}

template <int C>
__device__ __forceinline__ void sweep_U(const DevNet& n, const double* __restrict__ lu, double* X, int lane, int team, int nteam) {
  for (int lev = 0; lev < n.nlevU; ++lev) {
    const int b1 = __ldg(n.levU_ptr + lev + 1);
    for (int bi = __ldg(n.levU_ptr + lev) + team; bi < b1; bi += nteam) {
      const int p = __ldg(n.levU_blk + bi);
      const int r0 = __ldg(n.blk_ptr + p);
      for (int r = __ldg(n.blk_ptr + p + 1) - 1; r >= r0; --r) {
        double acc = X[r * C + lane];
        const int d = __ldg(n.lu_diag + r), e1 = __ldg(n.lu_ptr + r + 1);
        for (int e = d + 1; e < e1; ++e) acc -= __ldg(lu + e) * X[__ldg(n.lu_idx + e) * C + lane];
        X[r * C + lane] = acc / __ldg(lu + d);
      }
    }
    __syncthreads();
  }
}

// Uᵀ z = h (forward, L level sets): z_r = (h_r − Σ_{k<r} u_kr z_k) / u_rr,
// the u_kr read through the transposed copy luT at row r's L positions.
template <int C>
__device__ __forceinline__ void sweep_UT(const DevNet& n, const double* __restrict__ lu, const double* __restrict__ luT,
                                         double* X, int lane, int team, int nteam) {
  for (int lev = 0; lev < n.nlevL; ++lev) {
    const int b1 = __ldg(n.levL_ptr + lev + 1);
    for (int bi = __ldg(n.levL_ptr + lev) + team; bi < b1; bi += nteam) {
      const int p = __ldg(n.levL_blk + bi);
      const int r1 = __ldg(n.blk_ptr + p + 1);
      for (int r = __ldg(n.blk_ptr + p); r < r1; ++r) {
        double acc = X[r * C + lane];
        const int d = __ldg(n.lu_diag + r);
        for (int e = __ldg(n.lu_ptr + r); e < d; ++e) acc -= __ldg(luT + e) * X[__ldg(n.lu_idx + e) * C + lane];
        X[r * C + lane] = acc / __ldg(lu + d);
      }
    }
    __syncthreads();
  }
}

// Lᵀ w = z (backward, U level sets): w_r = z_r − Σ_{j>r} l_jr w_j.
template <int C>
__device__ __forceinline__ void sweep_LT(const DevNet& n, const double* __restrict__ luT, double* X, int lane, int team, int nteam) {
  for (int lev = 0; lev < n.nlevU; ++lev) {
    const int b1 = __ldg(n.levU_ptr + lev + 1);
    for (int bi = __ldg(n.levU_ptr + lev) + team; bi < b1; bi += nteam) {
      const int p = __ldg(n.levU_blk + bi);
      const int r0 = __ldg(n.blk_ptr + p);
      for (int r = __ldg(n.blk_ptr + p + 1) - 1; r >= r0; --r) {
        double acc = X[r * C + lane];
        const int e1 = __ldg(n.lu_ptr + r + 1);
        for (int e = __ldg(n.lu_diag + r) + 1; e < e1; ++e) acc -= __ldg(luT + e) * X[__ldg(n.lu_idx + e) * C + lane];
        X[r * C + lane] = acc;
      }
    }
    __syncthreads();
  }
}

struct Coef { double gff, bff, gft, bft, gtf, btf, gtt, btt; };

__device__ __forceinline__ Coef coef(const DevNet& n, int l) {
  Coef c;
  c.gff = __ldg(n.coef + 0 * n.n_l + l); c.bff = __ldg(n.coef + 1 * n.n_l + l);
  c.gft = __ldg(n.coef + 2 * n.n_l + l); c.bft = __ldg(n.coef + 3 * n.n_l + l);
  c.gtf = __ldg(n.coef + 4 * n.n_l + l); c.btf = __ldg(n.coef + 5 * n.n_l + l);
  c.gtt = __ldg(n.coef + 6 * n.n_l + l); c.btt = __ldg(n.coef + 7 * n.n_l + l);
  return c;
}

template <int C>
__global__ void __launch_bounds__(kRedThreads) k_reduce(DevNet n, Work w, int n_scen, const double* __restrict__ V,
                                                        int col0, int N, double* __restrict__ KV) {
  __shared__ double T[C][kCH + 1];
  const int ntile = (N + C - 1) / C;
  const int tile = blockIdx.x, s = blockIdx.y;
  const size_t cta = (size_t)s * ntile + tile;
  const int lane = threadIdx.x % C, team = threadIdx.x / C, nteam = blockDim.x / C;
  const int j = tile * C + lane;
  const bool valid = j < N;
  const int n_x = n.n_x, n_u = n.n_u, n_l = n.n_l, n_b = n.n_b;
  double* X = w.slabZ + cta * n_x * C;
  double* Y = w.slabW + cta * n_x * C;
  double* Hs = w.hu + cta * n_u * C;
  double* MU = w.mu + cta * n.n_g * 2 * C;
  const double* lu = w.lu + (size_t)s * n.nnz_lu;
  const double* luT = w.luT + (size_t)s * n.nnz_lu;
  const double* gu = w.gu + (size_t)s * n.nnz_gu;
  const double* ls = w.ls + (size_t)s * LS_N * n_l;
  const double* bs = w.bs + (size_t)s * BS_N * n_b;
  const double* Vs = (V && valid) ? V + ((size_t)s * N + j) * n_u : nullptr;
  auto vdir = [&](int c) -> double {
    if (!valid) return 0.0;
    return Vs ? Vs[c] : (c == col0 + j ? 1.0 : 0.0);
  };

  // ---- a. tangent right-hand side B = −P G_u V (A7.1)
  if (V == nullptr) {
    for (int idx = threadIdx.x; idx < n_x * C; idx += blockDim.x) X[idx] = 0.0;
    __syncthreads();
    if (team == 0 && valid) {
      const int c = col0 + j;
      for (int e = __ldg(n.guc_ptr + c); e < __ldg(n.guc_ptr + c + 1); ++e)
        X[__ldg(n.guc_row + e) * C + lane] = -gu[__ldg(n.guc_src + e)];
    }
  } else {
    for (int r = team; r < n_x; r += nteam) {
      double acc = 0.0;
      for (int e = __ldg(n.gur_ptr + r); e < __ldg(n.gur_ptr + r + 1); ++e)
        acc += gu[__ldg(n.gur_src + e)] * vdir(__ldg(n.gur_col + e));
      X[r * C + lane] = -acc;
    }
  }
  __syncthreads();

  // ---- b. forward tangent solve Z̃ = U^{-1} L^{-1} B (A7.2)
  sweep_L<C>(n, lu, X, lane, team, nteam);
  sweep_U<C>(n, lu, X, lane, team, nteam);

  auto dth = [&](int i) -> double { const int p = __ldg(n.bus_pth + i); return p >= 0 ? X[p * C + lane] : 0.0; };
  auto dv = [&](int i) -> double { const int p = __ldg(n.bus_pv + i); return p >= 0 ? X[p * C + lane] : vdir(__ldg(n.u_v + i)); };

  // ---- c1. μ_A = Σ_r ⊙ dG_r at the r buses (generator buses), dG_r = R_r M dψ
  for (int gi = team; gi < n.n_gb; gi += nteam) {
    const int i = __ldg(n.gbus + gi);
    const double dvi = dv(i), dthi = dth(i);
    double dP = 0.0, dQ = 0.0;
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int l = __ldg(n.inc_line + e);
      const bool from = __ldg(n.lf + l) == i;
      const int o = from ? __ldg(n.lt + l) : __ldg(n.lf + l);
      const double dvo = dv(o), dtho = dth(o);
      const Coef k = coef(n, l);
      const double vf = ls[LS_VF * n_l + l], vt = ls[LS_VT * n_l + l];
      const double c = ls[LS_C * n_l + l], sn = ls[LS_S * n_l + l];
      const double dvf = from ? dvi : dvo, dvt = from ? dvo : dvi;
      const double dD = from ? dthi - dtho : dtho - dthi;
      const double pc = vf * vt * c, ps = vf * vt * sn;
      const double dpc = vt * c * dvf + vf * c * dvt - ps * dD;
      const double dps = vt * sn * dvf + vf * sn * dvt + pc * dD;
      if (from) {
        dP += k.gft * dpc + k.bft * dps + 2.0 * k.gff * vf * dvf;
        dQ += -k.bft * dpc + k.gft * dps - 2.0 * k.bff * vf * dvf;
      } else {
        dP += k.gtf * dpc - k.btf * dps + 2.0 * k.gtt * vt * dvt;
        dQ += -k.btf * dpc - k.gtf * dps - 2.0 * k.btt * vt * dvt;
      }
    }
    const double vi = bs[BS_V * n_b + i];
    dP += 2.0 * __ldg(n.gsh + i) * vi * dvi;
    dQ -= 2.0 * __ldg(n.bsh + i) * vi * dvi;
    const int g = __ldg(n.bus_gen + i);
    MU[(2 * g) * C + lane] = bs[BS_SRP * n_b + i] * dP;
    MU[(2 * g + 1) * C + lane] = bs[BS_SRQ * n_b + i] * dQ;
  }
  __syncthreads();

  // ---- c2. [H_u; H_x] = K [V; Z] per bus (A7.3), gathering the incident lines
  auto muP = [&](int b) -> double { const int g = __ldg(n.bus_gen + b); return g >= 0 ? MU[(2 * g) * C + lane] : 0.0; };
  auto muQ = [&](int b) -> double { const int g = __ldg(n.bus_gen + b); return g >= 0 ? MU[(2 * g + 1) * C + lane] : 0.0; };
  for (int i = team; i < n_b; i += nteam) {
    const double dvi = dv(i), dthi = dth(i);
    double hv = 0.0, hth = 0.0;
    for (int e = __ldg(n.inc_ptr + i); e < __ldg(n.inc_ptr + i + 1); ++e) {
      const int l = __ldg(n.inc_line + e);
      const int f = __ldg(n.lf + l), t = __ldg(n.lt + l);
      const bool from = f == i;
      const int o = from ? t : f;
      const double dvo = dv(o), dtho = dth(o);
      const Coef k = coef(n, l);
      const double vf = ls[LS_VF * n_l + l], vt = ls[LS_VT * n_l + l];
      const double c = ls[LS_C * n_l + l], sn = ls[LS_S * n_l + l];
      const double dvf = from ? dvi : dvo, dvt = from ? dvo : dvi;
      const double dD = from ? dthi - dtho : dtho - dthi;
      const double pc = vf * vt * c, ps = vf * vt * sn;
      // dψ = J_ψ d
      const double dpc = vt * c * dvf + vf * c * dvt - ps * dD;
      const double dps = vt * sn * dvf + vf * sn * dvt + pc * dD;
      // ds = L_line dψ
      const double dspf = k.gft * dpc + k.bft * dps + 2.0 * k.gff * vf * dvf;
      const double dsqf = -k.bft * dpc + k.gft * dps - 2.0 * k.bff * vf * dvf;
      const double dspt = k.gtf * dpc - k.btf * dps + 2.0 * k.gtt * vt * dvt;
      const double dsqt = -k.btf * dpc - k.gtf * dps - 2.0 * k.btt * vt * dvt;
      const double spf = ls[LS_SPF * n_l + l], sqf = ls[LS_SQF * n_l + l];
      const double spt = ls[LS_SPT * n_l + l], sqt = ls[LS_SQT * n_l + l];
      // dH = 2(s_p ds_p + s_q ds_q);  ḡ_s = 2ŷ⊙ds + 2 s ⊙ (Σ_h dH)
      const double sgf = ls[LS_SGF * n_l + l] * 2.0 * (spf * dspf + sqf * dsqf);
      const double sgt = ls[LS_SGT * n_l + l] * 2.0 * (spt * dspt + sqt * dsqt);
      const double y2f = ls[LS_Y2F * n_l + l], y2t = ls[LS_Y2T * n_l + l];
      // end efforts e = ḡ_s + μ_A (M's line columns equal L_line's, R4)
      const double efp = y2f * dspf + 2.0 * spf * sgf + muP(f);
      const double efq = y2f * dsqf + 2.0 * sqf * sgf + muQ(f);
      const double etp = y2t * dspt + 2.0 * spt * sgt + muP(t);
      const double etq = y2t * dsqt + 2.0 * sqt * sgt + muQ(t);
      // ḡ_ψ = L_lineᵀ ḡ_s + Mᵀ μ_A
      const double gc = k.gft * efp - k.bft * efq + k.gtf * etp - k.btf * etq;
      const double gs = k.bft * efp + k.gft * efq - k.btf * etp - k.gtf * etq;
      // Σ_k w̄_k ∇²ψ_k d (line-local 4×4)
      const double wc = ls[LS_WC * n_l + l], ws = ls[LS_WS * n_l + l];
      const double hD = wc * (-vt * sn * dvf - vf * sn * dvt - pc * dD) + ws * (vt * c * dvf + vf * c * dvt - ps * dD);
      const double jth = -ps * gc + pc * gs;
      if (from) {
        hv += vt * c * gc + vt * sn * gs + 2.0 * vf * (k.gff * efp - k.bff * efq)
            + wc * (c * dvt - vt * sn * dD) + ws * (sn * dvt + vt * c * dD);
        hth += jth + hD;
      } else {
        hv += vf * c * gc + vf * sn * gs + 2.0 * vt * (k.gtt * etp - k.btt * etq)
            + wc * (c * dvf - vf * sn * dD) + ws * (sn * dvf + vf * c * dD);
        hth -= jth + hD;
      }
    }
    const double vi = bs[BS_V * n_b + i];
    hv += bs[BS_WD2 * n_b + i] * dvi + 2.0 * vi * (__ldg(n.gsh + i) * muP(i) - __ldg(n.bsh + i) * muQ(i));
    hv += bs[BS_SXV * n_b + i] * dvi;
    hth += bs[BS_SXT * n_b + i] * dthi;
    const int pt = __ldg(n.bus_pth + i), pv = __ldg(n.bus_pv + i);
    if (pt >= 0) Y[pt * C + lane] = hth;
    if (pv >= 0) Y[pv * C + lane] = hv;
    else Hs[__ldg(n.u_v + i) * C + lane] = hv;
  }
  for (int g = team; g < n.n_g; g += nteam) {  // objective curvature on explicit p_g
    const int up = __ldg(n.u_p + g);
    if (up >= 0) Hs[up * C + lane] = 2.0 * __ldg(n.c_quad + g) * vdir(up);
  }
  __syncthreads();

  // ---- d. adjoint solve Ψ̃ = L^{-T} U^{-T} H̃_x (A7.4)
  sweep_UT<C>(n, lu, luT, Y, lane, team, nteam);
  sweep_LT<C>(n, luT, Y, lane, team, nteam);

  // ---- e. K̂V = H_u − (P G_u)ᵀ Ψ̃ (A7.5, R11)
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

}  // namespace

int pick_tile_cols(int n_x, int total_cols) {
  // Enough CTAs to fill 148 SMs twice, wide tiles when the work allows.
  if (total_cols >= 32 * 296) return 32;
  if (total_cols >= 16 * 296) return 16;
  return 8;
}

int launch_reduce(const DevNet& n, const Work& w, int C, int n_scen, const double* V, int col0,
                  int N, double* KV, cudaStream_t st) {
  dim3 grid((N + C - 1) / C, n_scen);
  switch (C) {
    case 32: k_reduce<32><<<grid, kRedThreads, 0, st>>>(n, w, n_scen, V, col0, N, KV); break;
    case 16: k_reduce<16><<<grid, kRedThreads, 0, st>>>(n, w, n_scen, V, col0, N, KV); break;
    default: k_reduce<8><<<grid, kRedThreads, 0, st>>>(n, w, n_scen, V, col0, N, KV); break;
  }
  return 1;
}

}  // namespace pf
