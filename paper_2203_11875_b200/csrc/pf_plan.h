// pf_plan.h — host-side structural plan of one network (A1 of SURVEY §8(a)).
// Everything here is integer structure computed once per topology on the host,
// the B200 analogue of the paper's first (KLU, CPU) factorization whose pattern
// and pivots the GPU then reuses.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pf {

#ifndef PF_FRONT_MAX
#define PF_FRONT_MAX 96
#endif
#ifndef PF_LU_IMB
#define PF_LU_IMB 30
#endif
constexpr int kFrontMax = PF_FRONT_MAX;  // rows of the dense LU front (k_lu: F (F + 1) doubles of SMEM)
constexpr int kLuPairs = 16 * 8;         // k_lu warp pairs: a 16-CTA cluster of 512-thread CTAs

struct Plan {
  int n_b = 0, n_l = 0, n_g = 0, n_x = 0, n_u = 0, m = 0, n_r = 0, n_h = 0;
  int r0 = -1, g_r = -1, n_gb = 0;

  // partition
  std::vector<int> x_th, x_v, u_v, u_p, bus_gen;
  std::vector<int> bus_rP, bus_rQ;    // index of P_i / Q_i in r (or -1)
  std::vector<int> line_hf, line_ht;  // index of H^f_l / H^t_l in h (or -1)
  std::vector<int> h_line, h_end;     // per h row

  // bus -> incident lines (ascending line index; deterministic gathers)
  std::vector<int> inc_ptr, inc_line;

  // J_bus: ∂[P_i; Q_i]/∂z, z = [u; x]; rows 0..n_b-1 = P, n_b..2n_b-1 = Q.
  // P_i and Q_i share one column pattern: vars of i and its neighbours.
  std::vector<int> jb_ptr, jb_idx;         // CSR, 2 n_b rows
  std::vector<int> jb_self_th, jb_self_v;  // per bus: offset of own θ / v within its rows (-1)
  std::vector<int> inc_off_th, inc_off_v;  // per incidence: offset of the other bus's θ / v

  // G_x, G_u, A patterns + gather maps from J_bus values (-1: constant -1, p_g)
  std::vector<int> gx_ptr, gx_idx, gx_src;
  std::vector<int> gu_ptr, gu_idx, gu_src;
  std::vector<int> a_ptr, a_idx, a_src;    // r rows: src = J_bus index; h rows: -1
  std::vector<int> ah_off;                 // per h row: 4 offsets (v_f, v_t, θ_f, θ_t) within its A row

  // ordering and symbolic LU of P G_x Pᵀ (R18)
  std::vector<int> bus_order, perm, iperm, blk_ptr, blk_bus, row_blk;
  std::vector<int> lu_ptr, lu_idx, lu_diag, lu_src, lu_tpos;
  std::vector<int> upd_ptr, upd_dst;       // per LU entry: range in upd_dst (L entries only); dst = offset in the row
  std::vector<int> upd_src;                // … and the lu index of the U value u_kj each update reads
  int lu_maxlen = 0;                       // longest row of the filled pattern
  std::vector<int> levL_ptr, levL_blk, levU_ptr, levU_blk;
  std::vector<double> row_scale_dummy;

  // G_u in permuted row coordinates, by column (CSC) and by row (CSR)
  std::vector<int> guc_ptr, guc_row, guc_src;   // src into Gu_val (CSR order)
  std::vector<int> gur_ptr, gur_col, gur_src;

  // bus -> permuted slab rows
  std::vector<int> bus_pth, bus_pv;
  std::vector<int> hvp_bus;   // elimination order, reference bus last

  // k_lu schedule (lu_schedule): dense front rows (levels ≥ fr_lev, ascending), bottom subtrees
  // per warp pair below lu_lev0 (lu_p1_blk[lu_p1_ptr[t] …]), per-level order longest rows first
  int fr_lev = 0, lu_lev0 = 0;
  std::vector<int> fr_row, lu_p1_blk, lu_p1_ptr, lu_lev_blk;
};

void lu_schedule(Plan& P);

// Returns "" on success, else an error message; *topology is set when the
// failure is a topology error (PF_ERR_TOPOLOGY) rather than an argument error.
std::string build_plan(int n_b, int n_l, int n_g, const int32_t* line_from,
                       const int32_t* line_to, const int32_t* gen_bus,
                       int ref_bus, const double* F_max, Plan& P,
                       bool* topology);

}  // namespace pf
