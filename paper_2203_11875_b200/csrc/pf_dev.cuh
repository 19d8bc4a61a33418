// pf_dev.cuh — device-side views of the network plan and per-handle workspaces.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace pf {

// A set of 2×2 bus blocks for the SMEM-staged block-SpMM kernel (pf_reduce.cu k_blk): per
// output bus (position p of `out`) the blocks of its neighbours j, the bus itself first; the
// chunks of consecutive output buses whose distinct rows fit the SMEM budget; and per chunk the
// rows it stages (slab row r < n_x of the direction tile, or μ_A row n_x + 2g / + 1).
struct BlkSet {
  const int *ptr;        // [nout + 1] blocks of output position p
  const int4 *meta;      // [nblk] {slot of θ_j (−1: ref), slot of v_j or −1−u(v_j), slot of μ^P_j (μ^Q next) or −1, 0}
  const int *self, *nbr; // [nblk] bus i, neighbour j (the per-scenario prep)
  const int2 *jt;        // [nblk] hb only: offsets of θ_i, v_i in J_bus rows P_j / Q_j of a generator bus j
  const int4 *out;       // [nout] hb: {bus, θ row, v row or −1−u, gen}; mb: {bus, gen, 0, 0}
  const int *ck_ptr;     // [nchunk + 1] output positions per chunk
  const int *st_ptr, *st_row;  // [nchunk + 1], [nstage]
  int nout, nblk, nchunk, st_max, blk_max, ck_max;
};

// Network-level device data (read-only, shared by all scenarios).
struct DevNet {
  int n_b, n_l, n_g, n_x, n_u, m, n_r, n_h, r0, g_r, n_gb, nblk;
  int nnz_jb, nnz_gx, nnz_gu, nnz_a, nnz_lu;
  int nlevL, nlevU;
  const int *lf, *lt;           // [n_l] C_f, C_t
  const double *coef;           // [8][n_l]: g_ff b_ff g_ft b_ft g_tf b_tf g_tt b_tt
  const double *gsh, *bsh;      // [n_b] Y_sh
  const int *gen_bus, *bus_gen; // [n_g], [n_b]
  const double *c_quad, *c_lin; // [n_g]
  const double *p_d0, *q_d0;    // [n_b] base loads
  const int *x_th, *x_v, *u_v, *u_p, *bus_rP, *bus_rQ, *line_hf, *line_ht;
  const int *inc_ptr, *inc_line, *inc_off_th, *inc_off_v;
  const int *jb_ptr, *jb_self_th, *jb_self_v;
  const int *gx_src, *gu_src, *a_ptr, *a_src, *ah_off, *h_line, *h_end;
  const int *blk_ptr, *lu_ptr, *lu_idx, *lu_diag, *lu_src, *lu_tpos, *upd_ptr, *upd_dst, *upd_src;
  const int *levL_ptr, *levL_blk, *levU_ptr, *levU_blk;
  const int *guc_ptr, *guc_row, *guc_src, *gur_ptr, *gur_col, *gur_src;
  const int *bus_pth, *bus_pv;
  const int *gbus;              // [n_gb] generator buses ascending (the r buses)
  const int4 *rowmeta;          // [n_x] {lu_ptr[r], lu_diag[r], lu_ptr[r+1], block of r}
  const int *hvp_bus;           // [n_b] buses in elimination order, the reference bus last
  const int4 *taskL, *taskU;    // [n_blocks] sweep tasks in level order (pf_reduce.cu sweep()): {r0|two<<31, segment, m, 0}
  const int2 *sw_src;           // [nsw] source of each sweep-stream slot (pf_api.cu, packed by k_lu)
  int nsw;
  // Sparse right-hand sides (Gilbert–Peierls reach): for unit directions the L sweep of
  // canonical column tile t (columns [tC, tC+C)) only visits the blocks on the
  // elimination-tree paths from G_u's nonzeros to the root; the Lᵀ sweep of the
  // adjoint only needs the ancestors of G_u's rows (the projection reads Ψ there).
  const int4 *taskLr;           // per canonical tile: its L tasks in level order (concatenated)
  const int *levLr_ptr;         // [ntc][nlevL+1] absolute offsets into taskLr
  const unsigned *rowbm;        // [ntc][bmw] bitmap of the tile's reach rows (permuted)
  const int4 *taskUa;           // U-list blocks that are ancestors of a G_u row
  const int *levUa_ptr;         // [nlevU+1]
  int ntc, bmw;
  const int4 *p1_task;          // bottom-subtree schedule of the LOWER sweeps: per team, its subtrees in postorder
  const int *p1_ptr;            // [teams per CTA + 1]
  int p1_lev0;                  // levels < p1_lev0 run from p1_task, the rest level by level
  const int4 *p1r_task;         // per canonical tile: p1_task restricted to the tile's reach blocks
  const int *p1r_ptr;           // [ntc][teams + 1] absolute offsets into p1r_task
  // UPPER sweeps: blocks above the cut by U level (u_top, [nlevU+1] pointers), then the
  // bottom subtrees per team parents-first (u_bot, [teams+1]); ua_*: the same restricted
  // to the ancestors of G_u's rows (the Lᵀ sweep)
  const int4 *u_top, *u_bot, *ua_top, *ua_bot;
  const int *u_top_ptr, *u_bot_ptr, *ua_top_ptr, *ua_bot_ptr;
  // step recovery / Newton (pf_step): permuted slab row <-> x index, the G row
  // (P_i = i, Q_i = n_b + i) of each permuted row, and A by columns (CSC over
  // z = [u; x]: rows and positions in the CSR value array)
  const int *perm, *iperm, *row_g;
  const int *a_cptr, *a_crow, *a_cpos, *a_idx;
  const int *u_gen;             // [n_u] generator of a p_g control, −1 for v controls
  BlkSet hb;                    // k_hvp: K's bus blocks (every bus) + A_rᵀ at generator neighbours
  BlkSet mb;                    // k_mu: ∂(P_g, Q_g)/∂(θ_j, v_j) blocks of the generator buses g
  // Dense front (k_lu): the rows of levels ≥ fr_lev (fr_n ≤ kFrontMax of them, ascending
  // permuted index fr_row; fr_pos[r] = front index of row r or −1).  Their pivots among
  // themselves are eliminated as one dense LU of the front Schur complement in SMEM
  // instead of fr_lev … nlevL−1 cluster-synchronised levels.
  int fr_lev, fr_n;
  // k_lu bottom levels (< lu_lev0): per warp pair of the cluster (lu_nteam of them) its subtrees'
  // blocks in postorder, lu_p1_blk[lu_p1_ptr[t] … lu_p1_ptr[t + 1])
  int lu_lev0, lu_nteam;
  const int *lu_p1_blk, *lu_p1_ptr;
  const int *lu_lev_blk;        // [n_blocks] levL_blk with each level's longest rows first (k_lu)
  const int *fr_row, *fr_pos;
  int C;                        // directions per tile (slab row width)
  int lu_maxlen;                // longest row of the filled LU pattern
};

// Per-scenario point state, SoA.  Line state (LS_*) and bus state (BS_*).
enum { LS_VF, LS_VT, LS_C, LS_S, LS_SPF, LS_SQF, LS_SPT, LS_SQT,
       LS_WC, LS_WS, LS_Y2F, LS_Y2T, LS_SGF, LS_SGT, LS_DF, LS_DT, LS_N };
enum { BS_V, BS_MUP, BS_MUQ, BS_WD2, BS_SRP, BS_SRQ, BS_SXT, BS_SXV, BS_N };
// Per-line K blocks (AoS, 18 doubles = 9 × 16 B): symmetric H (3×3) on
// (v_f, v_t, Δ) and J (4×3) = ∂(s_p^f, s_q^f, s_p^t, s_q^t)/∂(v_f, v_t, Δ).
enum { LB_H00, LB_H01, LB_H02, LB_H11, LB_H12, LB_H22, LB_J, LB_N = LB_J + 12 };

struct Work {
  double* jb;      // [max_scen][nnz_jb]  J_bus values
  double* gu;      // [max_scen][nnz_gu]  G_u values (internal copy)
  double* lu;      // [max_scen][nnz_lu]  LU values (row-wise)
  double2* swA;    // [max_scen][nsw]     sweep streams of L (LOWER) / U (UPPER) segments: {value, bits(column·C)} with
                   //                     1/u_rr for the diagonal, the block scalars {d_A, intra} {d_B, 0} at the end
  double2* swT;    // [max_scen][nsw]     … the same over the transposed values (Uᵀ LOWER / Lᵀ UPPER)
  double2* pkG;    // [max_scen][nnz_gu]  G_u by column (CSC): {value, bits(row*C)} for the projection
  double* rowmax;  // [max_scen][n_x]     pivot threshold scale (R18)
  double* invd;    // [max_scen][n_x]     1 / u_rr of the factorized rows
  double* ls;      // [max_scen][LS_N][n_l]
  double* bs;      // [max_scen][BS_N][n_b]
  double* lblk;    // [max_scen][n_l][LB_N]  line-local K blocks
  double* sflow;   // [max_scen][4][n_l]
  int* info;       // [max_scen] internal pivot info
  double* aval;    // [max_scen][nnz_a]   A values (CSR of pf_get_structure) of the last pf_jacobian
  double* zero;    // [max_scen][n_u + n_x + m]  zeros (V = 0 directions, λ = 0)
  double* gbuf;    // [max_scen][2 n_b]   G of the Newton iterations
  double* res;     // [max_scen]          ‖g‖∞ per scenario (Newton)
  int* active;     // [max_scen]          Newton: 1 while the scenario iterates
  double* hbval;   // [max_scen][hb.nblk][8] per bus block: B (θθ θv vθ vv) of K, then JT (θ←μP θ←μQ v←μP v←μQ)
  double* mbval;   // [max_scen][mb.nblk][8] per generator block: (∂P/∂θ ∂P/∂v ∂Q/∂θ ∂Q/∂v), 4 unused
  int* csidx;      // [max_scen]          regularization retries: caller scenario of each retried one
  double* cdelta;  // [max_scen]          … and its δ_w
  double* slabZ;   // [max_tiles][n_x][C]
  double* slabW;   // [max_tiles][n_x][C]
  double* hu;      // [max_tiles][n_u][C]
  double* mu;      // [max_tiles][n_gb][2][C]
  double* ctile;   // [max_scen][chol_tile_doubles]  packed lower 64×64 tiles of K_cond / L
  int* cflag;      // [max_scen][chol_flag_ints]     tile / forward / backward ready flags
  int* cticket;    // [1 + 1024]                     Cholesky DAG task counter, then per-SM critical-task counts
  double* cy;      // [max_scen][chol_vec_doubles]   forward / backward solve vectors
  int max_tiles;
};

}  // namespace pf
