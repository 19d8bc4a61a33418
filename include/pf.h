/*
 * pf.h — C-ABI of the B200-native batched reduced-Hessian hot path of the
 * condensed (linearize-then-reduce) reduced-space IPM for ACOPF
 * (Pacaud et al., arXiv 2203.11875; citations "P:Lnnn" are lines of the
 * paper text /root/reference/PAPER.md, "§8" refers to SURVEY.md).
 *
 * Conventions
 *   - All floating point is IEEE fp64; all indices int32, 0-based.
 *   - Complex inputs are interleaved (re, im) pairs.
 *   - [host] pointers are read during the call only.  Every other array
 *     pointer is a DEVICE pointer on the handle's device (e.g. a torch CUDA
 *     tensor's data_ptr), used stream-ordered on `stream` (a cudaStream_t;
 *     NULL = legacy default stream); the call returns after enqueueing.
 *   - Batched arrays are [n_scen][...] contiguous, last index fastest.
 *   - Variable partition:
 *       x = [θ_i : i ≠ ref ascending ; v_i : i ∈ PQ ascending]        (n_x)
 *       u = [v_i : i ∈ B_g ascending ; p_g : g ≠ g_ref ascending]      (n_u)
 *       g rows = x rows (row of θ_i is P_i, row of v_i is Q_i)
 *       y / Σ_s rows = [r ; h], r = [P_ref ; Q_ref ; Q_i : i ∈ PV ascending]
 *       (P:L226–253), h = [H^f_l : F_l > 0 ; H^t_l : F_l > 0].
 *   - Ownership: the caller owns every array argument.  The handle owns the
 *     device copies of the network, patterns, ordering, level sets, the
 *     per-scenario LU numeric storage and all workspaces, sized by
 *     max_batch × max_scen at build: no device allocation happens after
 *     pf_build_network, so every compute call is CUDA-graph capturable.
 *   - Errors: argument/size/topology errors are detected on the host and
 *     return non-PF_OK with nothing enqueued.  Numerical failures never
 *     abort: they are written to per-scenario device `info` arrays (LAPACK
 *     convention).  CUDA errors return PF_ERR_CUDA; pf_last_error() explains.
 *   - A handle is not thread-safe; one handle serves one device / rank.
 */
#ifndef PF_H
#define PF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_net pf_net; /* opaque handle */

typedef enum {
  PF_OK = 0,
  PF_ERR_ARG = 1,       /* bad pointer / size / negative count */
  PF_ERR_TOPOLOGY = 2,  /* no/invalid ref bus, gen bus with != 1 generator (R21),
                           out-of-range index, self-loop, disconnected grid */
  PF_ERR_CAPACITY = 3,  /* N > max_batch or n_scen > max_scen; at build: a filled-LU row too long
                           for k_lu's SMEM row workspace (pf_build_error says by how much) */
  PF_ERR_CUDA = 4,      /* CUDA runtime error (see pf_last_error) */
  PF_ERR_STATE = 5      /* call order violated (e.g. no pf_jacobian before a reduction) */
} pf_status;

typedef struct {
  int32_t n_b, n_l, n_g;          /* buses, lines, generators                  */
  int32_t n_x, n_u, m, n_r, n_h;  /* partition sizes, m = n_r + n_h            */
  int32_t ref_bus, ref_gen;
  int32_t nnz_gx, nnz_gu, nnz_a;  /* CSR patterns of G_x, G_u, A (§8.0)         */
  int32_t nnz_lu;                 /* filled pattern of P G_x Pᵀ = L U           */
  int32_t n_blocks;               /* bus blocks (θ_i[, v_i]) of the ordering    */
  int32_t n_levels_l, n_levels_u; /* block level sets of the L / U sweeps       */
  int32_t max_batch, max_scen, tile_cols;
  /* sparse right-hand sides (device handles; 0 for host-only ones): rows the
     forward L sweep visits, summed over the canonical column tiles of width
     tile_cols; rows the adjoint Lᵀ sweep visits (ancestors of G_u's rows);
     distinct rows of G_u (where the projection G_uᵀΨ reads Ψ). */
  int32_t reach_rows_l, reach_rows_ua, gu_rows;
  /* LU schedule (A5): rows of the dense front (levels >= front_level, at most
     96, eliminated as one dense LU in SMEM); levels < lu_cut_level run as
     per-warp-pair subtree walks over lu_pairs pairs (PF_LU_SUBTREE_*).     */
  int32_t front_level, front_rows, lu_cut_level, lu_pairs;
} pf_dims;

/* Host copies of the integer structure, for bit-exact tests (R19, P15). */
typedef enum {
  PF_X_THETA = 0,   /* [n_b] x index of θ_i, -1 for the ref bus            */
  PF_X_V = 1,       /* [n_b] x index of v_i, -1 at generator buses          */
  PF_U_V = 2,       /* [n_b] u index of v_i, -1 at PQ buses                 */
  PF_U_P = 3,       /* [n_g] u index of p_g, -1 for the ref generator       */
  PF_GX_PTR = 4,    /* [n_x+1] CSR of G_x (rows = g rows, cols = x)          */
  PF_GX_IDX = 5,    /* [nnz_gx]                                              */
  PF_GU_PTR = 6,    /* [n_x+1] CSR of G_u (cols = u)                         */
  PF_GU_IDX = 7,    /* [nnz_gu]                                              */
  PF_A_PTR = 8,     /* [m+1] CSR of A = ∂[r;h]/∂[u;x] (cols = [u;x])          */
  PF_A_IDX = 9,     /* [nnz_a]                                               */
  PF_BUS_ORDER = 10,/* [n_blocks] bus elimination order (R18 rule)          */
  PF_PERM = 11,     /* [n_x] perm[k] = x index at permuted position k        */
  PF_BLOCK_PTR = 12,/* [n_blocks+1] permuted rows of each block              */
  PF_LU_PTR = 13,   /* [n_x+1] CSR of the filled pattern (permuted coords)   */
  PF_LU_IDX = 14,   /* [nnz_lu]                                              */
  PF_LEVEL_L_PTR = 15, /* [n_levels_l+1]                                    */
  PF_LEVEL_L_BLK = 16, /* [n_blocks] blocks by forward level, ascending      */
  PF_LEVEL_U_PTR = 17, /* [n_levels_u+1]                                    */
  PF_LEVEL_U_BLK = 18, /* [n_blocks] blocks by backward level, ascending     */
  PF_FRONT_ROW = 19,   /* [front_rows] permuted rows of the dense LU front     */
  PF_LU_SUBTREE_PTR = 20, /* [lu_pairs+1] per warp pair: its bottom blocks in  */
  PF_LU_SUBTREE_BLK = 21, /* PF_LU_SUBTREE_BLK[ptr[t] … ptr[t+1]), postorder   */
  PF_LU_LEVEL_BLK = 22 /* [n_blocks] PF_LEVEL_L_BLK, each level longest rows first */
} pf_structure;

/*
 * pf_build_network — analyse a network once per topology (A1, §8(a)).
 * Arguments follow the paper's problem statement: C_f, C_t as line_from /
 * line_to, the π-model vectors Y_ff, Y_ft, Y_tf, Y_tt and the
 * shunts Y_sh, C_g as gen_bus, base loads p_d, q_d
 * (P:L73–74), line limits F_max (<= 0 means no H rows for the line),
 * quadratic cost c_quad, c_lin (c_{i,1}, c_{i,2} of P:L187).
 * Host work: validation, index maps, CSR patterns, the static symmetric
 * bus-level minimum-degree ordering (R18), the symbolic LU and its level
 * sets (the paper's first KLU factorization).
 *   [host] line_from, line_to: n_l;  Y_ff..Y_tt: 2*n_l;  Y_sh: 2*n_b;
 *   [host] gen_bus: n_g;  p_d, q_d: n_b;  F_max: n_l;  c_quad, c_lin: n_g.
 * max_batch = most directions per pf_reduced_hessian_batch call,
 * max_scen = most scenarios per call; device = CUDA ordinal, or -1 for a
 * host-only handle (structure analysis only: pf_query / pf_get_structure
 * work, every compute call returns PF_ERR_STATE; used by CPU-only tests).
 * Returns PF_ERR_TOPOLOGY for an invalid grid (no handle is created).
 */
pf_status pf_build_network(int32_t n_b, int32_t n_l, int32_t n_g,
                           const int32_t *line_from, const int32_t *line_to,
                           const double *Y_ff, const double *Y_ft,
                           const double *Y_tf, const double *Y_tt,
                           const double *Y_sh, const int32_t *gen_bus,
                           int32_t ref_bus, const double *p_d,
                           const double *q_d, const double *F_max,
                           const double *c_quad, const double *c_lin,
                           int32_t max_batch, int32_t max_scen, int32_t device,
                           pf_net **out);

/*
 * pf_build_network_ex — pf_build_network with an explicit direction-tile
 * width of the reduction kernels: tile_cols ∈ {8, 16, 32, 64} directions per
 * CTA tile, or 0 = automatic (what pf_build_network does: the widest tile that
 * still gives ≥ 2 CTAs per SM for max_batch × max_scen directions).  Results
 * are bit-identical for every tile width.  PF_ERR_ARG for any
 * other value.
 */
pf_status pf_build_network_ex(int32_t n_b, int32_t n_l, int32_t n_g,
                              const int32_t *line_from, const int32_t *line_to,
                              const double *Y_ff, const double *Y_ft,
                              const double *Y_tf, const double *Y_tt,
                              const double *Y_sh, const int32_t *gen_bus,
                              int32_t ref_bus, const double *p_d,
                              const double *q_d, const double *F_max,
                              const double *c_quad, const double *c_lin,
                              int32_t max_batch, int32_t max_scen, int32_t device,
                              int32_t tile_cols, pf_net **out);

void pf_destroy(pf_net *net);
pf_status pf_query(const pf_net *net, pf_dims *out /* [host] */);
/* Copy one integer structure array (sizes in pf_structure) to [host] out. */
pf_status pf_get_structure(const pf_net *net, int32_t which, int32_t *out);
const char *pf_last_error(const pf_net *net);
/* Pointers to the handle's own error text when no handle exists. */
const char *pf_build_error(void);

/*
 * pf_eval_constraints — A2/A3: ψ basis (one sincos per line, P:L173–179,
 * P:L1133–1135), power balance G = Mψ + [p_d − C_g p_g ; q_d − C_g q_g]
 * (eq. base:powerflow), line flows s = L_line ψ (eq.
 * base:powerlines, with readings R1–R3) and line limits
 * H = s_p² + s_q² (eq. linelimitsvec).
 *   v, theta: [n_scen][n_b];  p_g, q_g: [n_scen][n_g];
 *   p_d, q_d: [n_scen][n_b] or NULL = the base loads;
 *   out G: [n_scen][2 n_b] ([P rows ; Q rows], bus order);
 *   out H: [n_scen][2 n_l] ([H^f ; H^t], every line) or NULL;
 *   out s_flow: [n_scen][4][n_l] (s_p^f, s_q^f, s_p^t, s_q^t) or NULL.
 */
pf_status pf_eval_constraints(pf_net *net, int32_t n_scen, const double *v,
                              const double *theta, const double *p_g,
                              const double *q_g, const double *p_d,
                              const double *q_d, double *G, double *H,
                              double *s_flow, void *stream);

/*
 * pf_jacobian — A4/A5: Jacobian values through the ψ chain (P:L513–545,
 * P:L1137–1141) and the numeric LU refactorization P G_x Pᵀ = L U with the
 * fixed pattern and static pivots of pf_build_network (SpRF, P:L1110–1116,
 * P:L1189–1193).  The factors stay in the handle for the next
 * pf_reduced_hessian_batch at the same point.
 *   v, theta: [n_scen][n_b];
 *   out Gx_val [n_scen][nnz_gx], Gu_val [n_scen][nnz_gu], A_val
 *   [n_scen][nnz_a] in the pf_get_structure patterns; each may be NULL.
 *   out info [n_scen]: 0, or k+1 for the first permuted pivot k with
 *   |u_kk| < 1e-12 · max_j |(P G_x Pᵀ)_kj| (R18) or non-finite.
 */
pf_status pf_jacobian(pf_net *net, int32_t n_scen, const double *v,
                      const double *theta, double *Gx_val, double *Gu_val,
                      double *A_val, int32_t *info, void *stream);

/*
 * pf_reduced_hessian_batch — A6/A7: N reduced-Hessian–vector products at
 * once by the batched adjoint-adjoint algorithm (with R11):
 *   Z = −G_x^{-1}(G_u V);  [H_u; H_x] = K [V; Z];  Ψ = G_x^{-T} H_x;
 *   K̂ V = H_u − G_uᵀ Ψ,
 * K = ∇²ℒ + AᵀΣ_sA + blkdiag(0, Σ_x) (R14), ℒ = f + λᵀg
 * + yᵀ[r; h], f with the implicit p_ref (R8).  K is never formed: K·[V;Z]
 * is evaluated matrix-free through ψ.  Uses the point and the LU factors of
 * the last successful pf_jacobian (factorize once per
 * iteration, reuse for every right-hand side).
 *   v, theta: the SAME device arrays passed to that pf_jacobian (contents
 *   unchanged since), or NULL = that point; other pointers → PF_ERR_STATE,
 *   as is a call with more scenarios than that pf_jacobian factorized;
 *   p_d: [n_scen][n_b] or NULL = base loads
 *   (only p_d[ref] enters, through p_ref);
 *   lambda: [n_scen][n_x];  y: [n_scen][m];
 *   sigma_s: [n_scen][m] or NULL (= 0);  sigma_x: [n_scen][n_x] or NULL;
 *   V: [n_scen][N][n_u] directions, or NULL = unit columns col0..col0+N−1;
 *   out KV: [n_scen][N][n_u] = K̂ V (each direction a contiguous column, so
 *   N = n_u, col0 = 0 yields K̂ column-major).
 * Stream semantics: ordered on `stream`; internally the A6 prep kernels run on
 * the handle's helper stream, forked from and joined back into `stream` with
 * events (so the call is CUDA-graph capturable and a single handle must not be
 * used from two host threads at once).
 */
pf_status pf_reduced_hessian_batch(pf_net *net, int32_t n_scen,
                                   const double *v, const double *theta,
                                   const double *p_d, const double *lambda,
                                   const double *y, const double *sigma_s,
                                   const double *sigma_x, const double *V,
                                   int32_t col0, int32_t N, double *KV,
                                   void *stream);

/*
 * pf_condensed_kkt_solve — A9: K_cond = sym(K̂) + diag(Σ_u) + δ_w I
 * (Theorem 2 with R9; regularisation P:L1341–1342),
 * sym(K̂) = (K̂ + K̂ᵀ)/2; blocked FP64 Cholesky K_cond = L Lᵀ (cusolver's
 * role in P:L1339–1341; success certifies the inertia, Theorem 3
 * P:L856–866) and the solve L Lᵀ p = b.
 *   K: [n_scen][n_u][n_u] column-major; in K̂, out L in the lower triangle
 *   (strict upper triangle zeroed) — for the scenarios that factorized; a
 *   scenario whose factorization failed keeps its K̂ (so it can be retried);
 *   sigma_u: [n_scen][n_u] or NULL;  delta_w: scalar shift;
 *   rhs: [n_scen][nrhs][n_u]; in b, out K_cond^{-1} b (untouched for a
 *   scenario whose factorization failed); nrhs >= 0;
 *   out info [n_scen]: 0, or j+1 for the first column whose pivot is <= 0
 *   or non-finite.
 */
pf_status pf_condensed_kkt_solve(pf_net *net, int32_t n_scen, double *K,
                                 const double *sigma_u, double delta_w,
                                 double *rhs, int32_t nrhs, int32_t *info,
                                 void *stream);

/*
 * ---- NEXT-1: condensed right-hand side and step recovery ----
 * One LinRed iteration's remaining linear algebra (Algorithm 1)
 * around pf_condensed_kkt_solve, at the point of the last pf_jacobian (v,
 * theta as in pf_reduced_hessian_batch) with the multipliers and barrier
 * diagonals of the reduction (lambda, y, sigma_s, sigma_x, p_d as there).
 *   r: [n_scen][n_u + n_x + m + n_x + m] device — the right-hand side
 *   (r₁, r₂, r₃, r₄, r₅) of eq. kktmatrix:normal, blocks
 *   ordered like the unknowns (p_u, p_x, p_s, p_λ, p_y); K_aug p = −r.
 *
 * pf_condensed_rhs — Theorem 1's r̂₁, r̂₂, r̂₃ and Theorem 2's
 * right-hand side with reading R10 (sign of the r̂₂ terms):
 *   b = −(r̂₁ + Â_uᵀ Σ_s r̂₃ + Â_uᵀ r̂₂),   K_cond p_u = b;
 * computed matrix-free as ONE direction of the HVP pipeline per scenario
 * (DESIGN.md §"Step recovery"), never forming Â_u.
 *   out b: [n_scen][n_u] (pass it as pf_condensed_kkt_solve's rhs).
 *
 * pf_recover_step — Algorithm 1's dual, slack, state and adjoint steps:
 *   p_y = Σ_s(Â_u p_u + r̂₃ + Σ_s⁻¹ r̂₂),  p_s = Σ_s⁻¹(p_y − r̂₂),
 *   p_x = −G_x⁻¹(r₄ + G_u p_u),
 *   p_λ = −G_x⁻ᵀ(r₂ + A_xᵀ p_y + W_xu p_u + (W_xx + Σ_x) p_x).
 *   p_u: [n_scen][n_u] (the condensed solve's solution);
 *   out p: [n_scen][n_u + n_x + m + n_x + m] = (p_u, p_x, p_s, p_λ, p_y).
 * sigma_s must be non-NULL for the recovery when m > 0 (Theorem 2 needs Σ_s
 * nonsingular); NULL is read as 0 elsewhere.
 */
pf_status pf_condensed_rhs(pf_net *net, int32_t n_scen, const double *v,
                           const double *theta, const double *p_d,
                           const double *lambda, const double *y,
                           const double *sigma_s, const double *sigma_x,
                           const double *r, double *b, void *stream);
pf_status pf_recover_step(pf_net *net, int32_t n_scen, const double *v,
                          const double *theta, const double *p_d,
                          const double *lambda, const double *y,
                          const double *sigma_s, const double *sigma_x,
                          const double *r, const double *p_u, double *p,
                          void *stream);

/*
 * ---- NEXT-2: power flow, first-order adjoint, reduced gradient ----
 * pf_power_flow — the RedLin projection step (Algorithm 2):
 * Newton–Raphson on g(x, u) = 0 for every scenario at once, x ← x − G_x⁻¹g
 * with the A4/A5 Jacobian and LU and the k_fwd sweeps (N = 1), until
 * ‖g‖∞ ≤ tol (the paper's 1e-10) or max_iter steps.
 *   v, theta: [n_scen][n_b] device, IN the start point (u = v at generator
 *   buses and p_g fixed), OUT the solution (state entries updated in place);
 *   p_g, q_g, p_d, q_d as pf_eval_constraints (q_g may be NULL: it enters no
 *   g row); out [host] iters, resid (final ‖g‖∞), info: 0 converged, −1 no
 *   convergence in max_iter (or NaN), k+1 singular Jacobian (R18 pivot k).
 *   Each may be NULL.  Synchronizes the stream once per iteration (host
 *   convergence test; not graph-capturable).  Ends with a factorization at
 *   the final point: pf_reduced_hessian_batch / pf_reduced_gradient /
 *   pf_condensed_rhs may follow with these v, theta arrays.
 *
 * pf_reduced_gradient — the adjoint step and the reduced gradient
 * (Algorithm 2; Theorem "Reduced derivatives"):
 *   ∇_z ℓ = ∇_z(f + yᵀ[r; h]) (f with the implicit p_ref, R8),
 *   λ = −G_x⁻ᵀ ∇_x ℓ,   ∇_u ℓ_r = ∇_u ℓ − G_uᵀ G_x⁻ᵀ ∇_x ℓ.
 * At the point of the last pf_jacobian / pf_power_flow (v, theta as in
 * pf_reduced_hessian_batch).
 *   p_g: [n_scen][n_g]; p_d: [n_scen][n_b] or NULL; y: [n_scen][m];
 *   out lambda: [n_scen][n_x] or NULL; out grad: [n_scen][n_u].
 */
pf_status pf_power_flow(pf_net *net, int32_t n_scen, double *v, double *theta,
                        const double *p_g, const double *q_g,
                        const double *p_d, const double *q_d, double tol,
                        int32_t max_iter, int32_t *iters, double *resid,
                        int32_t *info, void *stream);
pf_status pf_reduced_gradient(pf_net *net, int32_t n_scen, const double *v,
                              const double *theta, const double *p_g,
                              const double *p_d, const double *y,
                              double *lambda, double *grad, void *stream);

/*
 * ---- NEXT-3: inertia-correcting regularization ----
 * pf_condensed_kkt_solve_reg — pf_condensed_kkt_solve inside the paper's
 * regularization loop ("if the factorization fails, we apply
 * a primal regularization δ_w and refactorize"; Theorem 3: the
 * Cholesky succeeds iff K_cond is positive definite iff K_aug has the
 * inertia (n_x+n_u+m, n_x+m, 0), so success certifies a descent direction).
 * Trial 1 factorizes every scenario with δ_w = delta_init; a scenario that
 * fails is retried with δ_w = delta_first (if its δ_w was 0) or growth × its
 * δ_w, while that stays ≤ delta_max.  Each retry factorizes all failed
 * scenarios of the call at once (one DAG launch per trial, the others
 * untouched).  Arguments as pf_condensed_kkt_solve; delta_init ≥ 0,
 * delta_first > 0, growth > 1, delta_max ≥ delta_init.
 *   out [host] delta_out [n_scen]: the δ_w of the last trial (the accepted one
 *   when info = 0); trials [n_scen]: factorizations attempted; info [n_scen]:
 *   0, or the last trial's first failing column + 1.  Each may be NULL.
 * Synchronizes the stream once per trial (not graph-capturable).
 */
pf_status pf_condensed_kkt_solve_reg(pf_net *net, int32_t n_scen, double *K,
                                     const double *sigma_u, double delta_init,
                                     double delta_first, double growth,
                                     double delta_max, double *rhs,
                                     int32_t nrhs, double *delta_out,
                                     int32_t *trials, int32_t *info,
                                     void *stream);

/* Number of kernels this handle has launched so far (bench evidence). */
int64_t pf_launch_count(const pf_net *net);

/*
 * Instrumentation (bench / profiling only).  pf_profile(net, 1) makes the
 * compute calls record CUDA events on their stream around the hot kernels;
 * pf_kernel_times writes the last calls' per-kernel milliseconds, in the
 * order k_fwd, k_mu, k_hvp, k_adj (pf_reduced_hessian_batch), k_lu
 * (pf_jacobian), k_proj (pf_reduced_hessian_batch) and k_chol_dag
 * (pf_condensed_kkt_solve[_reg], its first trial), synchronizing on the
 * events; returns how many were written (0 when profiling is off; at most 7).
 */
pf_status pf_profile(pf_net *net, int32_t enable);
int32_t pf_kernel_times(pf_net *net, float *ms /* [host] cap */, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* PF_H */
