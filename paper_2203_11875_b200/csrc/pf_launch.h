// pf_launch.h — host launchers of the sm_100a kernels (one per hot-path step).
#pragma once
#include "pf_dev.cuh"
#include "pf_plan.h"

namespace pf {


// A2/A3: line kernel (ψ, flows, H) then bus gather (G).  Returns launches.
int launch_eval(const DevNet& n, const Work& w, int n_scen, const double* v, const double* th,
                const double* p_g, const double* q_g, const double* p_d, const double* q_d,
                double* G, double* H, double* s_flow, cudaStream_t st);

// A4/A5: line state, J_bus values, gathers into G_x/G_u/A, numeric LU + transposed values.
int launch_jacobian(const DevNet& n, const Work& w, int n_scen, const double* v, const double* th,
                    double* Gx, double* Gu, double* A, int* info, cudaStream_t st, int lu_cs,
                    cudaEvent_t* ev = nullptr /* optional: [2] around k_lu */);
// k_lu cluster size supported on the current device (sets k_lu's function attributes there)
int lu_cluster_size(const DevNet& n);
// k_lu's dynamic SMEM (per-warp dense row workspaces of lu_maxlen doubles + staging areas, or the dense front)
size_t lu_smem_bytes(const DevNet& n);

// A6: per-scenario ψ weights w̄ and bus/line state for the HVP.
int launch_prep(const DevNet& n, const Work& w, int n_scen, const double* p_d, const double* lam,
                const double* y, const double* sigma_s, const double* sigma_x, cudaStream_t st);

// A7.1–A7.5 fused: RHS, L/U sweeps, matrix-free K·[V;Z], Uᵀ/Lᵀ sweeps, projection.
int launch_reduce(const DevNet& n, const Work& w, int C, int n_scen, const double* V, int col0,
                  int N, double* KV, cudaStream_t st,
                  cudaEvent_t* ev = nullptr /* optional: [5] around k_fwd, k_mu, k_hvp, k_adj */,
                  cudaEvent_t after_fwd = nullptr /* optional: waited for between k_fwd and k_blk */);

// A9: symmetrize + shift + pack, tile-DAG FP64 Cholesky (DMMA updates) with the solves fused in.
int launch_chol(const DevNet& n, const Work& w, int n_scen, double* K, const double* sigma_u, double delta_w,
                double* rhs, int nrhs, int* info, int* info_ws, cudaStream_t st, int grid_max,
                const int* sidx = nullptr /* [n_scen] caller scenario of each, device */,
                const double* dvec = nullptr /* [n_scen] per-scenario δ_w, device */,
                cudaEvent_t* ev = nullptr /* optional: [2] around the DAG launch(es) */);
// resident k_chol_dag CTAs on the current device (sets its SMEM attribute there)
int chol_grid_max();

// NEXT-1 / NEXT-2 single-direction passes (pf_reduce.cu): what = 0 condensed rhs (out = b),
// 1 step recovery (out = p), 2 reduced gradient (out = ∇f_r, out2 = λ).
int launch_step(int what, const DevNet& n, const Work& w, int C, int n_scen, const double* r, const double* sig_s,
                const double* y, const double* p_g, const double* p_u, double* out, double* out2, cudaStream_t st);
// Newton: ‖g‖∞ of w.gbuf per scenario into w.res; one step x −= G_x⁻¹ g on the active scenarios.
int launch_pf_resid(const DevNet& n, const Work& w, int n_scen, cudaStream_t st);
int launch_newton_step(const DevNet& n, const Work& w, int C, int n_scen, double* v, double* th, cudaStream_t st);

int pick_tile_cols(int n_x, int n_scen_x_N);
int hvp_stage_rows(int C);  // slab rows one k_hvp chunk may stage in SMEM (pf_reduce.cu)
#ifdef PF_LU_TRACE
void set_lu_trace(unsigned long long* p);  // debug builds: per-level k_lu timestamps
#endif
#ifdef PF_SWEEP_TRACE
void set_sweep_trace(unsigned long long* p);  // debug builds: per-phase sweep timestamps of CTA (0, 0)
#endif
size_t chol_tile_doubles(int n_u);  // Cholesky workspaces per scenario (pf_chol.cu)
size_t chol_flag_ints(int n_u);
size_t chol_vec_doubles(int n_u);

}  // namespace pf
