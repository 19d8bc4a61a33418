// pf_api.cu — the C-ABI of include/pf.h: handle lifetime, host→device upload
// of the plan, capacity/state checks, and stream-ordered kernel launches.
#include "../../include/pf.h"
#include "pf_launch.h"
#include "pf_plan.h"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <numeric>
#include <cstring>
#include <string>
#include <vector>

using namespace pf;

struct pf_net {
  Plan P;
  DevNet dn{};
  Work w{};
  int device = 0;
  int C = 8;
  int max_batch = 0, max_scen = 0;
  int lu_scen = 0;  // scenarios factorized by the last successful pf_jacobian (0 = none)
  const double *lu_v = nullptr, *lu_th = nullptr;  // … and the point it was called with
  int lu_cs = 0;     // k_lu cluster size on this handle's device (set at build)
  int chol_grid = 0; // k_chol_dag resident CTAs on this handle's device (set at build)
  std::vector<void*> allocs;
  std::string err;
  long long launches = 0;
  bool prof = false;         // instrumentation: events around the hot kernels
  int reach_rows_l = 0, reach_rows_ua = 0, gu_rows = 0;  // sparse-RHS statistics (pf_dims)
  std::vector<int4> p1_task;  // bottom-subtree schedules (host copies for the upload)
  std::vector<int> p1_ptr;
  std::vector<int4> p1r_task;  // … restricted to each canonical tile's reach ([ntc][teams + 1] pointers)
  std::vector<int> p1r_ptr;
  std::vector<int4> u_top, u_bot, ua_top, ua_bot;
  std::vector<int> u_top_ptr, u_bot_ptr, ua_top_ptr, ua_bot_ptr;
  std::vector<int> hvp_order;  // k_hvp bus order (elimination-forest postorder)
  cudaEvent_t ev[10] = {};   // [0..4] k_fwd/k_mu/k_hvp/k_adj, [5..6] k_lu, [4..7] k_proj, [8..9] k_chol_dag
  // the reduction's fork/join: the ψ-weight prep kernels (A6) run on `side` while k_fwd sweeps
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

#ifndef PF_P1_IMB
#define PF_P1_IMB 10
#endif


static std::string g_build_err;

namespace {

template <class T>
bool up(pf_net* h, const std::vector<T>& v, const T** out) {
  void* p = nullptr;
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return false;
  h->allocs.push_back(p);
  if (!v.empty() && cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  *out = static_cast<const T*>(p);
  return true;
}

template <class T>
bool alloc(pf_net* h, size_t count, T** out) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)) != cudaSuccess) return false;
  h->allocs.push_back(p);
  *out = static_cast<T*>(p);
  return true;
}

pf_status cuda_check(pf_net* h, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->err = std::string(where) + ": " + cudaGetErrorString(e);
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

bool set_device(pf_net* h) {
  if (h->device < 0) { h->err = "host-only handle (device < 0): no compute"; return false; }
  return cudaSetDevice(h->device) == cudaSuccess;
}

}  // namespace

extern "C" {

const char* pf_build_error(void) { return g_build_err.c_str(); }

pf_status pf_build_network(int32_t n_b, int32_t n_l, int32_t n_g, const int32_t* line_from,
                           const int32_t* line_to, const double* Y_ff, const double* Y_ft,
                           const double* Y_tf, const double* Y_tt, const double* Y_sh,
                           const int32_t* gen_bus, int32_t ref_bus, const double* p_d,
                           const double* q_d, const double* F_max, const double* c_quad,
                           const double* c_lin, int32_t max_batch, int32_t max_scen,
                           int32_t device, pf_net** out) {
  return pf_build_network_ex(n_b, n_l, n_g, line_from, line_to, Y_ff, Y_ft, Y_tf, Y_tt, Y_sh, gen_bus, ref_bus, p_d,
                             q_d, F_max, c_quad, c_lin, max_batch, max_scen, device, 0, out);
}

pf_status pf_build_network_ex(int32_t n_b, int32_t n_l, int32_t n_g, const int32_t* line_from,
                              const int32_t* line_to, const double* Y_ff, const double* Y_ft,
                              const double* Y_tf, const double* Y_tt, const double* Y_sh,
                              const int32_t* gen_bus, int32_t ref_bus, const double* p_d,
                              const double* q_d, const double* F_max, const double* c_quad,
                              const double* c_lin, int32_t max_batch, int32_t max_scen,
                              int32_t device, int32_t tile_cols, pf_net** out) {
  g_build_err.clear();
  if (!out || !line_from || !line_to || !Y_ff || !Y_ft || !Y_tf || !Y_tt || !Y_sh || !gen_bus || !p_d ||
      !q_d || !F_max || !c_quad || !c_lin) {
    g_build_err = "null argument";
    return PF_ERR_ARG;
  }
  *out = nullptr;
  if (max_batch < 1 || max_scen < 1) { g_build_err = "max_batch and max_scen must be >= 1"; return PF_ERR_ARG; }
  if (tile_cols != 0 && tile_cols != 8 && tile_cols != 16 && tile_cols != 32 && tile_cols != 64) {
    g_build_err = "tile_cols must be 0 (automatic), 8, 16, 32 or 64";
    return PF_ERR_ARG;
  }
  pf_net* h = new pf_net();
  bool topo = false;
  std::string e = build_plan(n_b, n_l, n_g, line_from, line_to, gen_bus, ref_bus, F_max, h->P, &topo);
  if (!e.empty()) {
    g_build_err = e;
    delete h;
    return topo ? PF_ERR_TOPOLOGY : PF_ERR_ARG;
  }
  h->device = device;
  const Plan& P = h->P;
  h->max_batch = max_batch;
  h->max_scen = max_scen;
  h->C = tile_cols ? tile_cols : pick_tile_cols(P.n_x, max_batch * max_scen);
  if (device < 0) {  // host analysis only: structure queries work, compute calls return PF_ERR_STATE
    *out = h;
    return PF_OK;
  }
  if (!set_device(h)) { g_build_err = "cudaSetDevice failed"; delete h; return PF_ERR_CUDA; }

  DevNet& d = h->dn;
  d.n_b = P.n_b; d.n_l = P.n_l; d.n_g = P.n_g; d.n_x = P.n_x; d.n_u = P.n_u; d.m = P.m;
  d.n_r = P.n_r; d.n_h = P.n_h; d.r0 = P.r0; d.g_r = P.g_r; d.n_gb = P.n_gb;
  d.nblk = (int)P.blk_bus.size();
  d.nnz_jb = (int)P.jb_idx.size(); d.nnz_gx = (int)P.gx_idx.size(); d.nnz_gu = (int)P.gu_idx.size();
  d.nnz_a = (int)P.a_idx.size(); d.nnz_lu = (int)P.lu_idx.size();
  d.nlevL = (int)P.levL_ptr.size() - 1; d.nlevU = (int)P.levU_ptr.size() - 1;

  std::vector<double> coef(8 * (size_t)n_l), gsh(n_b), bsh(n_b), cq(c_quad, c_quad + n_g), cl(c_lin, c_lin + n_g);
  for (int l = 0; l < n_l; ++l) {
    coef[0 * n_l + l] = Y_ff[2 * l]; coef[1 * n_l + l] = Y_ff[2 * l + 1];
    coef[2 * n_l + l] = Y_ft[2 * l]; coef[3 * n_l + l] = Y_ft[2 * l + 1];
    coef[4 * n_l + l] = Y_tf[2 * l]; coef[5 * n_l + l] = Y_tf[2 * l + 1];
    coef[6 * n_l + l] = Y_tt[2 * l]; coef[7 * n_l + l] = Y_tt[2 * l + 1];
  }
  for (int i = 0; i < n_b; ++i) { gsh[i] = Y_sh[2 * i]; bsh[i] = Y_sh[2 * i + 1]; }
  std::vector<double> pd(p_d, p_d + n_b), qd(q_d, q_d + n_b);
  std::vector<int> lf(line_from, line_from + n_l), lt(line_to, line_to + n_l), gb(gen_bus, gen_bus + n_g);
  std::vector<int> gbus;
  for (int i = 0; i < n_b; ++i) if (P.bus_gen[i] >= 0) gbus.push_back(i);
  std::vector<int4> rowmeta(P.n_x);
  for (int r = 0; r < P.n_x; ++r) rowmeta[r] = make_int4(P.lu_ptr[r], P.lu_diag[r], P.lu_ptr[r + 1], P.row_blk[r]);
  d.C = h->C;
  d.lu_maxlen = P.lu_maxlen;
  // Sweep entry streams (pf_reduce.cu run_seq): per block and orientation one contiguous
  // segment  [row A gathers, m][row B gathers, m (two-row blocks)][{d_A, intra}, {d_B, 0}]
  // with row A the row solved first (LOWER: θ, UPPER: v).  A two-row block lists both rows
  // over the union of their columns in one order (entry k of each row names the same column;
  // a column a row lacks is a zero-valued pad), so the sweep gathers each column once for both
  // rows — 54% of the gathers of two separate lists at case9241; m = the list length rounded
  // up to even, a last pad {0, a column the block gathers} (a zero product with a final row).  The task is {r0 | two << 31, segment start, m, 0}.
  // sw_src says where each slot comes from (k_lu packs the L/U and Lᵀ/Uᵀ value streams):
  //   {e, -1} gather {v(e), column(e)·C};  {e, -2} pad {0, column(e)·C};
  //   {a, b ≥ 0} scalars {v(a), v(b)};     {a, -3} scalars {v(a) or 0 if a < 0, 0}
  const int nblk = (int)P.blk_bus.size();
  std::vector<int4> taskL(nblk), taskU(nblk);
  std::vector<int2> sw_src;
  auto segment = [&](int p, bool lower) {
    const int r0 = P.blk_ptr[p];
    const bool two = P.blk_ptr[p + 1] - r0 == 2;
    const int rA = r0 + (!lower && two), rB = r0 + lower;
    int a0, a1, b0 = 0, b1 = 0, intra = -1;
    if (lower) {
      a0 = P.lu_ptr[rA]; a1 = P.lu_diag[rA];
      if (two) { b0 = P.lu_ptr[rB]; b1 = P.lu_diag[rB] - 1; intra = b1; }
    } else {
      a0 = P.lu_diag[rA] + 1; a1 = P.lu_ptr[rA + 1];
      if (two) { intra = P.lu_diag[rB] + 1; b0 = intra + 1; b1 = P.lu_ptr[rB + 1]; }
    }
    if (two && P.lu_idx[intra] != rA) { fprintf(stderr, "pf: intra-block entry missing\n"); abort(); }
    const int any = a1 > a0 ? a0 : b0;  // a gathered column for the pads
    const int start = (int)sw_src.size();
    int m;
    if (!two) {
      m = (a1 - a0 + 1) & ~1;
      for (int k = 0; k < m; ++k) sw_src.push_back(a0 + k < a1 ? make_int2(a0 + k, -1) : make_int2(any, -2));
    } else {
      // both rows over the UNION of their (ascending) columns, in the same order: entry k of
      // row A and of row B name the same column, so the sweep gathers it once for both rows
      // (a row's missing columns are zero-valued pads; each row keeps its own entry order)
      std::vector<int> ea, eb;
      for (int i = a0, j = b0; i < a1 || j < b1;) {
        const int ci = i < a1 ? P.lu_idx[i] : INT_MAX, cj = j < b1 ? P.lu_idx[j] : INT_MAX;
        ea.push_back(ci <= cj ? i++ : -1);
        eb.push_back(cj <= ci ? j++ : -1);
      }
      const int u = (int)ea.size();
      m = (u + 1) & ~1;
      for (int k = 0; k < m; ++k)
        sw_src.push_back(k >= u ? make_int2(any, -2) : ea[k] >= 0 ? make_int2(ea[k], -1) : make_int2(eb[k], -2));
      for (int k = 0; k < m; ++k)
        sw_src.push_back(k >= u ? make_int2(any, -2) : eb[k] >= 0 ? make_int2(eb[k], -1) : make_int2(ea[k], -2));
    }
    sw_src.push_back(two ? make_int2(P.lu_diag[rA], intra) : make_int2(P.lu_diag[rA], -3));
    sw_src.push_back(make_int2(two ? P.lu_diag[rB] : -1, -3));
    return make_int4(r0 | (two ? (int)0x80000000u : 0), start, m, 0);
  };
  {
    std::vector<int4> segL(nblk), segU(nblk);
    for (int p = 0; p < nblk; ++p) { segL[p] = segment(p, true); segU[p] = segment(p, false); }
    for (int bi = 0; bi < nblk; ++bi) { taskL[bi] = segL[P.levL_blk[bi]]; taskU[bi] = segU[P.levU_blk[bi]]; }
  }
  d.nsw = (int)sw_src.size();
  // sparse-RHS reach (pf_dev.cuh): elimination tree of the filled L, then per
  // canonical tile the union of the tree paths from its columns' G_u rows
  std::vector<int> parent(P.n_x, -1);
  for (int r = 0; r < P.n_x; ++r)
    for (int e = P.lu_ptr[r]; e < P.lu_diag[r]; ++e)
      if (parent[P.lu_idx[e]] < 0) parent[P.lu_idx[e]] = r;
  const int TC = h->C, ntc = (P.n_u + TC - 1) / TC, bmw = (P.n_x + 31) / 32, nlevL = d.nlevL, nlevU = d.nlevU;
  std::vector<int4> taskLr;
  std::vector<int> levLr_ptr((size_t)ntc * (nlevL + 1), 0), row_mark(P.n_x, -1), blk_mark(nblk, -1);
  std::vector<unsigned> rowbm((size_t)ntc * bmw, 0u);
  auto climb = [&](int r, int stamp) {
    for (; r >= 0 && row_mark[r] != stamp; r = parent[r]) { row_mark[r] = stamp; blk_mark[P.row_blk[r]] = stamp; }
  };
  for (int t = 0; t < ntc; ++t) {
    for (int c = t * TC; c < std::min(P.n_u, (t + 1) * TC); ++c)
      for (int e = P.guc_ptr[c]; e < P.guc_ptr[c + 1]; ++e) climb(P.guc_row[e], t);
    for (int r = 0; r < P.n_x; ++r)
      if (row_mark[r] == t) rowbm[(size_t)t * bmw + r / 32] |= 1u << (r % 32);
    levLr_ptr[(size_t)t * (nlevL + 1)] = (int)taskLr.size();
    for (int l = 0; l < nlevL; ++l) {
      for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi)
        if (blk_mark[P.levL_blk[bi]] == t) taskLr.push_back(taskL[bi]);
      levLr_ptr[(size_t)t * (nlevL + 1) + l + 1] = (int)taskLr.size();
    }
  }
  for (int c = 0; c < P.n_u; ++c)
    for (int e = P.guc_ptr[c]; e < P.guc_ptr[c + 1]; ++e) climb(P.guc_row[e], ntc);
  std::vector<int4> taskUa;
  std::vector<int> levUa_ptr(nlevU + 1, 0);
  for (int l = 0; l < nlevU; ++l) {
    for (int bi = P.levU_ptr[l]; bi < P.levU_ptr[l + 1]; ++bi)
      if (blk_mark[P.levU_blk[bi]] == ntc) taskUa.push_back(taskU[bi]);
    levUa_ptr[l + 1] = (int)taskUa.size();
  }
  d.ntc = ntc; d.bmw = bmw;
  // k_lu schedule (host plan, pf_plan.cpp lu_schedule)
  std::vector<int> fr_pos(P.n_x, -1);
  for (size_t f = 0; f < P.fr_row.size(); ++f) fr_pos[P.fr_row[f]] = (int)f;
  d.fr_lev = P.fr_lev; d.fr_n = (int)P.fr_row.size();
  d.lu_lev0 = P.lu_lev0; d.lu_nteam = kLuPairs;
  for (size_t k = 0; k < rowbm.size(); ++k) h->reach_rows_l += __builtin_popcount(rowbm[k]);
  for (int r = 0; r < P.n_x; ++r) h->reach_rows_ua += row_mark[r] == ntc;
  for (int r = 0; r < P.n_x; ++r) h->gu_rows += P.gur_ptr[r + 1] > P.gur_ptr[r];
  // bottom-subtree schedule of the LOWER sweeps over all blocks (pf_reduce.cu sweep(),
  // phase 1): levels < lev0 are split into the subtrees of the block elimination tree
  // hanging below level lev0; each team of a CTA walks its subtrees in postorder.
  // lev0 is the deepest cut whose largest team load stays within PF_P1_IMB% of the mean.
  {
    const int nteam = 256 / std::min(TC, 32);
    std::vector<int> blk_lev(nblk), bpar(nblk, -1), root(nblk), task_of(nblk);
    for (int l = 0; l < nlevL; ++l)
      for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) { blk_lev[P.levL_blk[bi]] = l; task_of[P.levL_blk[bi]] = bi; }
    for (int p = 0; p < nblk; ++p) {
      const int last = P.blk_ptr[p + 1] - 1;
      if (parent[last] >= 0) bpar[p] = P.row_blk[parent[last]];
    }
    // the deepest cut ≤ max_lev0 whose team loads stay within PF_P1_IMB% of the mean
    auto schedule = [&](int nteam, int max_lev0, int imb, std::vector<int>& best_order, std::vector<int>& best_ptr,
                        int& best_lev0) {
    best_order.clear(); best_ptr.assign(nteam + 1, 0);
    best_lev0 = 0;
    for (int lev0 = 1; lev0 <= max_lev0; ++lev0) {
      // subtree roots: blocks below lev0 whose parent is at or above lev0
      for (int l = lev0 - 1; l >= 0; --l)
        for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
          const int b = P.levL_blk[bi], q = bpar[b];
          root[b] = (q >= 0 && blk_lev[q] < lev0) ? root[q] : b;
        }
      std::vector<std::vector<int>> kids(nblk);
      std::vector<int> roots;
      for (int l = 0; l < lev0; ++l)
        for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
          const int b = P.levL_blk[bi];
          if (root[b] == b) roots.push_back(b); else kids[bpar[b]].push_back(b);
        }
      std::vector<int> size(nblk, 1);
      for (int l = 0; l < lev0; ++l)  // subtree sizes, children before parents
        for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
          const int b = P.levL_blk[bi];
          if (root[b] != b) size[bpar[b]] += size[b];
        }
      std::sort(roots.begin(), roots.end(), [&](int x, int y) { return size[x] != size[y] ? size[x] > size[y] : x < y; });
      std::vector<long long> load(nteam, 0);
      std::vector<std::vector<int>> mine(nteam);
      for (int r : roots) {
        const int t = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[t] += size[r];
        mine[t].push_back(r);
      }
      const long long tot = std::accumulate(load.begin(), load.end(), 0LL);
      const long long mx = *std::max_element(load.begin(), load.end());
      if (lev0 > 1 && mx * 100 > tot * (100 + imb) / nteam) break;  // imbalance beyond imb %: keep the previous cut
      std::vector<int> order, ptr(nteam + 1, 0);
      for (int t = 0; t < nteam; ++t) {
        for (int r : mine[t]) {  // iterative postorder of the subtree of r
          std::vector<std::pair<int, size_t>> st{{r, 0}};
          while (!st.empty()) {
            auto& [b, c] = st.back();
            if (c < kids[b].size()) { const int ch = kids[b][c++]; st.push_back({ch, 0}); }
            else { order.push_back(b); st.pop_back(); }
          }
        }
        ptr[t + 1] = (int)order.size();
      }
      best_order.swap(order); best_ptr.swap(ptr); best_lev0 = lev0;
    }
    };
    std::vector<int> best_order, best_ptr;
    int best_lev0 = 0;
    schedule(nteam, nlevL, PF_P1_IMB, best_order, best_ptr, best_lev0);

    std::vector<int4> p1_task(best_order.size());
    for (size_t k = 0; k < best_order.size(); ++k) p1_task[k] = taskL[task_of[best_order[k]]];
    d.p1_lev0 = best_lev0;
    h->p1_task = p1_task;
    h->p1_ptr = best_ptr;
    // k_fwd's reach-restricted L sweep (unit directions of canonical tile t): the same bottom
    // lists filtered to the tile's reach blocks (postorder kept), then its reach levels ≥ lev0
    // (own marks: blk_mark still holds the ancestor pass's stamps for the Lᵀ lists below)
    h->p1r_task.clear();
    h->p1r_ptr.assign((size_t)ntc * (nteam + 1), 0);
    std::vector<int> rmk(P.n_x, -1), bmk(nblk, -1);
    for (int t = 0; t < ntc; ++t) {
      for (int c = t * TC; c < std::min(P.n_u, (t + 1) * TC); ++c)
        for (int e = P.guc_ptr[c]; e < P.guc_ptr[c + 1]; ++e)
          for (int r = P.guc_row[e]; r >= 0 && rmk[r] != t; r = parent[r]) { rmk[r] = t; bmk[P.row_blk[r]] = t; }
      for (int tm = 0; tm < nteam; ++tm) {
        h->p1r_ptr[(size_t)t * (nteam + 1) + tm] = (int)h->p1r_task.size();
        for (int k = best_ptr[tm]; k < best_ptr[tm + 1]; ++k)
          if (bmk[best_order[k]] == t) h->p1r_task.push_back(taskL[task_of[best_order[k]]]);
      }
      h->p1r_ptr[(size_t)t * (nteam + 1) + nteam] = (int)h->p1r_task.size();
    }
    // UPPER sweeps (parents before children): the blocks above the cut in U-level
    // order, then each team's bottom subtrees in reverse postorder; once over all
    // blocks (U sweep) and once over the ancestors of G_u's rows (Lᵀ sweep).
    std::vector<int> taskU_of(nblk);
    for (int bi = 0; bi < nblk; ++bi) taskU_of[P.levU_blk[bi]] = bi;
    auto build_upper = [&](bool only_anc, std::vector<int4>& top, std::vector<int>& top_ptr, std::vector<int4>& bot,
                           std::vector<int>& bot_ptr) {
      top.clear(); top_ptr.assign(nlevU + 1, 0); bot.clear(); bot_ptr.assign(nteam + 1, 0);
      for (int l = 0; l < nlevU; ++l) {
        for (int bi = P.levU_ptr[l]; bi < P.levU_ptr[l + 1]; ++bi) {
          const int b = P.levU_blk[bi];
          if (blk_lev[b] >= best_lev0 && (!only_anc || blk_mark[b] == ntc)) top.push_back(taskU[bi]);
        }
        top_ptr[l + 1] = (int)top.size();
      }
      for (int t = 0; t < nteam; ++t) {
        for (int k = best_ptr[t + 1] - 1; k >= best_ptr[t]; --k) {
          const int b = best_order[k];
          if (!only_anc || blk_mark[b] == ntc) bot.push_back(taskU[taskU_of[b]]);
        }
        bot_ptr[t + 1] = (int)bot.size();
      }
    };
    build_upper(false, h->u_top, h->u_top_ptr, h->u_bot, h->u_bot_ptr);
    build_upper(true, h->ua_top, h->ua_top_ptr, h->ua_bot, h->ua_bot_ptr);
    // k_hvp bus order: postorder of the block elimination forest, so the 64 buses of
    // a CTA (and their neighbours' slab rows) come from a few compact subtrees; the
    // reference bus (no state rows) last
    std::vector<std::vector<int>> ch(nblk);
    std::vector<int> roots_all;
    for (int b = 0; b < nblk; ++b) (bpar[b] >= 0 ? ch[bpar[b]] : roots_all).push_back(b);
    h->hvp_order.clear();
    for (int r : roots_all) {
      std::vector<std::pair<int, size_t>> st{{r, 0}};
      while (!st.empty()) {
        auto& [b, c] = st.back();
        if (c < ch[b].size()) { const int x = ch[b][c++]; st.push_back({x, 0}); }
        else { h->hvp_order.push_back(P.blk_bus[b]); st.pop_back(); }
      }
    }
    for (int i = 0; i < n_b; ++i)
      if (P.bus_pth[i] < 0 && P.bus_pv[i] < 0) h->hvp_order.push_back(i);
  }

  const std::vector<int>& hvp_order = h->hvp_order.size() == (size_t)n_b ? h->hvp_order : P.hvp_bus;
  // step recovery / Newton maps: G row of each permuted row, A by columns
  std::vector<int> row_g(P.n_x);
  for (int r = 0; r < P.n_x; ++r) row_g[r] = -1;
  for (int i = 0; i < n_b; ++i) {
    if (P.x_th[i] >= 0) row_g[P.iperm[P.x_th[i]]] = i;
    if (P.x_v[i] >= 0) row_g[P.iperm[P.x_v[i]]] = n_b + i;
  }
  const int n_z = P.n_u + P.n_x;
  std::vector<int> a_cptr(n_z + 1, 0), a_crow(P.a_idx.size()), a_cpos(P.a_idx.size());
  for (int c : P.a_idx) ++a_cptr[c + 1];
  for (int z = 0; z < n_z; ++z) a_cptr[z + 1] += a_cptr[z];
  {
    std::vector<int> fill(a_cptr.begin(), a_cptr.end() - 1);
    for (int k = 0; k < P.m; ++k)
      for (int e = P.a_ptr[k]; e < P.a_ptr[k + 1]; ++e) {
        const int q = fill[P.a_idx[e]]++;
        a_crow[q] = k; a_cpos[q] = e;   // ascending rows within a column (deterministic sums)
      }
  }
  // Bus-block sets of the staged block-SpMM kernels (pf_reduce.cu k_blk): k_hvp over every bus in
  // hvp_order (μ rows of generator neighbours staged too), k_mu over the generator buses in the
  // same order; consecutive output buses form a chunk while its distinct staged rows fit the cap.
  std::vector<int4> hvp_out(n_b);
  for (int kb = 0; kb < n_b; ++kb) {
    const int i = h->hvp_order.size() == (size_t)n_b ? h->hvp_order[kb] : P.hvp_bus[kb];
    hvp_out[kb] = make_int4(i, P.bus_pth[i], P.bus_pv[i] >= 0 ? P.bus_pv[i] : -1 - P.u_v[i], P.bus_gen[i]);
  }
  std::vector<int4> mu_out;
  for (const int4& o : hvp_out) if (P.bus_gen[o.x] >= 0) mu_out.push_back(make_int4(o.x, P.bus_gen[o.x], 0, 0));
  auto build_set = [&](const std::vector<int4>& outs, bool with_mu, BlkSet& B) {
    const int row_cap = hvp_stage_rows(h->C), bus_cap = 64;
    std::vector<int> ptr(1, 0), self, nbr, ck(1, 0), stp(1, 0), str, slot(P.n_x + 2 * n_g, -1), rows;
    std::vector<int4> meta;
    std::vector<int2> jt;
    auto nbrs = [&](int i) {
      std::vector<int> nb{i};
      for (int e = P.inc_ptr[i]; e < P.inc_ptr[i + 1]; ++e) {
        const int l = P.inc_line[e];
        nb.push_back(line_from[l] == i ? line_to[l] : line_from[l]);
      }
      std::sort(nb.begin() + 1, nb.end());  // the bus itself first (the difference form), then ascending
      nb.erase(std::unique(nb.begin() + 1, nb.end()), nb.end());
      return nb;
    };
    // rows of bus j: θ_j and v_j slab rows (< n_x); with_mu: μ_A rows n_x + 2g, + 1 of a generator bus j
    auto rows_of = [&](int j, int* r) {
      r[0] = P.bus_pth[j]; r[1] = P.bus_pv[j];
      r[2] = with_mu && P.bus_gen[j] >= 0 ? P.n_x + 2 * P.bus_gen[j] : -1;
    };
    auto close_chunk = [&]() {
      for (int r : rows) slot[r] = -1;
      str.insert(str.end(), rows.begin(), rows.end());
      stp.push_back((int)str.size());
      ck.push_back((int)ptr.size() - 1);
      rows.clear();
    };
    for (const int4& o : outs) {
      const int i = o.x;
      const std::vector<int> nb = nbrs(i);
      int extra = 0;  // rows this bus adds to the open chunk
      for (int j : nb) { int r[3]; rows_of(j, r); for (int q = 0; q < 3; ++q) extra += (r[q] >= 0 && slot[r[q]] < 0) * (q == 2 ? 2 : 1); }
      const int nbus = (int)ptr.size() - 1 - ck.back();
      if (nbus > 0 && ((int)rows.size() + extra > row_cap || nbus >= bus_cap)) close_chunk();
      for (int j : nb) {
        int r[3]; rows_of(j, r);
        for (int q = 0; q < 3; ++q)
          if (r[q] >= 0 && slot[r[q]] < 0) {
            slot[r[q]] = (int)rows.size(); rows.push_back(r[q]);
            if (q == 2) rows.push_back(r[q] + 1);  // μ^Q row right after μ^P
          }
        const int vs = r[1] >= 0 ? slot[r[1]] : -1 - P.u_v[j];
        meta.push_back(make_int4(r[0] >= 0 ? slot[r[0]] : -1, vs, r[2] >= 0 ? slot[r[2]] : -1, 0));
        self.push_back(i);
        nbr.push_back(j);
        // θ_i / v_i within J_bus row P_j (Q_j shares the pattern): own columns or an incidence of j towards i
        int ot = -1, ov = -1;
        if (with_mu && P.bus_gen[j] >= 0) {
          if (j == i) { ot = P.jb_self_th[i]; ov = P.jb_self_v[i]; }
          else
            for (int e = P.inc_ptr[j]; e < P.inc_ptr[j + 1]; ++e) {
              const int l = P.inc_line[e];
              if ((line_from[l] == j ? line_to[l] : line_from[l]) == i) { ot = P.inc_off_th[e]; ov = P.inc_off_v[e]; break; }
            }
        }
        jt.push_back(make_int2(ot, ov));
      }
      ptr.push_back((int)meta.size());
    }
    close_chunk();
    B.nout = (int)outs.size(); B.nblk = (int)meta.size(); B.nchunk = (int)ck.size() - 1;
    B.st_max = B.blk_max = B.ck_max = 0;
    for (int c = 0; c < B.nchunk; ++c) {
      B.st_max = std::max(B.st_max, stp[c + 1] - stp[c]);
      B.blk_max = std::max(B.blk_max, ptr[ck[c + 1]] - ptr[ck[c]]);
      B.ck_max = std::max(B.ck_max, ck[c + 1] - ck[c]);
    }
    return up(h, ptr, &B.ptr) && up(h, meta, &B.meta) && up(h, self, &B.self) && up(h, nbr, &B.nbr) &&
           up(h, jt, &B.jt) && up(h, outs, &B.out) && up(h, ck, &B.ck_ptr) && up(h, stp, &B.st_ptr) &&
           up(h, str, &B.st_row);
  };
  bool blk_ok = build_set(hvp_out, true, d.hb) && build_set(mu_out, false, d.mb);
  std::vector<int> u_gen(P.n_u, -1);
  for (int g = 0; g < n_g; ++g) if (P.u_p[g] >= 0) u_gen[P.u_p[g]] = g;
  bool ok = blk_ok && up(h, lf, &d.lf) && up(h, lt, &d.lt) && up(h, coef, &d.coef) && up(h, gsh, &d.gsh) &&
            up(h, bsh, &d.bsh) && up(h, gb, &d.gen_bus) && up(h, P.bus_gen, &d.bus_gen) &&
            up(h, cq, &d.c_quad) && up(h, cl, &d.c_lin) && up(h, pd, &d.p_d0) && up(h, qd, &d.q_d0) &&
            up(h, P.x_th, &d.x_th) && up(h, P.x_v, &d.x_v) && up(h, P.u_v, &d.u_v) && up(h, P.u_p, &d.u_p) &&
            up(h, P.bus_rP, &d.bus_rP) && up(h, P.bus_rQ, &d.bus_rQ) && up(h, P.line_hf, &d.line_hf) &&
            up(h, P.line_ht, &d.line_ht) && up(h, P.inc_ptr, &d.inc_ptr) && up(h, P.inc_line, &d.inc_line) &&
            up(h, P.inc_off_th, &d.inc_off_th) && up(h, P.inc_off_v, &d.inc_off_v) &&
            up(h, P.jb_ptr, &d.jb_ptr) && up(h, P.jb_self_th, &d.jb_self_th) && up(h, P.jb_self_v, &d.jb_self_v) &&
            up(h, P.gx_src, &d.gx_src) && up(h, P.gu_src, &d.gu_src) && up(h, P.a_ptr, &d.a_ptr) &&
            up(h, P.a_src, &d.a_src) && up(h, P.ah_off, &d.ah_off) && up(h, P.h_line, &d.h_line) &&
            up(h, P.h_end, &d.h_end) && up(h, P.blk_ptr, &d.blk_ptr) && up(h, P.lu_ptr, &d.lu_ptr) &&
            up(h, P.lu_idx, &d.lu_idx) && up(h, P.lu_diag, &d.lu_diag) && up(h, P.lu_src, &d.lu_src) &&
            up(h, P.lu_tpos, &d.lu_tpos) && up(h, P.upd_ptr, &d.upd_ptr) && up(h, P.upd_dst, &d.upd_dst) && up(h, P.upd_src, &d.upd_src) &&
            up(h, P.levL_ptr, &d.levL_ptr) && up(h, P.levL_blk, &d.levL_blk) && up(h, P.levU_ptr, &d.levU_ptr) &&
            up(h, P.levU_blk, &d.levU_blk) && up(h, P.guc_ptr, &d.guc_ptr) && up(h, P.guc_row, &d.guc_row) &&
            up(h, P.guc_src, &d.guc_src) && up(h, P.gur_ptr, &d.gur_ptr) && up(h, P.gur_col, &d.gur_col) &&
            up(h, P.gur_src, &d.gur_src) && up(h, P.bus_pth, &d.bus_pth) && up(h, P.bus_pv, &d.bus_pv) &&
            up(h, gbus, &d.gbus) && up(h, rowmeta, &d.rowmeta) && up(h, hvp_order, &d.hvp_bus) &&
            up(h, taskL, &d.taskL) && up(h, taskU, &d.taskU) && up(h, sw_src, &d.sw_src) &&
            up(h, P.fr_row, &d.fr_row) && up(h, fr_pos, &d.fr_pos) && up(h, P.lu_p1_blk, &d.lu_p1_blk) &&
            up(h, P.lu_p1_ptr, &d.lu_p1_ptr) && up(h, P.lu_lev_blk, &d.lu_lev_blk) &&
            up(h, taskLr, &d.taskLr) && up(h, levLr_ptr, &d.levLr_ptr) && up(h, rowbm, &d.rowbm) &&
            up(h, taskUa, &d.taskUa) && up(h, levUa_ptr, &d.levUa_ptr) && up(h, h->p1_task, &d.p1_task) &&
            up(h, h->p1_ptr, &d.p1_ptr) && up(h, h->p1r_task, &d.p1r_task) && up(h, h->p1r_ptr, &d.p1r_ptr) && up(h, h->u_top, &d.u_top) && up(h, h->u_top_ptr, &d.u_top_ptr) &&
            up(h, h->u_bot, &d.u_bot) && up(h, h->u_bot_ptr, &d.u_bot_ptr) && up(h, h->ua_top, &d.ua_top) &&
            up(h, h->ua_top_ptr, &d.ua_top_ptr) && up(h, h->ua_bot, &d.ua_bot) && up(h, h->ua_bot_ptr, &d.ua_bot_ptr) &&
            up(h, P.perm, &d.perm) && up(h, P.iperm, &d.iperm) && up(h, row_g, &d.row_g) &&
            up(h, a_cptr, &d.a_cptr) && up(h, P.a_idx, &d.a_idx) && up(h, a_crow, &d.a_crow) && up(h, a_cpos, &d.a_cpos) &&
            up(h, u_gen, &d.u_gen);
  Work& w = h->w;
  const size_t S = max_scen;
  w.max_tiles = max_scen * ((max_batch + h->C - 1) / h->C);
  const size_t T = w.max_tiles, C = h->C;
  ok = ok && alloc(h, S * d.nnz_jb, &w.jb) && alloc(h, S * d.nnz_gu, &w.gu) && alloc(h, S * d.nnz_lu, &w.lu) &&
       alloc(h, S * d.nsw, &w.swA) && alloc(h, S * d.nsw, &w.swT) && alloc(h, S * d.nnz_gu, &w.pkG) && alloc(h, S * d.n_x, &w.rowmax) && alloc(h, S * d.n_x, &w.invd) && alloc(h, S * LS_N * d.n_l, &w.ls) &&
       alloc(h, S * BS_N * d.n_b, &w.bs) && alloc(h, S * LB_N * d.n_l, &w.lblk) && alloc(h, S * 4 * d.n_l, &w.sflow) && alloc(h, 2 * S, &w.info) &&
       alloc(h, T * d.n_x * C, &w.slabZ) && alloc(h, T * d.n_x * C, &w.slabW) &&
       alloc(h, T * d.n_u * C, &w.hu) && alloc(h, T * d.n_g * 2 * C, &w.mu) &&
       alloc(h, S * chol_tile_doubles(d.n_u), &w.ctile) && alloc(h, S * chol_flag_ints(d.n_u), &w.cflag) &&
       alloc(h, 1 + 1024, &w.cticket) && alloc(h, S * chol_vec_doubles(d.n_u), &w.cy) &&
       alloc(h, S * d.nnz_a, &w.aval) && alloc(h, S * (d.n_u + d.n_x + d.m), &w.zero) &&
       alloc(h, S * 2 * d.n_b, &w.gbuf) && alloc(h, S, &w.res) && alloc(h, S, &w.active) &&
       alloc(h, S, &w.csidx) && alloc(h, S, &w.cdelta) && alloc(h, S * (size_t)d.hb.nblk * 8, &w.hbval) &&
       alloc(h, S * (size_t)d.mb.nblk * 8, &w.mbval);
  ok = ok && cudaMemset(w.zero, 0, S * (d.n_u + d.n_x + d.m) * sizeof(double)) == cudaSuccess;
  if (!ok) {
    g_build_err = std::string("device allocation/upload failed: ") + cudaGetErrorString(cudaGetLastError());
    pf_destroy(h);
    return PF_ERR_CUDA;
  }
  // launch geometry that depends on the device (cluster support, SM count): per handle.
  // k_lu keeps one dense row workspace per warp in SMEM: a filled-LU row longer than that
  // allows (lu_maxlen ≳ 1,250 on a B200) has no fallback — refuse the network here, clearly
  {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    if (lu_smem_bytes(d) > (size_t)optin) {
      g_build_err = "k_lu needs " + std::to_string(lu_smem_bytes(d)) + " B of SMEM per CTA (longest filled-LU row " +
                    std::to_string(P.lu_maxlen) + " entries) > the device's " + std::to_string(optin) +
                    " B: network too dense for this build";
      pf_destroy(h);
      return PF_ERR_CAPACITY;
    }
  }
  h->lu_cs = lu_cluster_size(d);
  h->chol_grid = chol_grid_max();
  if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->join, cudaEventDisableTiming) != cudaSuccess) {
    g_build_err = std::string("stream/event creation: ") + cudaGetErrorString(cudaGetLastError());
    pf_destroy(h);
    return PF_ERR_CUDA;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    g_build_err = std::string("build sync: ") + cudaGetErrorString(cudaGetLastError());
    pf_destroy(h);
    return PF_ERR_CUDA;
  }
  *out = h;
  return PF_OK;
}

void pf_destroy(pf_net* h) {
  if (!h) return;
  if (h->device >= 0) cudaSetDevice(h->device);
  for (auto& e : h->ev) if (e) cudaEventDestroy(e);
  if (h->fork) cudaEventDestroy(h->fork);
  if (h->join) cudaEventDestroy(h->join);
  if (h->side) cudaStreamDestroy(h->side);
  for (void* p : h->allocs) cudaFree(p);
  delete h;
}

pf_status pf_query(const pf_net* h, pf_dims* o) {
  if (!h || !o) return PF_ERR_ARG;
  const Plan& P = h->P;
  o->n_b = P.n_b; o->n_l = P.n_l; o->n_g = P.n_g; o->n_x = P.n_x; o->n_u = P.n_u; o->m = P.m;
  o->n_r = P.n_r; o->n_h = P.n_h; o->ref_bus = P.r0; o->ref_gen = P.g_r;
  o->nnz_gx = (int)P.gx_idx.size(); o->nnz_gu = (int)P.gu_idx.size(); o->nnz_a = (int)P.a_idx.size();
  o->nnz_lu = (int)P.lu_idx.size(); o->n_blocks = (int)P.blk_bus.size();
  o->n_levels_l = (int)P.levL_ptr.size() - 1; o->n_levels_u = (int)P.levU_ptr.size() - 1;
  o->max_batch = h->max_batch; o->max_scen = h->max_scen; o->tile_cols = h->C;
  o->reach_rows_l = h->reach_rows_l; o->reach_rows_ua = h->reach_rows_ua; o->gu_rows = h->gu_rows;
  o->front_level = P.fr_lev; o->front_rows = (int)P.fr_row.size(); o->lu_cut_level = P.lu_lev0;
  o->lu_pairs = (int)P.lu_p1_ptr.size() - 1;
  return PF_OK;
}

pf_status pf_get_structure(const pf_net* h, int32_t which, int32_t* out) {
  if (!h || !out) return PF_ERR_ARG;
  const Plan& P = h->P;
  const std::vector<int>* v = nullptr;
  switch (which) {
    case PF_X_THETA: v = &P.x_th; break;
    case PF_X_V: v = &P.x_v; break;
    case PF_U_V: v = &P.u_v; break;
    case PF_U_P: v = &P.u_p; break;
    case PF_GX_PTR: v = &P.gx_ptr; break;
    case PF_GX_IDX: v = &P.gx_idx; break;
    case PF_GU_PTR: v = &P.gu_ptr; break;
    case PF_GU_IDX: v = &P.gu_idx; break;
    case PF_A_PTR: v = &P.a_ptr; break;
    case PF_A_IDX: v = &P.a_idx; break;
    case PF_BUS_ORDER: v = &P.bus_order; break;
    case PF_PERM: v = &P.perm; break;
    case PF_BLOCK_PTR: v = &P.blk_ptr; break;
    case PF_LU_PTR: v = &P.lu_ptr; break;
    case PF_LU_IDX: v = &P.lu_idx; break;
    case PF_LEVEL_L_PTR: v = &P.levL_ptr; break;
    case PF_LEVEL_L_BLK: v = &P.levL_blk; break;
    case PF_LEVEL_U_PTR: v = &P.levU_ptr; break;
    case PF_LEVEL_U_BLK: v = &P.levU_blk; break;
    case PF_FRONT_ROW: v = &P.fr_row; break;
    case PF_LU_SUBTREE_PTR: v = &P.lu_p1_ptr; break;
    case PF_LU_SUBTREE_BLK: v = &P.lu_p1_blk; break;
    case PF_LU_LEVEL_BLK: v = &P.lu_lev_blk; break;
    default: return PF_ERR_ARG;
  }
  if (!v->empty()) std::memcpy(out, v->data(), v->size() * sizeof(int32_t));
  return PF_OK;
}

const char* pf_last_error(const pf_net* h) { return h ? h->err.c_str() : g_build_err.c_str(); }

int64_t pf_launch_count(const pf_net* h) { return h ? h->launches : 0; }

pf_status pf_eval_constraints(pf_net* h, int32_t n_scen, const double* v, const double* theta,
                              const double* p_g, const double* q_g, const double* p_d, const double* q_d,
                              double* G, double* H, double* s_flow, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!v || !theta || !p_g || !q_g || !G || n_scen < 1) { h->err = "pf_eval_constraints: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_eval_constraints: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  h->launches += launch_eval(h->dn, h->w, n_scen, v, theta, p_g, q_g, p_d, q_d, G, H, s_flow, (cudaStream_t)stream);
  return cuda_check(h, "pf_eval_constraints");
}

pf_status pf_jacobian(pf_net* h, int32_t n_scen, const double* v, const double* theta, double* Gx_val,
                      double* Gu_val, double* A_val, int32_t* info, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!v || !theta || n_scen < 1) { h->err = "pf_jacobian: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_jacobian: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  h->lu_scen = 0;  // the factors are being overwritten
  h->launches += launch_jacobian(h->dn, h->w, n_scen, v, theta, Gx_val, Gu_val, A_val, info, (cudaStream_t)stream,
                                 h->lu_cs, h->prof ? h->ev + 5 : nullptr);
  const pf_status st = cuda_check(h, "pf_jacobian");
  if (st == PF_OK) { h->lu_scen = n_scen; h->lu_v = v; h->lu_th = theta; }
  return st;
}

pf_status pf_reduced_hessian_batch(pf_net* h, int32_t n_scen, const double* v, const double* theta,
                                   const double* p_d, const double* lambda, const double* y,
                                   const double* sigma_s, const double* sigma_x, const double* V,
                                   int32_t col0, int32_t N, double* KV, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!lambda || !y || (!KV && N > 0) || n_scen < 1 || N < 0) { h->err = "pf_reduced_hessian_batch: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen || N > h->max_batch) { h->err = "pf_reduced_hessian_batch: capacity"; return PF_ERR_CAPACITY; }
  if (!V && (col0 < 0 || col0 + N > h->P.n_u)) { h->err = "pf_reduced_hessian_batch: columns out of range"; return PF_ERR_ARG; }
  if (h->lu_scen < n_scen) { h->err = "pf_reduced_hessian_batch: call pf_jacobian first"; return PF_ERR_STATE; }
  if ((v && v != h->lu_v) || (theta && theta != h->lu_th)) {
    h->err = "pf_reduced_hessian_batch: v/theta are not the arrays of the last pf_jacobian (its point and LU are used)";
    return PF_ERR_STATE;
  }
  if (N == 0) return PF_OK;
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  // fork: A6 (ψ weights, bus blocks) on the side stream, concurrent with A7.1–A7.2 (k_fwd needs
  // only the LU); k_blk joins it (graph-capture safe: the side stream rejoins `st`)
  if (cudaEventRecord(h->fork, st) != cudaSuccess || cudaStreamWaitEvent(h->side, h->fork, 0) != cudaSuccess)
    return cuda_check(h, "pf_reduced_hessian_batch");
  h->launches += launch_prep(h->dn, h->w, n_scen, p_d, lambda, y, sigma_s, sigma_x, h->side);
  if (cudaEventRecord(h->join, h->side) != cudaSuccess) return cuda_check(h, "pf_reduced_hessian_batch");
  h->launches += launch_reduce(h->dn, h->w, h->C, n_scen, V, col0, N, KV, st, h->prof ? h->ev : nullptr, h->join);
  return cuda_check(h, "pf_reduced_hessian_batch");
}

pf_status pf_condensed_kkt_solve(pf_net* h, int32_t n_scen, double* K, const double* sigma_u, double delta_w,
                                 double* rhs, int32_t nrhs, int32_t* info, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!K || n_scen < 1 || nrhs < 0 || (nrhs > 0 && !rhs)) { h->err = "pf_condensed_kkt_solve: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_condensed_kkt_solve: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  h->launches += launch_chol(h->dn, h->w, n_scen, K, sigma_u, delta_w, rhs, nrhs, info, h->w.info + h->max_scen,
                             (cudaStream_t)stream, h->chol_grid, nullptr, nullptr, h->prof ? h->ev + 8 : nullptr);
  return cuda_check(h, "pf_condensed_kkt_solve");
}

// ---------------------------------------------------------------- NEXT-1 / NEXT-2
namespace {
pf_status point_check(pf_net* h, const char* who, int n_scen, const double* v, const double* theta) {
  if (h->lu_scen < n_scen) { h->err = std::string(who) + ": call pf_jacobian first (for these scenarios)"; return PF_ERR_STATE; }
  if ((v && v != h->lu_v) || (theta && theta != h->lu_th)) {
    h->err = std::string(who) + ": v/theta are not the arrays of the last pf_jacobian (its point and LU are used)";
    return PF_ERR_STATE;
  }
  return PF_OK;
}
}  // namespace

pf_status pf_condensed_rhs(pf_net* h, int32_t n_scen, const double* v, const double* theta, const double* p_d,
                           const double* lambda, const double* y, const double* sigma_s, const double* sigma_x,
                           const double* r, double* b, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!lambda || !y || !r || !b || n_scen < 1) { h->err = "pf_condensed_rhs: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_condensed_rhs: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  if (pf_status st = point_check(h, "pf_condensed_rhs", n_scen, v, theta)) return st;
  cudaStream_t st = (cudaStream_t)stream;
  h->launches += launch_prep(h->dn, h->w, n_scen, p_d, lambda, y, sigma_s, sigma_x, st);
  h->launches += launch_step(0, h->dn, h->w, h->C, n_scen, r, sigma_s, nullptr, nullptr, nullptr, b, nullptr, st);
  return cuda_check(h, "pf_condensed_rhs");
}

pf_status pf_recover_step(pf_net* h, int32_t n_scen, const double* v, const double* theta, const double* p_d,
                          const double* lambda, const double* y, const double* sigma_s, const double* sigma_x,
                          const double* r, const double* p_u, double* p, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!lambda || !y || !r || !p_u || !p || n_scen < 1) { h->err = "pf_recover_step: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_recover_step: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  if (pf_status st = point_check(h, "pf_recover_step", n_scen, v, theta)) return st;
  cudaStream_t st = (cudaStream_t)stream;
  h->launches += launch_prep(h->dn, h->w, n_scen, p_d, lambda, y, sigma_s, sigma_x, st);
  h->launches += launch_step(1, h->dn, h->w, h->C, n_scen, r, sigma_s, nullptr, nullptr, p_u, p, nullptr, st);
  return cuda_check(h, "pf_recover_step");
}

pf_status pf_reduced_gradient(pf_net* h, int32_t n_scen, const double* v, const double* theta, const double* p_g,
                              const double* p_d, const double* y, double* lambda, double* grad, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!p_g || !y || !grad || n_scen < 1) { h->err = "pf_reduced_gradient: bad argument"; return PF_ERR_ARG; }
  if (n_scen > h->max_scen) { h->err = "pf_reduced_gradient: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  if (pf_status st = point_check(h, "pf_reduced_gradient", n_scen, v, theta)) return st;
  cudaStream_t st = (cudaStream_t)stream;
  // μ̃^P_r0 = y_0 + (2c₁p_ref + c₂) is the only prep output used (λ = 0, no Σ)
  h->launches += launch_prep(h->dn, h->w, n_scen, p_d, h->w.zero, y, nullptr, nullptr, st);
  h->launches += launch_step(2, h->dn, h->w, h->C, n_scen, nullptr, nullptr, y, p_g, nullptr, grad, lambda, st);
  return cuda_check(h, "pf_reduced_gradient");
}

pf_status pf_power_flow(pf_net* h, int32_t n_scen, double* v, double* theta, const double* p_g, const double* q_g,
                        const double* p_d, const double* q_d, double tol, int32_t max_iter, int32_t* iters,
                        double* resid, int32_t* info, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!v || !theta || !p_g || n_scen < 1 || max_iter < 0 || !(tol >= 0.0)) {
    h->err = "pf_power_flow: bad argument";
    return PF_ERR_ARG;
  }
  if (n_scen > h->max_scen) { h->err = "pf_power_flow: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const Work& w = h->w;
  std::vector<double> res(n_scen);
  std::vector<int> act(n_scen, 1), it(n_scen, 0), inf(n_scen, 0), lui(n_scen, 0);
  h->lu_scen = 0;
  for (int k = 0;; ++k) {
    h->launches += launch_eval(h->dn, w, n_scen, v, theta, p_g, q_g ? q_g : w.zero, p_d, q_d, w.gbuf, nullptr,
                               nullptr, st);
    h->launches += launch_pf_resid(h->dn, w, n_scen, st);
    if (cudaMemcpyAsync(res.data(), w.res, n_scen * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return cuda_check(h, "pf_power_flow");
    int n_act = 0;
    for (int s = 0; s < n_scen; ++s) {
      if (!act[s]) continue;
      if (res[s] <= tol) act[s] = 0;                                  // converged
      else if (!(res[s] == res[s]) || k == max_iter) { act[s] = 0; inf[s] = -1; }  // diverged / no convergence
      n_act += act[s];
    }
    if (!n_act) break;
    if (cudaMemcpyAsync(w.active, act.data(), n_scen * sizeof(int), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return cuda_check(h, "pf_power_flow");
    h->launches += launch_jacobian(h->dn, w, n_scen, v, theta, nullptr, nullptr, nullptr, nullptr, st, h->lu_cs);
    if (cudaMemcpyAsync(lui.data(), w.info, n_scen * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return cuda_check(h, "pf_power_flow");
    for (int s = 0; s < n_scen; ++s)
      if (act[s] && lui[s]) { act[s] = 0; inf[s] = lui[s]; }          // singular Jacobian (R18 pivot k+1)
    if (cudaMemcpyAsync(w.active, act.data(), n_scen * sizeof(int), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return cuda_check(h, "pf_power_flow");
    h->launches += launch_newton_step(h->dn, w, h->C, n_scen, v, theta, st);
    for (int s = 0; s < n_scen; ++s) it[s] += act[s];
  }
  // factorize at the final point, so a reduction / gradient / recovery can follow (RedLin, Algorithm 2)
  h->launches += launch_jacobian(h->dn, w, n_scen, v, theta, nullptr, nullptr, nullptr, nullptr, st, h->lu_cs);
  if (pf_status e = cuda_check(h, "pf_power_flow")) return e;
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(h, "pf_power_flow");
  h->lu_scen = n_scen; h->lu_v = v; h->lu_th = theta;
  for (int s = 0; s < n_scen; ++s) {
    if (iters) iters[s] = it[s];
    if (resid) resid[s] = res[s];
    if (info) info[s] = inf[s];
  }
  return PF_OK;
}

// ---------------------------------------------------------------- NEXT-3
pf_status pf_condensed_kkt_solve_reg(pf_net* h, int32_t n_scen, double* K, const double* sigma_u, double delta_init,
                                     double delta_first, double growth, double delta_max, double* rhs, int32_t nrhs,
                                     double* delta_out, int32_t* trials, int32_t* info, void* stream) {
  if (!h) return PF_ERR_ARG;
  if (!K || n_scen < 1 || nrhs < 0 || (nrhs > 0 && !rhs) || !(delta_init >= 0.0) || !(delta_first > 0.0) ||
      !(growth > 1.0) || !(delta_max >= delta_init)) {
    h->err = "pf_condensed_kkt_solve_reg: bad argument";
    return PF_ERR_ARG;
  }
  if (n_scen > h->max_scen) { h->err = "pf_condensed_kkt_solve_reg: n_scen > max_scen"; return PF_ERR_CAPACITY; }
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  int* info_ws = h->w.info + h->max_scen;
  std::vector<double> delta(n_scen, delta_init);
  std::vector<int> tr(n_scen, 1), inf(n_scen, 0), idx, got(n_scen);
  // trial 1: every scenario at δ_init
  h->launches += launch_chol(h->dn, h->w, n_scen, K, sigma_u, delta_init, rhs, nrhs, nullptr, info_ws, st,
                             h->chol_grid, nullptr, nullptr, h->prof ? h->ev + 8 : nullptr);
  if (cudaMemcpyAsync(inf.data(), info_ws, n_scen * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check(h, "pf_condensed_kkt_solve_reg");
  for (;;) {
    // next trial: the failed scenarios whose next δ_w stays within δ_max (K̂ and rhs were left untouched)
    idx.clear();
    std::vector<double> dv;
    for (int s = 0; s < n_scen; ++s) {
      if (!inf[s]) continue;
      const double nd = delta[s] == 0.0 ? delta_first : delta[s] * growth;
      if (nd > delta_max) continue;
      delta[s] = nd;
      ++tr[s];
      idx.push_back(s);
      dv.push_back(nd);
    }
    if (idx.empty()) break;
    const int nv = (int)idx.size();
    if (cudaMemcpyAsync(h->w.csidx, idx.data(), nv * sizeof(int), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(h->w.cdelta, dv.data(), nv * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return cuda_check(h, "pf_condensed_kkt_solve_reg");
    h->launches += launch_chol(h->dn, h->w, nv, K, sigma_u, 0.0, rhs, nrhs, nullptr, info_ws, st, h->chol_grid,
                               h->w.csidx, h->w.cdelta);
    if (cudaMemcpyAsync(got.data(), info_ws, nv * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return cuda_check(h, "pf_condensed_kkt_solve_reg");
    for (int v = 0; v < nv; ++v) inf[idx[v]] = got[v];
  }
  for (int s = 0; s < n_scen; ++s) {
    if (delta_out) delta_out[s] = delta[s];
    if (trials) trials[s] = tr[s];
    if (info) info[s] = inf[s];
  }
  return cuda_check(h, "pf_condensed_kkt_solve_reg");
}

#ifdef PF_SWEEP_TRACE  // debug builds only (tools/sweep_trace.py)
int pf_debug_set_sweep_trace(void* dev_ptr) {
  pf::set_sweep_trace(static_cast<unsigned long long*>(dev_ptr));
  return 0;
}
#endif

#ifdef PF_LU_TRACE  // debug builds only (tools/lu_trace.py)
int pf_debug_set_lu_trace(void* dev_ptr) {
  pf::set_lu_trace(static_cast<unsigned long long*>(dev_ptr));
  return 0;
}
#endif

pf_status pf_profile(pf_net* h, int32_t enable) {
  if (!h) return PF_ERR_ARG;
  if (!set_device(h)) return h->device < 0 ? PF_ERR_STATE : PF_ERR_CUDA;
  if (enable && !h->ev[0])
    for (auto& e : h->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return cuda_check(h, "pf_profile");
  h->prof = enable != 0;
  return PF_OK;
}

int32_t pf_kernel_times(pf_net* h, float* ms, int32_t cap) {
  if (!h || !h->prof || !ms) return 0;
  const int pairs[7][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {5, 6}, {4, 7}, {8, 9}};
  int k = 0;
  for (; k < 7 && k < cap; ++k) {
    float t = -1.0f;
    if (cudaEventSynchronize(h->ev[pairs[k][1]]) == cudaSuccess &&
        cudaEventElapsedTime(&t, h->ev[pairs[k][0]], h->ev[pairs[k][1]]) != cudaSuccess)
      t = -1.0f;
    ms[k] = t;
  }
  cudaGetLastError();
  return k;
}

}  // extern "C"
