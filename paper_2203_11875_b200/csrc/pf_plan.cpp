// pf_plan.cpp — host structural analysis (A1): validation,
// partition (§8.0), CSR patterns (R19: topological, sorted int32 columns),
// the static symmetric bus-level minimum-degree ordering (R18), the block
// symbolic LU, the numeric-refactorization update lists and level sets.
#include "pf_plan.h"

#include <algorithm>
#include <functional>
#include <queue>
#include <set>

namespace pf {

namespace {

int find_in_row(const std::vector<int>& ptr, const std::vector<int>& idx, int row, int col) {
  auto b = idx.begin() + ptr[row], e = idx.begin() + ptr[row + 1];
  auto it = std::lower_bound(b, e, col);
  if (it == e || *it != col) return -1;
  return (int)(it - idx.begin());
}

}  // namespace

// k_lu's schedule (A5).  (1) The dense front: the rows of levels ≥ fr_lev, the lowest cut that
// leaves at most kFrontMax rows, ascending permuted index.  The set is closed upwards (a row's
// L pivots lie in lower levels), so no row outside the front has a front pivot.  (2) Below
// lu_lev0 the bottom subtrees of the block elimination forest (a block's parent is the block of
// its last row's first L-column successor), balanced over kLuPairs warp pairs: the deepest cut
// ≤ fr_lev whose largest pair load stays within PF_LU_IMB % of the mean; each pair's subtrees in
// postorder (children first).  (3) For the levels between, each level's blocks with the longest
// rows first (only the low pairs have SMEM staging areas).
void lu_schedule(Plan& P) {
  const int n_x = P.n_x, nblk = (int)P.blk_bus.size(), nlev = (int)P.levL_ptr.size() - 1;
  std::vector<int> row_lev(n_x, 0), blk_lev(nblk, 0), cnt_ge(nlev + 1, 0);
  for (int l = 0; l < nlev; ++l)
    for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
      const int b = P.levL_blk[bi];
      blk_lev[b] = l;
      for (int r = P.blk_ptr[b]; r < P.blk_ptr[b + 1]; ++r) row_lev[r] = l;
    }
  for (int r = 0; r < n_x; ++r) ++cnt_ge[row_lev[r]];
  for (int l = nlev - 1; l >= 0; --l) cnt_ge[l] += cnt_ge[l + 1];
  int cut = nlev;
  while (cut > 0 && cnt_ge[cut - 1] <= kFrontMax) --cut;
  P.fr_lev = cut;
  P.fr_row.clear();
  for (int r = 0; r < n_x; ++r) if (row_lev[r] >= cut) P.fr_row.push_back(r);
  // block elimination forest
  std::vector<int> parent(n_x, -1), bpar(nblk, -1);
  for (int r = 0; r < n_x; ++r)
    for (int e = P.lu_ptr[r]; e < P.lu_diag[r]; ++e)
      if (parent[P.lu_idx[e]] < 0) parent[P.lu_idx[e]] = r;
  for (int b = 0; b < nblk; ++b) {
    const int last = P.blk_ptr[b + 1] - 1;
    if (parent[last] >= 0) bpar[b] = P.row_blk[parent[last]];
  }
  const int nteam = kLuPairs;
  std::vector<int> root(nblk);
  P.lu_lev0 = 0;
  P.lu_p1_blk.clear();
  P.lu_p1_ptr.assign(nteam + 1, 0);
  for (int lev0 = 1; lev0 <= cut; ++lev0) {
    for (int l = lev0 - 1; l >= 0; --l)
      for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
        const int b = P.levL_blk[bi], q = bpar[b];
        root[b] = (q >= 0 && blk_lev[q] < lev0) ? root[q] : b;
      }
    std::vector<std::vector<int>> kids(nblk);
    std::vector<int> roots, size(nblk, 1);
    for (int l = 0; l < lev0; ++l)
      for (int bi = P.levL_ptr[l]; bi < P.levL_ptr[l + 1]; ++bi) {
        const int b = P.levL_blk[bi];
        if (root[b] == b) roots.push_back(b); else kids[bpar[b]].push_back(b);
      }
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
    long long tot = 0, mx = 0;
    for (long long x : load) { tot += x; mx = std::max(mx, x); }
    if (lev0 > 1 && mx * 100 > tot * (100 + PF_LU_IMB) / nteam) break;
    std::vector<int> order, ptr(nteam + 1, 0);
    for (int t = 0; t < nteam; ++t) {
      for (int r : mine[t]) {  // iterative postorder of the subtree of r
        std::vector<std::pair<int, size_t>> st{{r, 0}};
        while (!st.empty()) {
          auto& top = st.back();
          if (top.second < kids[top.first].size()) {
            const int ch = kids[top.first][top.second++];
            st.push_back({ch, 0});
          } else {
            order.push_back(top.first);
            st.pop_back();
          }
        }
      }
      ptr[t + 1] = (int)order.size();
    }
    P.lu_p1_blk.swap(order); P.lu_p1_ptr.swap(ptr); P.lu_lev0 = lev0;
  }
  P.lu_lev_blk = P.levL_blk;
  auto piv = [&](int b) {
    int m = 0;
    for (int r = P.blk_ptr[b]; r < P.blk_ptr[b + 1]; ++r) m = std::max(m, P.lu_diag[r] - P.lu_ptr[r]);
    return m;
  };
  for (int l = 0; l < nlev; ++l)
    std::stable_sort(P.lu_lev_blk.begin() + P.levL_ptr[l], P.lu_lev_blk.begin() + P.levL_ptr[l + 1],
                     [&](int x, int y) { return piv(x) > piv(y); });
}

std::string build_plan(int n_b, int n_l, int n_g, const int32_t* lf, const int32_t* lt,
                       const int32_t* gen_bus, int ref_bus, const double* F_max, Plan& P,
                       bool* topology) {
  *topology = false;
  if (n_b < 2 || n_l < 1 || n_g < 1) return "n_b >= 2, n_l >= 1, n_g >= 1 required";
  auto topo = [&](const std::string& s) { *topology = true; return s; };
  if (ref_bus < 0 || ref_bus >= n_b) return topo("reference bus out of range");
  for (int l = 0; l < n_l; ++l) {
    if (lf[l] < 0 || lf[l] >= n_b || lt[l] < 0 || lt[l] >= n_b) return topo("line endpoint out of range");
    if (lf[l] == lt[l]) return topo("self-loop line");
  }
  std::vector<int> gcount(n_b, 0);
  P.bus_gen.assign(n_b, -1);
  for (int g = 0; g < n_g; ++g) {
    if (gen_bus[g] < 0 || gen_bus[g] >= n_b) return topo("generator bus out of range");
    gcount[gen_bus[g]]++;
    P.bus_gen[gen_bus[g]] = g;
  }
  if (gcount[ref_bus] != 1) return topo("reference bus must host exactly one generator");
  for (int i = 0; i < n_b; ++i)
    if (gcount[i] > 1) return topo("more than one generator on a bus (R21)");

  P.n_b = n_b; P.n_l = n_l; P.n_g = n_g; P.r0 = ref_bus; P.g_r = P.bus_gen[ref_bus];

  // adjacency + connectivity
  std::vector<std::vector<int>> adj(n_b);
  for (int l = 0; l < n_l; ++l) { adj[lf[l]].push_back(lt[l]); adj[lt[l]].push_back(lf[l]); }
  for (auto& a : adj) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
  {
    std::vector<char> seen(n_b, 0);
    std::vector<int> st{ref_bus};
    seen[ref_bus] = 1;
    int cnt = 1;
    while (!st.empty()) {
      int i = st.back(); st.pop_back();
      for (int j : adj[i]) if (!seen[j]) { seen[j] = 1; ++cnt; st.push_back(j); }
    }
    if (cnt != n_b) return topo("disconnected grid");
  }

  // ---------------- partition
  P.x_th.assign(n_b, -1); P.x_v.assign(n_b, -1); P.u_v.assign(n_b, -1); P.u_p.assign(n_g, -1);
  int k = 0;
  for (int i = 0; i < n_b; ++i) if (i != ref_bus) P.x_th[i] = k++;
  for (int i = 0; i < n_b; ++i) if (gcount[i] == 0) P.x_v[i] = k++;
  P.n_x = k;
  k = 0;
  for (int i = 0; i < n_b; ++i) if (gcount[i] > 0) P.u_v[i] = k++;
  P.n_gb = k;
  for (int g = 0; g < n_g; ++g) if (g != P.g_r) P.u_p[g] = k++;
  P.n_u = k;
  P.bus_rP.assign(n_b, -1); P.bus_rQ.assign(n_b, -1);
  P.bus_rP[ref_bus] = 0; P.bus_rQ[ref_bus] = 1;
  int nr = 2;
  for (int i = 0; i < n_b; ++i) if (gcount[i] > 0 && i != ref_bus) P.bus_rQ[i] = nr++;
  P.n_r = nr;
  P.line_hf.assign(n_l, -1); P.line_ht.assign(n_l, -1);
  int nlim = 0;
  for (int l = 0; l < n_l; ++l) if (F_max[l] > 0) ++nlim;
  P.n_h = 2 * nlim;
  P.h_line.resize(P.n_h); P.h_end.resize(P.n_h);
  int q = 0;
  for (int l = 0; l < n_l; ++l) if (F_max[l] > 0) {
    P.line_hf[l] = q; P.line_ht[l] = q + nlim; P.h_line[q] = l; P.h_end[q] = 0;
    P.h_line[q + nlim] = l; P.h_end[q + nlim] = 1; ++q;
  }
  P.m = P.n_r + P.n_h;
  const int n_u = P.n_u, n_x = P.n_x;
  auto zv = [&](int i) { return P.u_v[i] >= 0 ? P.u_v[i] : n_u + P.x_v[i]; };
  auto zth = [&](int i) { return P.x_th[i] >= 0 ? n_u + P.x_th[i] : -1; };

  // ---------------- incidence (ascending line per bus)
  P.inc_ptr.assign(n_b + 1, 0);
  for (int l = 0; l < n_l; ++l) { P.inc_ptr[lf[l] + 1]++; P.inc_ptr[lt[l] + 1]++; }
  for (int i = 0; i < n_b; ++i) P.inc_ptr[i + 1] += P.inc_ptr[i];
  P.inc_line.resize(2 * n_l);
  {
    std::vector<int> fill(P.inc_ptr.begin(), P.inc_ptr.end() - 1);
    for (int l = 0; l < n_l; ++l) { P.inc_line[fill[lf[l]]++] = l; P.inc_line[fill[lt[l]]++] = l; }
  }

  // ---------------- J_bus pattern
  P.jb_ptr.assign(2 * n_b + 1, 0);
  std::vector<std::vector<int>> jrow(n_b);
  for (int i = 0; i < n_b; ++i) {
    std::vector<int>& r = jrow[i];
    auto add = [&](int j) { r.push_back(zv(j)); if (zth(j) >= 0) r.push_back(zth(j)); };
    add(i);
    for (int j : adj[i]) add(j);
    std::sort(r.begin(), r.end());
  }
  for (int t = 0; t < 2; ++t)
    for (int i = 0; i < n_b; ++i) P.jb_ptr[t * n_b + i + 1] = (int)jrow[i].size();
  for (int r = 0; r < 2 * n_b; ++r) P.jb_ptr[r + 1] += P.jb_ptr[r];
  P.jb_idx.resize(P.jb_ptr[2 * n_b]);
  for (int t = 0; t < 2; ++t)
    for (int i = 0; i < n_b; ++i)
      std::copy(jrow[i].begin(), jrow[i].end(), P.jb_idx.begin() + P.jb_ptr[t * n_b + i]);
  auto off_in = [&](int i, int z) {
    if (z < 0) return -1;
    auto it = std::lower_bound(jrow[i].begin(), jrow[i].end(), z);
    return (int)(it - jrow[i].begin());
  };
  P.jb_self_th.resize(n_b); P.jb_self_v.resize(n_b);
  for (int i = 0; i < n_b; ++i) { P.jb_self_th[i] = off_in(i, zth(i)); P.jb_self_v[i] = off_in(i, zv(i)); }
  P.inc_off_th.resize(2 * n_l); P.inc_off_v.resize(2 * n_l);
  for (int i = 0; i < n_b; ++i)
    for (int e = P.inc_ptr[i]; e < P.inc_ptr[i + 1]; ++e) {
      int l = P.inc_line[e];
      int j = lf[l] == i ? lt[l] : lf[l];
      P.inc_off_th[e] = off_in(i, zth(j));
      P.inc_off_v[e] = off_in(i, zv(j));
    }

  // ---------------- G_x, G_u (rows = x index)
  std::vector<int> xrow_bus(n_x), xrow_type(n_x);
  for (int i = 0; i < n_b; ++i) {
    if (P.x_th[i] >= 0) { xrow_bus[P.x_th[i]] = i; xrow_type[P.x_th[i]] = 0; }
    if (P.x_v[i] >= 0) { xrow_bus[P.x_v[i]] = i; xrow_type[P.x_v[i]] = 1; }
  }
  P.gx_ptr.assign(n_x + 1, 0); P.gu_ptr.assign(n_x + 1, 0);
  for (int r = 0; r < n_x; ++r) {
    int i = xrow_bus[r], jr = xrow_type[r] * n_b + i;
    for (int e = P.jb_ptr[jr]; e < P.jb_ptr[jr + 1]; ++e) {
      int z = P.jb_idx[e];
      if (z >= n_u) { P.gx_idx.push_back(z - n_u); P.gx_src.push_back(e); }
      else { P.gu_idx.push_back(z); P.gu_src.push_back(e); }
    }
    int g = P.bus_gen[i];
    if (xrow_type[r] == 0 && g >= 0 && P.u_p[g] >= 0) { P.gu_idx.push_back(P.u_p[g]); P.gu_src.push_back(-1); }
    P.gx_ptr[r + 1] = (int)P.gx_idx.size();
    P.gu_ptr[r + 1] = (int)P.gu_idx.size();
  }

  // ---------------- A = [r rows (J_bus rows); h rows (line-local)]
  P.a_ptr.assign(P.m + 1, 0);
  for (int rr = 0; rr < P.n_r; ++rr) {
    int i, t;
    if (rr == 0) { i = ref_bus; t = 0; }
    else if (rr == 1) { i = ref_bus; t = 1; }
    else { i = -1; t = 1; }
    if (rr >= 2) { for (int b = 0; b < n_b; ++b) if (P.bus_rQ[b] == rr) { i = b; break; } }
    int jr = t * n_b + i;
    for (int e = P.jb_ptr[jr]; e < P.jb_ptr[jr + 1]; ++e) { P.a_idx.push_back(P.jb_idx[e]); P.a_src.push_back(e); }
    P.a_ptr[rr + 1] = (int)P.a_idx.size();
  }
  P.ah_off.assign(4 * P.n_h, -1);
  for (int h = 0; h < P.n_h; ++h) {
    int l = P.h_line[h];
    int loc[4] = {zv(lf[l]), zv(lt[l]), zth(lf[l]), zth(lt[l])};
    std::vector<int> cols;
    for (int c : loc) if (c >= 0) cols.push_back(c);
    std::sort(cols.begin(), cols.end());
    for (int a = 0; a < 4; ++a)
      if (loc[a] >= 0) P.ah_off[4 * h + a] = (int)(std::lower_bound(cols.begin(), cols.end(), loc[a]) - cols.begin());
    for (int c : cols) { P.a_idx.push_back(c); P.a_src.push_back(-1); }
    P.a_ptr[P.n_r + h + 1] = (int)P.a_idx.size();
  }

  // ---------------- R18: exact minimum degree on the bus elimination graph
  // (buses with state variables = all but the reference), ties to the lowest
  // bus index; eliminating a bus joins its remaining neighbours into a clique.
  std::vector<std::set<int>> g(n_b);
  for (int i = 0; i < n_b; ++i)
    if (i != ref_bus)
      for (int j : adj[i]) if (j != ref_bus) g[i].insert(j);
  typedef std::pair<int, int> DI;
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap;
  for (int i = 0; i < n_b; ++i) if (i != ref_bus) heap.push(DI((int)g[i].size(), i));
  std::vector<char> done(n_b, 0);
  std::vector<std::vector<int>> nbr_elim(n_b);
  while (!heap.empty()) {
    DI top = heap.top(); heap.pop();
    int i = top.second;
    if (done[i] || top.first != (int)g[i].size()) continue;
    done[i] = 1;
    P.bus_order.push_back(i);
    std::vector<int> nb(g[i].begin(), g[i].end());
    nbr_elim[i] = nb;
    for (int a : nb) {
      g[a].erase(i);
      for (int b : nb) if (b != a) g[a].insert(b);
    }
    g[i].clear();
    for (int a : nb) heap.push(DI((int)g[a].size(), a));
  }
  const int nblk = (int)P.bus_order.size();
  std::vector<int> bus_pos(n_b, -1);
  for (int p = 0; p < nblk; ++p) bus_pos[P.bus_order[p]] = p;

  // permutation: each bus block = θ then v
  P.blk_ptr.assign(nblk + 1, 0);
  P.blk_bus = P.bus_order;
  for (int p = 0; p < nblk; ++p) {
    int i = P.bus_order[p];
    P.perm.push_back(P.x_th[i]);
    if (P.x_v[i] >= 0) P.perm.push_back(P.x_v[i]);
    P.blk_ptr[p + 1] = (int)P.perm.size();
  }
  P.iperm.assign(n_x, -1);
  for (int r = 0; r < n_x; ++r) P.iperm[P.perm[r]] = r;
  P.row_blk.resize(n_x);
  for (int p = 0; p < nblk; ++p) for (int r = P.blk_ptr[p]; r < P.blk_ptr[p + 1]; ++r) P.row_blk[r] = p;

  // block symbolic LU: U blocks of p = p ∪ N(p) (neighbours at elimination),
  // L blocks of p = {q < p : p ∈ N(q)}.
  std::vector<std::vector<int>> Ublk(nblk), Lblk(nblk);
  for (int p = 0; p < nblk; ++p) {
    for (int b : nbr_elim[P.bus_order[p]]) Ublk[p].push_back(bus_pos[b]);
    std::sort(Ublk[p].begin(), Ublk[p].end());
    for (int qb : Ublk[p]) Lblk[qb].push_back(p);
  }
  P.lu_ptr.assign(n_x + 1, 0);
  for (int p = 0; p < nblk; ++p) {
    std::vector<int> cols;
    for (int qb : Lblk[p]) for (int c = P.blk_ptr[qb]; c < P.blk_ptr[qb + 1]; ++c) cols.push_back(c);
    for (int c = P.blk_ptr[p]; c < P.blk_ptr[p + 1]; ++c) cols.push_back(c);
    for (int qb : Ublk[p]) for (int c = P.blk_ptr[qb]; c < P.blk_ptr[qb + 1]; ++c) cols.push_back(c);
    for (int r = P.blk_ptr[p]; r < P.blk_ptr[p + 1]; ++r) {
      P.lu_idx.insert(P.lu_idx.end(), cols.begin(), cols.end());
      P.lu_ptr[r + 1] = (int)P.lu_idx.size();
    }
  }
  const int nnz = (int)P.lu_idx.size();
  P.lu_diag.resize(n_x);
  for (int r = 0; r < n_x; ++r) P.lu_diag[r] = find_in_row(P.lu_ptr, P.lu_idx, r, r);
  P.lu_src.assign(nnz, -1);
  P.lu_tpos.assign(nnz, -1);
  for (int r = 0; r < n_x; ++r)
    for (int e = P.lu_ptr[r]; e < P.lu_ptr[r + 1]; ++e) {
      int c = P.lu_idx[e];
      int gpos = find_in_row(P.gx_ptr, P.gx_idx, P.perm[r], P.perm[c]);
      if (gpos >= 0) P.lu_src[e] = P.gx_src[gpos];
      P.lu_tpos[e] = find_in_row(P.lu_ptr, P.lu_idx, c, r);
    }
  // IKJ update lists: for L entry (r,k): for j in U(k), j > k: w[r,j] -= l_rk u_kj
  P.upd_ptr.assign(nnz + 1, 0);
  for (int r = 0; r < n_x; ++r)
    for (int e = P.lu_ptr[r]; e < P.lu_ptr[r + 1]; ++e) {
      int kk = P.lu_idx[e];
      if (kk < r)
        for (int s = P.lu_diag[kk] + 1; s < P.lu_ptr[kk + 1]; ++s)
        {
          P.upd_dst.push_back(find_in_row(P.lu_ptr, P.lu_idx, r, P.lu_idx[s]) - P.lu_ptr[r]);  // offset in row r
          P.upd_src.push_back(s);  // the U value u_kj (lu index)
        }
      P.upd_ptr[e + 1] = (int)P.upd_dst.size();
    }
  for (int d : P.upd_dst) if (d < 0) return "internal error: fill pattern not closed";
  for (int r = 0; r < n_x; ++r) P.lu_maxlen = std::max(P.lu_maxlen, P.lu_ptr[r + 1] - P.lu_ptr[r]);

  // level sets (longest path in the block DAGs)
  std::vector<int> levL(nblk, 0), levU(nblk, 0);
  int maxL = 0, maxU = 0;
  for (int p = 0; p < nblk; ++p) {
    for (int qb : Lblk[p]) levL[p] = std::max(levL[p], levL[qb] + 1);
    maxL = std::max(maxL, levL[p]);
  }
  for (int p = nblk - 1; p >= 0; --p) {
    for (int qb : Ublk[p]) levU[p] = std::max(levU[p], levU[qb] + 1);
    maxU = std::max(maxU, levU[p]);
  }
  auto sets = [&](const std::vector<int>& lev, int mx, std::vector<int>& ptr, std::vector<int>& blk) {
    ptr.assign(mx + 2, 0);
    for (int p = 0; p < nblk; ++p) ptr[lev[p] + 1]++;
    for (int l = 0; l <= mx; ++l) ptr[l + 1] += ptr[l];
    blk.resize(nblk);
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int p = 0; p < nblk; ++p) blk[fill[lev[p]]++] = p;
  };
  sets(levL, maxL, P.levL_ptr, P.levL_blk);
  sets(levU, maxU, P.levU_ptr, P.levU_blk);

  // G_u in permuted rows
  const int nnz_gu = (int)P.gu_idx.size();
  P.gur_ptr.assign(n_x + 1, 0);
  for (int r = 0; r < n_x; ++r) {
    int xr = P.perm[r];
    for (int e = P.gu_ptr[xr]; e < P.gu_ptr[xr + 1]; ++e) { P.gur_col.push_back(P.gu_idx[e]); P.gur_src.push_back(e); }
    P.gur_ptr[r + 1] = (int)P.gur_col.size();
  }
  P.guc_ptr.assign(n_u + 1, 0);
  for (int e = 0; e < nnz_gu; ++e) P.guc_ptr[P.gur_col[e] + 1]++;
  for (int c = 0; c < n_u; ++c) P.guc_ptr[c + 1] += P.guc_ptr[c];
  P.guc_row.resize(nnz_gu); P.guc_src.resize(nnz_gu);
  {
    std::vector<int> fill(P.guc_ptr.begin(), P.guc_ptr.end() - 1);
    for (int r = 0; r < n_x; ++r)  // ascending permuted row within each column
      for (int e = P.gur_ptr[r]; e < P.gur_ptr[r + 1]; ++e) {
        int c = P.gur_col[e];
        P.guc_row[fill[c]] = r; P.guc_src[fill[c]] = P.gur_src[e]; fill[c]++;
      }
  }
  lu_schedule(P);
  P.hvp_bus = P.bus_order;
  P.hvp_bus.push_back(ref_bus);
  P.bus_pth.assign(n_b, -1); P.bus_pv.assign(n_b, -1);
  for (int i = 0; i < n_b; ++i) {
    if (P.x_th[i] >= 0) P.bus_pth[i] = P.iperm[P.x_th[i]];
    if (P.x_v[i] >= 0) P.bus_pv[i] = P.iperm[P.x_v[i]];
  }
  return "";
}

}  // namespace pf
