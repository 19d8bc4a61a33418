"""Seeded synthetic power grids shaped like the paper's MATPOWER/PEGASE cases.

Recipe (DESIGN.md §"Input recipe", SURVEY §8(d) "Generator rules"):

* topology: n_b points uniform in the unit square; Euclidean MST of the
  Delaunay triangulation, plus the shortest remaining Delaunay edges, plus
  ⌈0.02 n_ℓ⌉ parallel duplicates of random tree edges (parallel lines);
  line order shuffled and orientation random;
* branches (p.u. on 100 MVA): lines x = 0.02 (d/median d) U[0.8,1.2],
  r = x/U[5,15], b_c = min(0.3, 2x U[0.5,1.5]); 15% transformers (r = b_c = 0,
  x = 0.02 U[0.5,2], tap U[0.95,1.05]); 1% of the other lines phase
  shifters (shift U[-10°,10°], so Y_ft ≠ Y_tf); MATPOWER π-model;
* shunts on 5% of buses;
* generators on n_g distinct buses, the first one drawn is the reference;
* operating point: θ a sum of three plane waves scaled to a 5° maximum line
  angle, θ_ref = 0; v = 1 + 0.02·wave/3 at PQ buses, U[1.00,1.05] at
  generator buses.  Loads and dispatch are drawn independently of the point:
  the hot path is evaluated at IPM iterates, which need not satisfy the power
  flow (r_4 = g(x,u) ≠ 0 in Theorem 1), and neither G_x nor
  any second derivative depends on the loads;
* multipliers / barrier diagonals, IPM-like: λ_P ~ U[1e3,4e3] (marginal-cost
  sized), λ_Q ~ N(0,50²); y_r ~ N(0,0.1²); y_h = 0 on 90% of line ends, U[0,1]
  otherwise; Σ_s ~ logU[1e-2,1e2]; Σ_x ~ logU[1e-3,1e1] on v-states, 0 on θ;
  Σ_u ~ logU[1e-3,1e1].

Only structural counting (which index is a θ/v state, which y is an r/h row)
is used to lay out multiplier vectors; it follows SURVEY §8.0's partition rule.
"""
from __future__ import annotations

import math
import numpy as np
from scipy.spatial import Delaunay
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import minimum_spanning_tree

# PAPER.md Table 1 (L1275–1281): n_b, n_l, n_g
TABLE1 = {
    "case118": (118, 186, 54),
    "case300": (300, 411, 69),
    "case1354": (1354, 1991, 260),
    "case2869": (2869, 4582, 510),
    "case9241": (9241, 16049, 1445),
}


def pi_model(r, x, b, tap, shift):
    """MATPOWER π-model (the paper omits the formulas)."""
    ys = 1.0 / (r + 1j * x)
    t = tap * np.exp(1j * shift)
    Ytt = ys + 0.5j * b
    Yff = Ytt / (tap * tap)
    Yft = -ys / np.conj(t)
    Ytf = -ys / t
    return Yff, Yft, Ytf, Ytt


def counts(n_b, gen_bus, F_max):
    """Partition sizes of SURVEY §8.0 (one generator per generator bus)."""
    n_gb = len(np.unique(gen_bus))
    n_g = len(gen_bus)
    n_pq = n_b - n_gb
    n_x = (n_b - 1) + n_pq
    n_u = n_gb + n_g - 1
    n_lim = int(np.sum(np.asarray(F_max) > 0))
    n_r = 1 + n_gb
    m = n_r + 2 * n_lim
    return dict(n_x=n_x, n_u=n_u, m=m, n_r=n_r, n_h=2 * n_lim, n_pq=n_pq, n_gb=n_gb)


def _wave(rng, pts):
    f = np.zeros(len(pts))
    for _ in range(3):
        kk = rng.uniform(0.5, 2.0, size=2) * rng.choice([-1.0, 1.0], size=2)
        phi = rng.uniform(0, 2 * math.pi)
        f += np.sin(2 * math.pi * (pts @ kk) + phi)
    return f


def _point(rng, pts, line_from, line_to, gen_bus, ref_bus, n_b):
    th = _wave(rng, pts)
    dmax = np.max(np.abs(th[line_from] - th[line_to]))
    th = th * (math.radians(5.0) / dmax)
    th = th - th[ref_bus]
    v = 1.0 + 0.02 * _wave(rng, pts) / 3.0
    v[gen_bus] = rng.uniform(1.00, 1.05, size=len(gen_bus))
    return v, th


def _multipliers(rng, n_b, n_g, cnt, n_l_lim):
    n_x, n_u, m, n_r = cnt["n_x"], cnt["n_u"], cnt["m"], cnt["n_r"]
    lam = np.empty(n_x)
    lam[: n_b - 1] = rng.uniform(1e3, 4e3, size=n_b - 1)          # P rows
    lam[n_b - 1:] = rng.normal(0.0, 50.0, size=n_x - (n_b - 1))   # Q rows
    y = np.empty(m)
    y[:n_r] = rng.normal(0.0, 0.1, size=n_r)
    yh = rng.uniform(0.0, 1.0, size=m - n_r)
    yh[rng.uniform(size=m - n_r) < 0.9] = 0.0
    y[n_r:] = yh
    sigma_s = np.exp(rng.uniform(math.log(1e-2), math.log(1e2), size=m))
    sigma_x = np.zeros(n_x)
    sigma_x[n_b - 1:] = np.exp(rng.uniform(math.log(1e-3), math.log(1e1), size=n_x - (n_b - 1)))
    sigma_u = np.exp(rng.uniform(math.log(1e-3), math.log(1e1), size=n_u))
    return dict(lam=lam, y=y, sigma_s=sigma_s, sigma_x=sigma_x, sigma_u=sigma_u)


def make_grid(n_b, n_l, n_g, seed, parallel_frac=0.02, tr_frac=0.15, ps_frac=0.01, shunt_frac=0.05,
              nolimit_frac=0.0):
    """Build one seeded synthetic network + operating point + multipliers.
    nolimit_frac: fraction of lines given F_max = 0 (no limit, no h rows: R23)."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(size=(n_b, 2))
    tri = Delaunay(pts)
    e = set()
    for s in tri.simplices:
        for a, b in ((s[0], s[1]), (s[1], s[2]), (s[0], s[2])):
            e.add((min(a, b), max(a, b)))
    edges = np.array(sorted(e), dtype=np.int64)
    length = np.linalg.norm(pts[edges[:, 0]] - pts[edges[:, 1]], axis=1)
    W = coo_matrix((length, (edges[:, 0], edges[:, 1])), shape=(n_b, n_b)).tocsr()
    T = minimum_spanning_tree(W).tocoo()
    tree = set((min(a, b), max(a, b)) for a, b in zip(T.row, T.col))
    n_par = int(math.ceil(parallel_frac * n_l)) if n_l > n_b else 0
    n_extra = n_l - n_par - len(tree)
    if n_extra < 0:
        raise ValueError("n_l too small for a connected grid")
    rest = [(l, tuple(ed)) for l, ed in zip(length, edges) if tuple(ed) not in tree]
    rest.sort()
    chosen = sorted(tree) + [ed for _, ed in rest[:n_extra]]
    tree_list = sorted(tree)
    par_idx = rng.choice(len(tree_list), size=n_par, replace=False)
    chosen += [tree_list[i] for i in sorted(par_idx)]
    br = np.array(chosen, dtype=np.int64)
    assert len(br) == n_l
    perm = rng.permutation(n_l)
    br = br[perm]
    flip = rng.uniform(size=n_l) < 0.5
    line_from = np.where(flip, br[:, 1], br[:, 0]).astype(np.int32)
    line_to = np.where(flip, br[:, 0], br[:, 1]).astype(np.int32)

    d = np.linalg.norm(pts[line_from] - pts[line_to], axis=1)
    x = 0.02 * (d / np.median(d)) * rng.uniform(0.8, 1.2, size=n_l)
    r = x / rng.uniform(5, 15, size=n_l)
    b = np.minimum(0.3, 2 * x * rng.uniform(0.5, 1.5, size=n_l))
    tap = np.ones(n_l)
    shift = np.zeros(n_l)
    is_tr = rng.uniform(size=n_l) < tr_frac
    r[is_tr] = 0.0
    b[is_tr] = 0.0
    x[is_tr] = 0.02 * rng.uniform(0.5, 2.0, size=int(is_tr.sum()))
    tap[is_tr] = rng.uniform(0.95, 1.05, size=int(is_tr.sum()))
    is_ps = (~is_tr) & (rng.uniform(size=n_l) < ps_frac)
    shift[is_ps] = np.radians(rng.uniform(-10, 10, size=int(is_ps.sum())))
    Yff, Yft, Ytf, Ytt = pi_model(r, x, b, tap, shift)

    Ysh = np.zeros(n_b, dtype=np.complex128)
    sh = rng.uniform(size=n_b) < shunt_frac
    Ysh[sh] = rng.uniform(0.0, 0.05, size=int(sh.sum())) + 1j * rng.uniform(-0.2, 0.5, size=int(sh.sum()))

    gen_bus = rng.choice(n_b, size=n_g, replace=False).astype(np.int32)
    ref_bus = int(gen_bus[0])
    c_quad = rng.uniform(0.01, 0.1, size=n_g) * 100.0 ** 2
    c_lin = rng.uniform(10, 40, size=n_g) * 100.0
    F_max = rng.uniform(2.0, 6.0, size=n_l)
    if nolimit_frac > 0:
        F_max[rng.uniform(size=n_l) < nolimit_frac] = 0.0

    v, theta = _point(rng, pts, line_from, line_to, gen_bus, ref_bus, n_b)
    p_d = rng.uniform(0.0, 0.6, size=n_b)
    q_d = p_d * rng.uniform(0.2, 0.4, size=n_b)
    p_g = rng.uniform(0.5, 2.0, size=n_g)
    q_g = rng.uniform(-0.5, 0.5, size=n_g)

    net = dict(n_b=n_b, n_l=n_l, n_g=n_g, line_from=line_from, line_to=line_to,
               Y_ff=Yff, Y_ft=Yft, Y_tf=Ytf, Y_tt=Ytt, Y_sh=Ysh,
               gen_bus=gen_bus, ref_bus=ref_bus, p_d=p_d, q_d=q_d, F_max=F_max,
               c_quad=c_quad, c_lin=c_lin, pts=pts, seed=seed)
    cnt = counts(n_b, gen_bus, F_max)
    point = dict(v=v, theta=theta, p_g=p_g, q_g=q_g, p_d=p_d, q_d=q_d)
    point.update(_multipliers(rng, n_b, n_g, cnt, int(np.sum(F_max > 0))))
    return net, point


def make_scenario(net, base_point, s, seed_base=None):
    """Load scenario s: perturb (θ, v) by 0.1·(fresh
    wave field), re-scaled to keep the 5° line cap; fresh loads and duals.
    Topology, ordering and level schedule are shared by all scenarios."""
    seed = (net["seed"] * 1000 + s) if seed_base is None else seed_base + s
    rng = np.random.default_rng(seed)
    pts = net["pts"]
    n_b, n_g = net["n_b"], net["n_g"]
    lf, lt = net["line_from"], net["line_to"]
    th = base_point["theta"] + 0.1 * math.radians(5.0) * _wave(rng, pts) / 3.0
    dmax = np.max(np.abs(th[lf] - th[lt]))
    if dmax > math.radians(5.0):
        th = th * (math.radians(5.0) / dmax)
    th = th - th[net["ref_bus"]]
    v = base_point["v"] + 0.1 * 0.02 * _wave(rng, pts) / 3.0
    v[net["gen_bus"]] = base_point["v"][net["gen_bus"]]
    p_d = rng.uniform(0.0, 0.6, size=n_b)
    q_d = p_d * rng.uniform(0.2, 0.4, size=n_b)
    p_g = rng.uniform(0.5, 2.0, size=n_g)
    q_g = rng.uniform(-0.5, 0.5, size=n_g)
    cnt = counts(n_b, net["gen_bus"], net["F_max"])
    point = dict(v=v, theta=th, p_g=p_g, q_g=q_g, p_d=p_d, q_d=q_d)
    point.update(_multipliers(rng, n_b, n_g, cnt, int(np.sum(net["F_max"] > 0))))
    return point


def table1_grid(name, seed=None):
    n_b, n_l, n_g = TABLE1[name]
    return make_grid(n_b, n_l, n_g, seed if seed is not None else n_b)


def opf_bounds(net, seed=None):
    """Seeded OPF bounds for a synthetic grid (NEXT-4 tests): v ∈ [0.9, 1.1];
    generator p_g ∈ [0, p_hi] with capacities drawn so the fleet covers the
    total load 1.5–2.5×; q_g ∈ [−q_hi, q_hi], q_hi = 0.5 p_hi + 0.3 (p.u.)."""
    rng = np.random.default_rng((net["seed"] if seed is None else seed) + 77)
    n_b, n_g = int(net["n_b"]), int(net["n_g"])
    share = rng.uniform(0.5, 1.5, size=n_g)
    total = float(np.sum(net["p_d"]))
    p_hi = share / share.sum() * total * rng.uniform(1.5, 2.5)
    q_hi = 0.5 * p_hi + 0.3
    return dict(v_lo=np.full(n_b, 0.9), v_hi=np.full(n_b, 1.1), p_lo=np.zeros(n_g), p_hi=p_hi,
                q_lo=-q_hi, q_hi=q_hi)


def opf_feasible(net, point, margin=1.25, seed=None):
    """A feasible-by-construction OPF instance around a synthetic operating point
    (NEXT-4 at scale): the seeded bounds of opf_bounds, with each generator's p_hi
    raised to ≥ margin·p_g and each limited line's F_max raised to ≥ margin·|s| at
    the point (both line ends), so the point itself is strictly feasible.  Returns
    (net copy, bounds).  Only input recipe: no method arithmetic beyond |s|² of the
    π-model flows the caller passes in as point["s_abs"] (per line, max of the ends)."""
    b = opf_bounds(net, seed)
    net2 = dict(net)
    b["p_hi"] = np.maximum(b["p_hi"], margin * np.asarray(point["p_g"]))
    F = np.asarray(net["F_max"], dtype=np.float64).copy()
    lim = F > 0
    F[lim] = np.maximum(F[lim], margin * np.asarray(point["s_abs"])[lim])
    net2["F_max"] = F
    return net2, b
