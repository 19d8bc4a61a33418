"""GPU parity of the NEXT rows through the C-ABI:

* NEXT-1 — pf_condensed_rhs (Theorem 1's r̂ and Theorem 2's right-hand side,
  R10) and pf_recover_step (Algorithm 1's dual / slack / state / adjoint
  steps) against the oracle's dense step-by-step formulas (themselves pinned
  against a direct K_aug solve, tests/test_oracle_pins.py), plus the GPU step's
  own K_aug residual on the small cases;
* NEXT-2 — pf_power_flow (Newton–Raphson, Algorithm 2's projection) against
  the oracle's dense Newton, the 2-bus closed form (P2), the WSCC textbook
  solution (P17) and constructive exact points of the Table-1 shapes from a
  flat start; pf_reduced_gradient (λ and ∇f_r) against the oracle.
Tolerance: 1e-10 relative, normwise per output block (R20); the condensed
solve's p_u carries cond(K_cond)·ε (its blocks downstream are then checked
from the GPU's own p_u, so the recovery map itself is held to 1e-10)."""
import numpy as np
import pytest

from oracle import pf_oracle as O
from synth import case9, make_scenario
from synth.case9 import case9_multipliers
from synth.grid import table1_grid
from tests.gpu_common import TOL, cond2_spd, dev, record, rel_err, stack
from tests.nets import rich_small, two_bus

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pfmod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2203_11875_b200 import _build
    _build.build()
    import paper_2203_11875_b200 as m
    return m


def _case9_point():
    net, pt = case9()
    part = O.partition(net)
    pt, _, _ = O.newton(net, part, pt)
    pt.update(case9_multipliers())
    return net, pt


def _cases(name):
    if name == "case9":
        net, pt = _case9_point()
        return net, [pt]
    if name == "rich8":
        return rich_small()[0], [rich_small()[1]]
    net, pt = table1_grid(name)
    return net, [pt, make_scenario(net, pt, 1)]


@pytest.mark.parametrize("name", ["case9", "rich8", "case118", "case1354"])
def test_condensed_rhs_and_step_recovery(pfmod, name):
    """NEXT-1 end to end on the device: K̂ (pf_reduced_hessian_batch), b
    (pf_condensed_rhs), p_u (pf_condensed_kkt_solve), the full step
    (pf_recover_step) — each vs the oracle's Theorem 1/2 route; on the small
    cases the GPU step also solves K_aug p = −r to round-off."""
    import torch
    net, pts = _cases(name)
    S = len(pts)
    part = O.partition(net)
    n_u, n_x, m = part["n_u"], part["n_x"], part["m"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    L = h.kkt_len()
    assert L == 2 * n_x + n_u + 2 * m
    rng = np.random.default_rng(31)
    r = rng.standard_normal((S, L))
    v, th = dev(stack(pts, "v")), dev(stack(pts, "theta"))
    lam, y, ss, sx = (dev(stack(pts, k)) for k in ("lam", "y", "sigma_s", "sigma_x"))
    pd = dev(stack(pts, "p_d"))
    info = torch.empty(S, dtype=torch.int32, device="cuda")
    h.pf_jacobian(S, v, th, info=info)
    KV = torch.empty(S, n_u, n_u, dtype=torch.float64, device="cuda")
    h.pf_reduced_hessian_batch(S, v, th, lam, y, KV, sigma_s=ss, sigma_x=sx, p_d=pd)
    rd = dev(r)
    b = h.pf_condensed_rhs(S, v, th, lam, y, rd, sigma_s=ss, sigma_x=sx, p_d=pd)
    torch.cuda.synchronize()
    Kh = KV.cpu().numpy()
    bg = b.cpu().numpy()
    delta = 0.0
    oracle = []
    perm, _ = O.permutation(part, O.md_ordering(net, part))
    for s, pt in enumerate(pts):
        Gx, Gu, A = O.jacobians(net, part, pt)
        W = O.lagrangian_hessian(net, part, pt, pt["lam"], pt["y"])
        bo, _, _ = O.condensed_rhs(W, Gx, Gu, A, pt["sigma_x"], pt["sigma_s"], r[s])
        assert rel_err(bg[s], bo) <= TOL, (name, s, rel_err(bg[s], bo))
        Ksym = 0.5 * (Kh[s] + Kh[s].T)
        lmin = np.linalg.eigvalsh(Ksym + np.diag(pt["sigma_u"])).min()
        delta = max(delta, 0.0 if lmin > 0 else -1.5 * lmin + 1.0)
        oracle.append((W, Gx, Gu, A, bo))
    K = KV.clone()
    p_u = b.clone()
    h.pf_condensed_kkt_solve(S, K, dev(stack(pts, "sigma_u")), delta, p_u, 1, info)
    p = h.pf_recover_step(S, v, th, lam, y, rd, p_u, sigma_s=ss, sigma_x=sx, p_d=pd)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * S
    pg = p.cpu().numpy()
    pug = p_u.cpu().numpy()
    for s, pt in enumerate(pts):
        W, Gx, Gu, A, bo = oracle[s]
        Kc = O.condensed(0.5 * (Kh[s] + Kh[s].T), pt["sigma_u"], delta)
        c2 = cond2_spd(Kc)
        # the condensed solve: p_u within cond(K_cond)·ε of the oracle's
        puo = np.linalg.solve(Kc, bo)
        tol_u = max(TOL, 10 * c2 * np.finfo(float).eps)
        assert rel_err(pug[s], puo) <= tol_u, (name, s, rel_err(pug[s], puo), tol_u)
        # the recovery (a linear map of r and p_u) from the GPU's own p_u, every block within
        # max(1e-10, 3 × the measured floor): the scatter of the oracle's recovery with two other,
        # independent LU codes for G_x (SuperLU minimum degree; the R18 static-pivot LU) — p_λ
        # solves with G_xᵀ a vector with heavy cancellation, so it carries κ(G_x)·ε (R20)
        po = O.recover_step(W, Gx, Gu, A, pt["sigma_x"], pt["sigma_s"], r[s], pug[s])
        blocks = lambda v: O.split_kkt(v, n_u, n_x, m)  # noqa: E731
        floor = np.zeros(5)
        for lu in (O.SparseLU(Gx, "mmd"), O.SparseLU(Gx, "static", perm)):
            alt = O.recover_step(W, Gx, Gu, A, pt["sigma_x"], pt["sigma_s"], r[s], pug[s], lu=lu)
            floor = np.maximum(floor, [rel_err(a, o) for a, o in zip(blocks(alt), blocks(po))])
        gates = np.maximum(TOL, 3 * floor)
        errs = [rel_err(a, o) for a, o in zip(blocks(pg[s]), blocks(po))]
        assert np.array_equal(pg[s, :n_u], pug[s])
        assert np.all(np.array(errs) <= gates), (name, s, errs, gates)
        rec = dict(case=name, scenario=s, b_rel_err=float(rel_err(bg[s], bo)), cond2_Kcond=c2,
                   p_u_rel_err=float(rel_err(pug[s], puo)), p_u_tol=tol_u,
                   block_rel_err=dict(zip(("p_u", "p_x", "p_s", "p_lambda", "p_y"), map(float, errs))),
                   block_floor=dict(zip(("p_u", "p_x", "p_s", "p_lambda", "p_y"), map(float, floor))))
        if n_x <= 300:  # brute force: the GPU step solves K_aug p = −r (δ_w on the uu block)
            Ka = O.kaug(W, Gx, Gu, A, pt["sigma_u"] + delta, pt["sigma_x"], pt["sigma_s"])
            res = np.abs(Ka @ pg[s] + r[s]).max() / (np.abs(Ka).max() * np.abs(pg[s]).max() + np.abs(r[s]).max())
            assert res <= 1e-12, res
            rec["kaug_backward_err"] = float(res)
        record("next1_step", **rec)
    h.close()


def test_step_recovery_state_errors(pfmod):
    """The NEXT-1 calls refuse a point other than the last pf_jacobian's."""
    import torch
    net, pts = _cases("case118")
    h = pfmod.Network(net, max_batch=8, max_scen=1)
    pt = pts[0]
    v, th = dev(pt["v"][None]), dev(pt["theta"][None])
    r = torch.zeros(1, h.kkt_len(), dtype=torch.float64, device="cuda")
    with pytest.raises(pfmod.PFError) as e:
        h.pf_condensed_rhs(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), r)
    assert e.value.status == 5
    h.pf_jacobian(1, v, th)
    with pytest.raises(pfmod.PFError) as e:
        h.pf_recover_step(1, v.clone(), th, dev(pt["lam"][None]), dev(pt["y"][None]), r,
                          torch.zeros(1, h.dims["n_u"], dtype=torch.float64, device="cuda"))
    assert e.value.status == 5
    h.close()


# ---------------------------------------------------------------------------- NEXT-2
def test_power_flow_two_bus_closed_form(pfmod):
    """P2: θ₂ = −½ asin(0.1), v₂ = cos(½ asin 0.1) from a flat start."""
    import math
    net, pt = two_bus()
    pt = dict(pt, p_g=np.array([0.5]))
    h = pfmod.Network(net, max_batch=1, max_scen=1)
    v, th = dev(pt["v"][None]), dev(pt["theta"][None])
    it, res, info = h.pf_power_flow(1, v, th, dev(pt["p_g"][None]), dev(pt["q_g"][None]), dev(pt["p_d"][None]),
                                    dev(pt["q_d"][None]), tol=1e-12)
    assert info.tolist() == [0] and res[0] <= 1e-12
    a = 0.5 * math.asin(0.1)
    assert abs(th[0, 1].item() + a) <= 1e-12 and abs(v[0, 1].item() - math.cos(a)) <= 1e-12
    h.close()


def test_power_flow_case9_textbook(pfmod):
    """P17 + O6: from case9's start (generator set points, flat elsewhere) the
    GPU Newton converges (‖g‖∞ ≤ 1e-10) in the oracle's iteration
    count to the oracle's solution (1e-10) and to the WSCC textbook values."""
    net, pt = case9()
    part = O.partition(net)
    ref, it_o, _ = O.newton(net, part, pt, tol=1e-10)
    h = pfmod.Network(net, max_batch=1, max_scen=1)
    v, th = dev(pt["v"][None]), dev(pt["theta"][None])
    it, res, info = h.pf_power_flow(1, v, th, dev(pt["p_g"][None]), dev(pt["q_g"][None]), dev(pt["p_d"][None]),
                                    dev(pt["q_d"][None]), tol=1e-10)
    assert info.tolist() == [0] and res[0] <= 1e-10
    assert it[0] == it_o
    assert rel_err(v[0].cpu().numpy(), ref["v"]) <= 1e-9
    assert np.abs(th[0].cpu().numpy() - ref["theta"]).max() <= 1e-9
    thdeg = np.degrees(th[0].cpu().numpy())
    assert np.allclose(thdeg[1:], [9.280, 4.665, -2.217, -3.687, 1.967, 0.728, 3.720, -3.989], atol=2e-3)
    assert np.allclose(v[0].cpu().numpy()[3:], [1.0258, 1.0127, 1.0324, 1.0159, 1.0258, 0.9956], atol=2e-4)
    record("power_flow", case="case9", iters=int(it[0]), oracle_iters=int(it_o), resid=float(res[0]))
    h.close()


@pytest.mark.parametrize("name", ["case118", "case1354", "case2869"])
def test_power_flow_constructive_points(pfmod, name):
    """SURVEY §8(d) constructive operating points: loads and dispatch set from
    the point by the oracle (p_d = −P_i at PQ buses, p_g = P_i at generator
    buses), so the point x* is an exact power-flow solution; two scenarios
    from a flat start (θ = 0, v = 1 at PQ buses) converge together to their
    own x* (1e-9) with ‖g‖∞ ≤ 1e-10, in the oracle's iteration count."""
    import torch
    net, base = table1_grid(name)
    part = O.partition(net)
    pts, starts = [], []
    for s, pt in enumerate([base, make_scenario(net, base, 1)]):
        p, q = O.injections(net, pt["v"], pt["theta"])
        gb = net["gen_bus"]
        pd = np.where(part["is_gen"], 0.0, -p)
        qd = np.where(part["is_gen"], 0.0, -q)
        pt = dict(pt, p_d=pd, q_d=qd, p_g=p[gb].copy(), q_g=q[gb].copy())
        assert np.abs(O.g_residual(net, part, pt)).max() <= 1e-12
        st = dict(pt, v=np.where(part["is_gen"], pt["v"], 1.0), theta=np.zeros(net["n_b"]))
        pts.append(pt)
        starts.append(st)
    h = pfmod.Network(net, max_batch=1, max_scen=2)
    v, th = dev(stack(starts, "v")), dev(stack(starts, "theta"))
    it, res, info = h.pf_power_flow(2, v, th, dev(stack(pts, "p_g")), dev(stack(pts, "q_g")), dev(stack(pts, "p_d")),
                                    dev(stack(pts, "q_d")), tol=1e-10, max_iter=20)
    torch.cuda.synchronize()
    assert info.tolist() == [0, 0], (info, res)
    for s in range(2):
        _, it_o, _ = O.newton(net, part, starts[s], tol=1e-10)
        assert res[s] <= 1e-10
        assert abs(int(it[s]) - it_o) <= 1, (it, it_o)
        assert np.abs(v[s].cpu().numpy() - pts[s]["v"]).max() <= 1e-9
        assert np.abs(th[s].cpu().numpy() - pts[s]["theta"]).max() <= 1e-9
        record("power_flow", case=name, scenario=s, iters=int(it[s]), oracle_iters=int(it_o), resid=float(res[s]))
    h.close()


@pytest.mark.parametrize("name", ["case9", "case118", "case1354"])
def test_reduced_gradient(pfmod, name):
    """NEXT-2 adjoint step and reduced gradient vs the oracle (R8)."""
    import torch
    net, pts = _cases(name)
    S = len(pts)
    part = O.partition(net)
    h = pfmod.Network(net, max_batch=8, max_scen=S)
    v, th = dev(stack(pts, "v")), dev(stack(pts, "theta"))
    h.pf_jacobian(S, v, th)
    lam = torch.empty(S, part["n_x"], dtype=torch.float64, device="cuda")
    _, g = h.pf_reduced_gradient(S, v, th, dev(stack(pts, "p_g")), dev(stack(pts, "y")), lam=lam,
                                 p_d=dev(stack(pts, "p_d")))
    torch.cuda.synchronize()
    for s, pt in enumerate(pts):
        lo, go = O.reduced_gradient(net, part, pt, pt["y"])
        assert rel_err(lam[s].cpu().numpy(), lo) <= TOL
        assert rel_err(g[s].cpu().numpy(), go) <= TOL
        record("reduced_gradient", case=name, scenario=s, lam_rel_err=float(rel_err(lam[s].cpu().numpy(), lo)),
               grad_rel_err=float(rel_err(g[s].cpu().numpy(), go)))
    h.close()


# ---------------------------------------------------------------------------- NEXT-3
@pytest.mark.parametrize("name", ["case118", "case1354"])
def test_regularized_condensed_solve(pfmod, name):
    """NEXT-3: pf_condensed_kkt_solve_reg runs the paper's δ_w loop for three
    scenarios at once — one PD at δ_w = 0 (large Σ_u), two needing different
    δ_w — with exactly the oracle loop's δ_w, trial count and info, its factor
    and solve (1e-10), and K̂/rhs untouched for a scenario capped by δ_max."""
    import torch
    net, pt = table1_grid(name)
    pts = [pt, make_scenario(net, pt, 1), make_scenario(net, pt, 2)]
    S = 3
    n_u = O.partition(net)["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    v, th = dev(stack(pts, "v")), dev(stack(pts, "theta"))
    h.pf_jacobian(S, v, th)
    KV = torch.empty(S, n_u, n_u, dtype=torch.float64, device="cuda")
    h.pf_reduced_hessian_batch(S, v, th, dev(stack(pts, "lam")), dev(stack(pts, "y")), KV,
                               sigma_s=dev(stack(pts, "sigma_s")), sigma_x=dev(stack(pts, "sigma_x")),
                               p_d=dev(stack(pts, "p_d")))
    torch.cuda.synchronize()
    Kh = KV.cpu().numpy()
    sig = stack(pts, "sigma_u").copy()
    sig[0] += 2 * np.abs(Kh[0]).sum(axis=0).max()       # scenario 0 diagonally dominant: PD at δ_w = 0
    b = np.random.default_rng(17).standard_normal((S, 2, n_u))
    args = dict(delta_init=0.0, delta_first=1e-4, growth=10.0, delta_max=1e12)
    K, rhs = dev(Kh.copy()), dev(b.copy())
    delta, trials, info = h.pf_condensed_kkt_solve_reg(S, K, dev(sig), rhs=rhs, nrhs=2, **args)
    torch.cuda.synchronize()
    Lg, xg = K.cpu().numpy(), rhs.cpu().numpy()
    assert trials[0] == 1 and delta[0] == 0.0
    for s in range(S):
        Kc0 = O.condensed(0.5 * (Kh[s] + Kh[s].T), sig[s], 0.0)
        do, to, io, Lo = O.regularized_cholesky(Kc0, **args)
        assert (delta[s], trials[s], info[s]) == (do, to, io), (s, delta, trials, info, do, to, io)
        assert io == 0
        assert rel_err(Lg[s].T, Lo) <= TOL
        for k in range(2):
            assert rel_err(xg[s, k], O.chol_solve(Lo, b[s, k])) <= TOL
        record("next3_reg", case=name, scenario=s, delta_w=float(do), trials=int(to))
    # δ_max below what scenario 1 needs: it stops failed, K̂ and rhs untouched, the others solve
    cap = delta[1] / 10.0
    K, rhs = dev(Kh.copy()), dev(b.copy())
    d2, t2, i2 = h.pf_condensed_kkt_solve_reg(S, K, dev(sig), rhs=rhs, nrhs=2, **dict(args, delta_max=cap))
    torch.cuda.synchronize()
    assert i2[1] > 0 and d2[1] <= cap
    assert np.array_equal(K.cpu().numpy()[1], Kh[1]) and np.array_equal(rhs.cpu().numpy()[1], b[1])
    assert i2[0] == 0
    h.close()


def test_single_direction_passes_beyond_smem(pfmod):
    """The single-direction passes keep the whole vector in SMEM (k_tri1) only while
    8·n_x ≤ 200 KB; a 13,600-bus grid (n_x = 25,899) takes the tiled one-CTA sweeps
    instead.  Both directions are checked: the adjoint (pf_reduced_gradient: λ and
    ∇f_r against the oracle) and the forward solve (pf_power_flow's Newton
    steps from a perturbed start reach the constructed solution x* to 1e-9 in ≤ 8
    iterations, ‖g‖∞ ≤ 1e-10)."""
    import torch
    from synth.grid import make_grid
    net, pt = make_grid(13600, 18600, 1300, 21)
    part = O.partition(net)
    assert 8 * part["n_x"] > 200 * 1024
    h = pfmod.Network(net, max_batch=1, max_scen=1)
    v, th = dev(pt["v"][None]), dev(pt["theta"][None])
    h.pf_jacobian(1, v, th)
    lam = torch.empty(1, part["n_x"], dtype=torch.float64, device="cuda")
    _, g = h.pf_reduced_gradient(1, v, th, dev(pt["p_g"][None]), dev(pt["y"][None]), lam=lam,
                                 p_d=dev(pt["p_d"][None]))
    torch.cuda.synchronize()
    lo, go = O.reduced_gradient(net, part, pt, pt["y"])
    assert rel_err(lam[0].cpu().numpy(), lo) <= TOL
    assert rel_err(g[0].cpu().numpy(), go) <= TOL
    # forward: constructive point (loads / dispatch from the point), started from a seeded
    # perturbation of x* (1e-3 in v, 2e-3 in θ; Newton's basin on this random grid is smaller
    # than a flat start — tools/newton_probe.py: the same on the k_tri1 path at 12,000 buses);
    # Newton only converges in a few steps if every solve G_x Z = g is right
    p, q = O.injections(net, pt["v"], pt["theta"])
    gb = net["gen_bus"]
    star = dict(pt, p_d=np.where(part["is_gen"], 0.0, -p), q_d=np.where(part["is_gen"], 0.0, -q),
                p_g=p[gb].copy(), q_g=q[gb].copy())
    rng = np.random.default_rng(5)
    v0 = dev(np.where(part["is_gen"], star["v"], star["v"] + 1e-3 * rng.standard_normal(net["n_b"]))[None])
    th0 = dev((star["theta"] + 2e-3 * rng.standard_normal(net["n_b"]) * (np.arange(net["n_b"]) != net["ref_bus"]))[None])
    it, res, info = h.pf_power_flow(1, v0, th0, dev(star["p_g"][None]), dev(star["q_g"][None]),
                                    dev(star["p_d"][None]), dev(star["q_d"][None]), tol=1e-10, max_iter=20)
    torch.cuda.synchronize()
    assert int(info[0]) == 0 and res[0] <= 1e-10 and int(it[0]) <= 8, (it, res, info)
    assert np.abs(v0[0].cpu().numpy() - star["v"]).max() <= 1e-9
    assert np.abs(th0[0].cpu().numpy() - star["theta"]).max() <= 1e-9
    record("beyond_smem", n_x=part["n_x"], lam_rel_err=float(rel_err(lam[0].cpu().numpy(), lo)),
           grad_rel_err=float(rel_err(g[0].cpu().numpy(), go)), newton_iters=int(it[0]), resid=float(res[0]))
    h.close()
