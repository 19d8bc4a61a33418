"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY §8(c) Table P).  None of these re-type the oracle's formulas: each
compares it with a closed form, a different formula for the same quantity,
finite differences, a brute-force identity, or a library routine."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pf_oracle as O
from synth import TABLE1, case9, counts
from synth.case9 import case9_multipliers
from synth.grid import pi_model, table1_grid
from tests import golden_data
from tests.nets import all_small, rich_small, two_bus


# --------------------------------------------------------------------- P1
def test_table1_dimensions():
    """Table 1 (tests/golden/table1_instances.tsv): n_x, n_u for the BASELINE shapes."""
    want = golden_data.table1()
    assert set(want) == set(TABLE1)
    for name, (n_b, n_l, n_g, nx, nu) in want.items():
        assert TABLE1[name] == (n_b, n_l, n_g), name
        net, _ = table1_grid(name)
        part = O.partition(net)
        assert (part["n_x"], part["n_u"]) == (nx, nu), name
        assert (net["n_b"], net["n_l"], net["n_g"]) == (n_b, n_l, n_g)


def test_case9_counts_and_patterns():
    """SURVEY Table S / App. B: case9 n_x=14, n_u=5, m=22, nnz(G_x)=82, nnz(G_u)=10."""
    net, _ = case9()
    part = O.partition(net)
    assert (part["n_x"], part["n_u"], part["m"]) == (14, 5, 22)
    (px, ix), (pu, iu) = O.gx_gu_patterns(net, part)
    assert len(ix) == 82 and len(iu) == 10


def test_pi_model_examples():
    """SPEC.md L93–95 examples of the MATPOWER π-model (tests/golden/spec_pi_model.txt)."""
    g = golden_data.spec_pi_model()
    r, x, bc, tau, sh = (float(v) for v in g["series_line"][:5])
    want = dict(kv.split("=") for kv in g["series_line"][5:])
    Yff, Yft, Ytf, Ytt = pi_model(np.array([r]), np.array([x]), np.array([bc]), np.array([tau]), np.array([sh]))
    for k, y in zip(("Yff", "Yft", "Ytf", "Ytt"), (Yff, Yft, Ytf, Ytt)):
        assert np.isclose(y[0], golden_data.complex_pair(want[k])), k
    tau2, scale = (float(v) for v in g["tap_ratio_scale"])
    a = pi_model(np.array([0.01]), np.array([0.1]), np.array([0.02]), np.array([1.0]), np.array([0.0]))
    b = pi_model(np.array([0.01]), np.array([0.1]), np.array([0.02]), np.array([tau2]), np.array([0.0]))
    assert np.isclose(b[0][0], a[0][0] / scale)
    ys = 1.0 / complex(0.01, 0.1)  # Y_ff = y_s + j b_c/2
    assert np.isclose(a[0][0], ys + 0.01j)


def test_ybus_two_bus():
    """one series line x = 0.1 → Y_bus = [[−10j, 10j], [10j, −10j]] (tests/golden/spec_pi_model.txt)."""
    net, _ = two_bus()
    want = [golden_data.complex_pair(v) for v in golden_data.spec_pi_model()["two_bus_ybus"]]
    assert np.allclose(O.ybus(net), np.array(want).reshape(2, 2))


# --------------------------------------------------------------------- P2 / P5 / P17
def test_two_bus_closed_form_and_newton():
    """SURVEY P2 closed form derived from eq. powerflow."""
    net, pt = two_bus()
    part = O.partition(net)
    th2 = -0.5 * math.asin(0.1)
    v2 = math.cos(0.5 * math.asin(0.1))
    star = dict(pt, v=np.array([1.0, v2]), theta=np.array([0.0, th2]),
                p_g=np.array([0.5]), q_g=np.array([10 * math.sin(th2) ** 2]))
    assert np.max(np.abs(O.balance(net, star))) < 1e-14
    sol, it, hist = O.newton(net, part, pt)
    assert abs(sol["theta"][1] - th2) < 1e-12 and abs(sol["v"][1] - v2) < 1e-12
    assert hist[-1] <= 1e-12
    # quadratic convergence on the last iterations (P5)
    assert hist[-2] <= 10 * hist[-3] ** 2 + 1e-14


def test_case9_textbook_power_flow():
    """WSCC 9-bus textbook solution (1e-3 level smoke of data + oracle)."""
    net, pt = case9()
    part = O.partition(net)
    sol, it, hist = O.newton(net, part, pt)
    p, q = O.injections(net, sol["v"], sol["theta"])
    g = golden_data.keyed("case9_powerflow.txt")
    assert abs((p[0] + net["p_d"][0]) * 100 - g["p_g1_mw"][0]) < 1e-3
    assert np.allclose((q[:3] + net["q_d"][:3]) * 100, g["q_g_mvar"], atol=1e-3)
    assert np.allclose(sol["v"][3:], g["vm_4_9"], atol=1e-4)
    assert np.allclose(np.degrees(sol["theta"][1:]),
                       [9.280, 4.665, -2.217, -3.687, 1.967, 0.728, 3.720, -3.989], atol=1e-3)


# --------------------------------------------------------------------- P4 identities
@pytest.mark.parametrize("seed", [5, 11])
def test_injections_equal_kirchhoff(seed):
    """Loop form of eq. powerflow (L59–60) = V ⊙ conj(Y_bus V) (Kirchhoff, L45),
    on a grid with taps, a phase shifter, a parallel line and shunts."""
    net, pt = rich_small(seed)
    rng = np.random.default_rng(seed)
    v = 1 + 0.1 * rng.standard_normal(net["n_b"])
    th = 0.2 * rng.standard_normal(net["n_b"])
    V = v * np.exp(1j * th)
    s = V * np.conj(O.ybus(net) @ V)
    p, q = O.injections(net, v, th)
    assert np.max(np.abs(p - s.real)) < 1e-12 and np.max(np.abs(q - s.imag)) < 1e-12


@pytest.mark.parametrize("seed", [5, 11])
def test_line_flows_sum_to_injections(seed):
    """Σ of line flows leaving bus i + shunt = s_i^inj (conservation; pins R1's conj:
    without it the identity fails by O(1))."""
    net, pt = rich_small(seed)
    rng = np.random.default_rng(seed + 1)
    v = 1 + 0.05 * rng.standard_normal(net["n_b"])
    th = 0.1 * rng.standard_normal(net["n_b"])
    sf, st = O.line_flows(net, v, th)
    tot = np.conj(net["Y_sh"]) * v * v
    np.add.at(tot, net["line_from"], sf)
    np.add.at(tot, net["line_to"], st)
    p, q = O.injections(net, v, th)
    assert np.max(np.abs(tot - (p + 1j * q))) < 1e-12


def test_lossless_line_symmetry():
    """Lossless line: s_p^f = −s_p^t."""
    net, _ = two_bus()
    sf, st = O.line_flows(net, np.array([1.02, 0.97]), np.array([0.0, -0.1]))
    assert abs(sf[0].real + st[0].real) < 1e-14


# --------------------------------------------------------------------- P6 finite differences
def _fd_jac(fun, z0, h=1e-6):
    cols = []
    for k in range(len(z0)):
        e = np.zeros_like(z0)
        e[k] = h
        cols.append((fun(z0 + e) - fun(z0 - e)) / (2 * h))
    return np.array(cols).T


def _z_point(part, point, z):
    n_u = part["n_u"]
    return O.set_x(part, O.set_u(part, point, z[:n_u]), z[n_u:])


def _z0(part, point):
    return np.concatenate([O.get_u(part, point), O.get_x(part, point)])


def _rh(net, part, pt):
    p, q = O.injections(net, pt["v"], pt["theta"])
    r = np.array([p[i] if t == 0 else q[i] for (i, t) in part["r_rows"]])
    sf, st = O.line_flows(net, pt["v"], pt["theta"])
    h = np.array([abs(sf[l]) ** 2 if e == 0 else abs(st[l]) ** 2 for (l, e) in part["h_rows"]])
    return np.concatenate([r, h])


@pytest.mark.parametrize("name,net,pt", all_small())
def test_jacobians_vs_fd(name, net, pt):
    """G = [G_u G_x] and A against central FD (h = 1e-6, rel 1e-6)."""
    part = O.partition(net)
    z0 = _z0(part, pt)
    Gx, Gu, A = O.jacobians(net, part, pt)
    Jg = _fd_jac(lambda z: O.g_residual(net, part, _z_point(part, pt, z)), z0)
    Ja = _fd_jac(lambda z: _rh(net, part, _z_point(part, pt, z)), z0)
    G = sp.hstack([Gu, Gx]).toarray()
    assert np.max(np.abs(G - Jg)) <= 1e-6 * max(1.0, np.abs(G).max())
    assert np.max(np.abs(A.toarray() - Ja)) <= 1e-6 * max(1.0, np.abs(A).max())


def _lag_grad(net, part, pt, lam, y):
    Gx, Gu, A = O.jacobians(net, part, pt)
    G = sp.hstack([Gu, Gx])
    return O.objective_gradient(net, part, pt) + G.T @ lam + A.T @ y


@pytest.mark.parametrize("name,net,pt", all_small())
def test_objective_gradient_vs_fd(name, net, pt):
    part = O.partition(net)
    z0 = _z0(part, pt)
    g = O.objective_gradient(net, part, pt)
    fd = _fd_jac(lambda z: np.array([O.objective(net, part, _z_point(part, pt, z))]), z0).ravel()
    assert np.max(np.abs(g - fd)) <= 1e-6 * max(1.0, np.abs(g).max())


@pytest.mark.parametrize("name,net,pt", all_small())
def test_lagrangian_hessian_vs_fd(name, net, pt):
    """W·d against FD of ∇ℒ (rel 1e-5), W symmetric (P6)."""
    part = O.partition(net)
    rng = np.random.default_rng(3)
    lam = pt["lam"] if "lam" in pt and len(pt["lam"]) == part["n_x"] else rng.standard_normal(part["n_x"]) * 100
    y = pt["y"] if "y" in pt and len(pt["y"]) == part["m"] else rng.standard_normal(part["m"])
    y = y + rng.uniform(0, 1, size=len(y))  # make the line-limit multipliers active
    W = O.lagrangian_hessian(net, part, pt, lam, y).toarray()
    z0 = _z0(part, pt)
    fd = _fd_jac(lambda z: _lag_grad(net, part, _z_point(part, pt, z), lam, y), z0)
    assert np.max(np.abs(W - fd)) <= 1e-5 * np.abs(W).max()
    assert np.max(np.abs(W - W.T)) <= 1e-12 * np.abs(W).max()


# --------------------------------------------------------------------- P9 / P10 / P11 / P12
def _case9_solved():
    net, pt = case9()
    part = O.partition(net)
    pt, _, _ = O.newton(net, part, pt, tol=1e-14)
    mult = case9_multipliers()
    y = mult["y"]
    lam = O.adjoint_multipliers(net, part, pt, y)
    return net, part, pt, lam, y, mult


def test_reduced_hessian_fd_through_newton():
    """P9: with σ = 0 and λ the adjoint, K̂ = ∇²_uu[f + yᵀ(r;h)](x(u), u),
    the Hessian of the reduced Lagrangian, by central
    second differences through Newton."""
    net, part, pt, lam, y, _ = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, lam, y)
    Kh = O.reduce_naive(K, Gx, Gu)
    u0 = O.get_u(part, pt)
    n = len(u0)
    h = 1e-4
    fd = np.zeros((n, n))
    phi = lambda u: O.reduced_value(net, part, pt, y, u)
    for i in range(n):
        for j in range(i, n):
            ei = np.zeros(n); ei[i] = h
            ej = np.zeros(n); ej[j] = h
            fd[i, j] = fd[j, i] = (phi(u0 + ei + ej) - phi(u0 + ei - ej) - phi(u0 - ei + ej) + phi(u0 - ei - ej)) / (4 * h * h)
    assert np.max(np.abs(Kh - fd)) <= 2e-6 * np.abs(Kh).max()
    assert np.max(np.abs(Kh - Kh.T)) <= 1e-12 * np.abs(Kh).max()   # P12


def test_reduced_gradient_fd_through_newton():
    """NEXT-2 pin: the adjoint-based reduced gradient equals the central
    finite difference of φ(u) = f + yᵀ[r; h] at x(u) from Newton (the reduced
    objective + constraint term), and λ satisfies the adjoint
    equation G_xᵀλ = −∇_x(f + yᵀ[r;h]) (Algorithm 2)."""
    net, part, pt, lam0, y, _ = _case9_solved()
    lam, g = O.reduced_gradient(net, part, pt, y)
    assert np.abs(lam - lam0).max() <= 1e-12 * np.abs(lam0).max()
    u0 = O.get_u(part, pt)
    h = 1e-5
    fd = np.zeros_like(u0)
    for i in range(len(u0)):
        e = np.zeros_like(u0); e[i] = h
        fd[i] = (O.reduced_value(net, part, pt, y, u0 + e) - O.reduced_value(net, part, pt, y, u0 - e)) / (2 * h)
    assert np.abs(g - fd).max() <= 1e-6 * np.abs(g).max()


def test_reduced_jacobian_term_fd():
    """P9 second part: K̂(σ_s) − K̂(0) = Â_uᵀΣ_sÂ_u with Â_u = ∂[r;h](x(u),u)/∂u by FD through Newton."""
    net, part, pt, lam, y, mult = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    sig = mult["sigma_s"]
    d = O.reduce_naive(O.kkt_K(net, part, pt, lam, y, sigma_s=sig), Gx, Gu) - \
        O.reduce_naive(O.kkt_K(net, part, pt, lam, y), Gx, Gu)
    u0 = O.get_u(part, pt)

    def rh(u):
        p2, _, _ = O.newton(net, part, O.set_u(part, pt, u), tol=1e-14)
        return _rh(net, part, p2)

    Ahat = _fd_jac(rh, u0, h=1e-6)
    ref = Ahat.T @ np.diag(sig) @ Ahat
    assert np.max(np.abs(d - ref)) <= 1e-6 * np.abs(ref).max()


def test_schur_pin_case9():
    """P10: (K_aug^{-1})_uu = (K̂ + Σ_u)^{-1} with K_aug of PAPER.md L626–634
    inverted by Gauss–Jordan (Theorems 1–2, L671–828, with R9)."""
    net, part, pt, lam, y, mult = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    W = O.lagrangian_hessian(net, part, pt, lam, y)
    K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    Kc = O.condensed(O.reduce_naive(K, Gx, Gu), mult["sigma_u"], 0.0)
    Ka = O.kaug(W, Gx, Gu, A, mult["sigma_u"], mult["sigma_x"], mult["sigma_s"])
    inv = O.gauss_jordan_inverse(Ka)
    n_u = part["n_u"]
    ref = np.linalg.inv(Kc)
    assert np.max(np.abs(inv[:n_u, :n_u] - ref)) <= 1e-9 * np.abs(ref).max()


def _next1_problem(name, seed=0):
    """A LinRed iteration's linear algebra on a small instance: W, G_x, G_u, A,
    Σ's, a random right-hand side r and the condensed matrix (δ_w making it PD)."""
    if name == "case9":
        net, part, pt, lam, y, mult = _case9_solved()
    else:
        net, pt = rich_small(seed=5 + seed) if name == "rich8" else table1_grid(name)
        part = O.partition(net)
        lam, y, mult = pt["lam"], pt["y"], pt
    Gx, Gu, A = O.jacobians(net, part, pt)
    W = O.lagrangian_hessian(net, part, pt, lam, y)
    K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    lmin = np.linalg.eigvalsh(O.condensed(Kh, mult["sigma_u"], 0.0)).min()
    delta = 0.0 if lmin > 0 else -2 * lmin + 1.0
    n_u, n_x, m = part["n_u"], part["n_x"], part["m"]
    r = np.random.default_rng(100 + seed).standard_normal(2 * n_x + n_u + 2 * m)
    return dict(W=W, Gx=Gx, Gu=Gu, A=A, Kh=Kh, su=mult["sigma_u"], sx=mult["sigma_x"], ss=mult["sigma_s"],
                delta=delta, r=r, n_u=n_u, n_x=n_x, m=m)


@pytest.mark.parametrize("name,seed", [("case9", 0), ("rich8", 0), ("rich8", 1), ("case118", 0)])
def test_step_recovery_vs_kaug(name, seed):
    """NEXT-1 pin (SURVEY §8(f), S:L356/361/391): the condensed route —
    Theorem 1's r̂ and Theorem 2's K_cond p_u = b (R10 signs), then Algorithm 1's
    dual/slack/state/adjoint steps — equals the direct dense solve of
    K_aug p = −r (eq. kktmatrix:normal) in all five blocks, with
    δ_w added to the uu block; and the r̂₂ sign as printed does not."""
    P = _next1_problem(name, seed)
    n_u = P["n_u"]
    b, (rh1, rh2, rh3), Ahat = O.condensed_rhs(P["W"], P["Gx"], P["Gu"], P["A"], P["sx"], P["ss"], P["r"])
    Kc = O.condensed(P["Kh"], P["su"], P["delta"])
    p_u = np.linalg.solve(Kc, b)
    got = O.recover_step(P["W"], P["Gx"], P["Gu"], P["A"], P["sx"], P["ss"], P["r"], p_u)
    Ka = O.kaug(P["W"], P["Gx"], P["Gu"], P["A"], P["su"] + P["delta"], P["sx"], P["ss"])
    ref = -np.linalg.solve(Ka, P["r"])
    assert np.abs(got - ref).max() <= 1e-8 * np.abs(ref).max()
    for blk_got, blk_ref in zip(O.split_kkt(got, n_u, P["n_x"], P["m"]), O.split_kkt(ref, n_u, P["n_x"], P["m"])):
        assert np.abs(blk_got - blk_ref).max() <= 1e-8 * max(np.abs(blk_ref).max(), 1e-300)
    # K_cond = Ŵ_uu + Σ_u + Â_uᵀΣ_sÂ_u (Theorem 2 with R9): the oracle's K̂ carries Â_uᵀΣ_sÂ_u
    Kc0 = O.condensed(O.reduce_naive(O.kkt_K_from(P["W"], P["A"], None, P["sx"], P["n_u"]), P["Gx"], P["Gu"]),
                      P["su"], P["delta"])
    assert np.abs(Kc0 + Ahat.T @ np.diag(P["ss"]) @ Ahat - Kc).max() <= 1e-10 * np.abs(Kc).max()
    printed = -(rh1 + Ahat.T @ (P["ss"] * rh3) - Ahat.T @ rh2)   # the sign printed in P:L787
    assert np.abs(np.linalg.solve(Kc, printed) - ref[:n_u]).max() > 1e-6 * np.abs(ref[:n_u]).max()


def test_inertia_theorem3():
    """P11: Cholesky of K_cond succeeds ⇔ inertia(K_aug) = (n_x+n_u+m, n_x+m, 0)
    (Theorem 3), over shifts δ straddling PD-ness."""
    net, part, pt, lam, y, mult = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    W = O.lagrangian_hessian(net, part, pt, lam, y)
    K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    base = O.condensed(Kh, mult["sigma_u"], 0.0)
    lmin = np.linalg.eigvalsh(base).min()
    n_u, n_x, m = part["n_u"], part["n_x"], part["m"]
    seen = set()
    for k, frac in enumerate([-3.0, -1.1, -0.9, 0.5, 2.0]):
        delta = -lmin + frac * max(abs(lmin), 1.0)
        su = mult["sigma_u"] + delta
        Kc = O.condensed(Kh, su, 0.0)
        _, info = O.cholesky(Kc)
        Ka = O.kaug(W, Gx, Gu, A, su, mult["sigma_x"], mult["sigma_s"])
        ev = O.jacobi_eigenvalues(Ka) if k < 2 else np.linalg.eigvalsh(Ka)
        tol = 1e-13 * np.abs(ev).max()
        inertia = (int(np.sum(ev > tol)), int(np.sum(ev < -tol)), int(np.sum(np.abs(ev) <= tol)))
        good = inertia == (n_x + n_u + m, n_x + m, 0)
        assert (info == 0) == good
        seen.add(good)
    assert seen == {True, False}


def test_regularized_cholesky_certificate():
    """NEXT-3 pin: the δ_w loop stops at the first δ_w of its geometric
    schedule above −λ_min(K_cond) (eigenvalues), and there K_aug has the
    inertia (n_x+n_u+m, n_x+m, 0) while the previous trial's K_aug does not
    (Theorem 3; Jacobi eigenvalues)."""
    net, part, pt, lam, y, mult = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    W = O.lagrangian_hessian(net, part, pt, lam, y)
    K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    shift = np.linalg.eigvalsh(O.condensed(Kh, mult["sigma_u"], 0.0)).min() + 3.7   # λ_min(K_cond) = −3.7
    base = O.condensed(Kh, mult["sigma_u"] - shift, 0.0)
    lmin = np.linalg.eigvalsh(base).min()
    assert lmin < 0
    delta, trials, info, L = O.regularized_cholesky(base, 0.0, 1e-8, 10.0, 1e12)
    assert info == 0 and trials > 2
    assert delta > -lmin and delta / 10.0 < -lmin
    sched = [0.0] + [1e-8 * 10.0 ** k for k in range(trials - 1)]
    assert np.isclose(delta, sched[trials - 1])
    n_u, n_x, m = part["n_u"], part["n_x"], part["m"]
    want = (n_x + n_u + m, n_x + m, 0)
    for d, ok in ((delta, True), (delta / 10.0, False)):
        Ka = O.kaug(W, Gx, Gu, A, mult["sigma_u"] - shift + d, mult["sigma_x"], mult["sigma_s"])
        ev = O.jacobi_eigenvalues(Ka)
        tol = 1e-13 * np.abs(ev).max()
        inertia = (int(np.sum(ev > tol)), int(np.sum(ev < -tol)), int(np.sum(np.abs(ev) <= tol)))
        assert (inertia == want) == ok
    # δ_max caps the loop: info stays the failing column
    d2, t2, i2, _ = O.regularized_cholesky(base, 0.0, 1e-8, 10.0, delta / 100.0)
    assert i2 > 0 and d2 <= delta / 100.0


def test_jacobi_matches_lapack():
    rng = np.random.default_rng(0)
    M = rng.standard_normal((12, 12))
    M = M + M.T
    assert np.allclose(np.sort(O.jacobi_eigenvalues(M)), np.linalg.eigvalsh(M), atol=1e-10)


# --------------------------------------------------------------------- P7 / P8 reduction routes
def _rand_problem(rng, n_u, n_x):
    Gx = sp.csr_matrix(rng.standard_normal((n_x, n_x)) + n_x * np.eye(n_x))
    Gu = sp.csr_matrix(rng.standard_normal((n_x, n_u)))
    B = rng.standard_normal((n_u + n_x, n_u + n_x))
    K = sp.csr_matrix(B + B.T)
    return K, Gx, Gu


def test_reduction_special_cases():
    """P7: G_u = 0 ⇒ K̂ = K_uu; K = I ⇒ K̂ = I + SᵀS."""
    rng = np.random.default_rng(1)
    K, Gx, Gu = _rand_problem(rng, 4, 7)
    Kh = O.reduce_naive(K, Gx, sp.csr_matrix((7, 4)))
    assert np.allclose(Kh, K.toarray()[:4, :4], atol=1e-14)
    I = sp.identity(11, format="csr")
    S = -np.linalg.solve(Gx.toarray(), Gu.toarray())
    assert np.allclose(O.reduce_naive(I, Gx, Gu), np.eye(4) + S.T @ S, atol=1e-12)


@pytest.mark.parametrize("N", [1, 3, 5])
def test_naive_vs_adjoint_routes(N):
    """P8: the naive-sensitivity route (L1180) and the paper's 3-step
    adjoint-adjoint route with R11 (L1203–1222) agree on case9."""
    net, part, pt, lam, y, mult = _case9_solved()
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    rng = np.random.default_rng(N)
    V = rng.standard_normal((part["n_u"], N))
    KV = O.reduce_adjoint(K, Gx, Gu.toarray(), V)
    assert np.max(np.abs(KV - Kh @ V)) <= 1e-11 * np.abs(Kh @ V).max()


def _khat_inputs(name):
    if name == "case9":
        net, part, pt, lam, y, mult = _case9_solved()
        K = O.kkt_K(net, part, pt, lam, y, mult["sigma_s"], mult["sigma_x"])
    else:
        net, pt = table1_grid(name)
        part = O.partition(net)
        K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
    Gx, Gu, _ = O.jacobians(net, part, pt)
    return K, Gx, Gu, part


def test_reduce_columns_vs_dense_adjoint_case9():
    """reduce_columns (sparse SuperLU solves, the full-size checker) against
    reduce_adjoint (dense LAPACK solves) and reduce_naive on case9, all n_u
    unit directions (P8 with a different solve primitive)."""
    K, Gx, Gu, part = _khat_inputs("case9")
    n_u = part["n_u"]
    got = O.reduce_columns(K, Gx, Gu, np.arange(n_u))
    dense = O.reduce_adjoint(K, Gx, Gu.toarray(), np.eye(n_u))
    naive = O.reduce_naive(K, Gx, Gu)
    assert np.abs(got - dense).max() <= 1e-13 * np.abs(dense).max()
    assert np.abs(got - naive).max() <= 1e-12 * np.abs(naive).max()


@pytest.mark.parametrize("name", ["case118", "case1354"])
@pytest.mark.parametrize("kind", ["colamd", "mmd", "static"])
def test_reduce_columns_vs_naive(name, kind):
    """reduce_columns (adjoint route) with each sparse-LU variant
    vs reduce_naive (sensitivity route): whole K̂ normwise ≤ 1e-10,
    every column ≤ 1e-8 (independent LU codes disagree per column up to ~3e-10
    at 1354, R20), and a scattered column subset equals the same columns of
    the full run (columns are independent)."""
    K, Gx, Gu, part = _khat_inputs(name)
    n_u = part["n_u"]
    perm = None
    if kind == "static":
        net, _ = table1_grid(name)
        perm, _ = O.permutation(part, O.md_ordering(net, part))
    full = O.reduce_columns(K, Gx, Gu, np.arange(n_u), kind, perm)
    naive = O.reduce_naive(K, Gx, Gu)
    assert np.abs(full - naive).max() <= 1e-10 * np.abs(naive).max()
    col = np.abs(full - naive).max(axis=0) / np.abs(naive).max(axis=0)
    assert col.max() <= 1e-8, col.max()
    cols = np.array([n_u - 1, 3, n_u // 2, 0])
    sub = O.reduce_columns(K, Gx, Gu, cols, kind, perm)
    assert np.abs(sub - full[:, cols]).max() <= 1e-14 * np.abs(full).max()


def test_static_sparse_lu_is_r18():
    """SparseLU("static") is the R18 factorization: SuperLU keeps the natural
    order and the diagonal pivots of P G_x Pᵀ, and its U equals the dense
    no-pivot LU (static_lu) of the same matrix."""
    net, pt = table1_grid("case118")
    part = O.partition(net)
    Gx, _, _ = O.jacobians(net, part, pt)
    perm, _ = O.permutation(part, O.md_ordering(net, part))
    lu = O.SparseLU(Gx, "static", perm)
    info, LU = O.static_lu(Gx, perm)
    assert info == 0
    U = np.triu(LU)
    assert np.abs(lu.lu.U.toarray() - U).max() <= 1e-13 * np.abs(U).max()
    b = np.random.default_rng(1).standard_normal(len(perm))
    assert np.abs(Gx @ lu.solve(b) - b).max() <= 1e-12 * np.abs(b).max()
    assert np.abs(Gx.T @ lu.solve(b, trans="T") - b).max() <= 1e-12 * np.abs(b).max()


def _ybus_loop(net):
    """Y_bus by the plain per-line accumulation (a third formulation)."""
    Y = {}
    def add(i, j, v):
        Y[(i, j)] = Y.get((i, j), 0.0) + v
    for i in range(int(net["n_b"])):
        add(i, i, net["Y_sh"][i])
    for l in range(int(net["n_l"])):
        f, t = int(net["line_from"][l]), int(net["line_to"][l])
        add(f, f, net["Y_ff"][l]); add(f, t, net["Y_ft"][l])
        add(t, f, net["Y_tf"][l]); add(t, t, net["Y_tt"][l])
    return Y


@pytest.mark.parametrize("name", ["case118", "case1354"])
def test_ybus_sparse_branch(name):
    """The sparse-storage branch of ybus_entries (taken above 3000 buses, i.e.
    by every case9241 oracle call) forced on smaller grids: same pattern and
    values as the dense branch and as a per-line accumulation."""
    net, _ = table1_grid(name)
    i0, j0, y0 = O.ybus_entries(net)                 # dense product
    i1, j1, y1 = O.ybus_entries(net, dense_max=0)    # sparse product
    assert np.array_equal(i0, i1) and np.array_equal(j0, j1)
    assert np.abs(y0 - y1).max() <= 1e-13 * np.abs(y0).max()
    Y = _ybus_loop(net)
    assert len(Y) == len(i1)
    ref = np.array([Y[(int(a), int(b))] for a, b in zip(i1, j1)])
    assert np.abs(ref - y1).max() <= 1e-13 * np.abs(ref).max()


def test_static_lu_pins():
    """R18 numeric rule: no pivoting, first failing pivot k → k+1.
    Hand cases: regular; exact cancellation (u_22 = 0); a zero leading pivot
    that partial pivoting would swap away; the 1e-12 row-relative threshold on
    both sides; a NaN; LU reproduces PAPᵀ; and on case118's G_x with the R18
    ordering the factors solve like LAPACK."""
    I2 = np.arange(2)
    assert O.static_lu(np.array([[1.0, 2.0], [3.0, 4.0]]), I2)[0] == 0
    assert O.static_lu(np.array([[1.0, 2.0], [2.0, 4.0]]), I2)[0] == 2
    assert O.static_lu(np.array([[0.0, 1.0], [1.0, 0.0]]), I2)[0] == 1
    assert O.static_lu(np.array([[0.5e-12, 1.0], [1.0, 1.0]]), I2)[0] == 1
    assert O.static_lu(np.array([[2e-12, 1.0], [1.0, 1.0]]), I2)[0] == 0
    assert O.static_lu(np.array([[1.0, 0.0], [0.0, np.nan]]), I2)[0] == 2
    assert O.static_lu(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([1, 0]))[0] == 0
    rng = np.random.default_rng(3)
    M = rng.standard_normal((6, 6)) + 6 * np.eye(6)
    p = rng.permutation(6)
    info, LU = O.static_lu(M, p)
    assert info == 0
    L, U = np.tril(LU, -1) + np.eye(6), np.triu(LU)
    assert np.abs(L @ U - M[np.ix_(p, p)]).max() <= 1e-14 * np.abs(M).max()
    net, pt = table1_grid("case118")
    part = O.partition(net)
    Gx, _, _ = O.jacobians(net, part, pt)
    perm, _ = O.permutation(part, O.md_ordering(net, part))
    info, LU = O.static_lu(Gx, perm)
    assert info == 0
    n = len(perm)
    L, U = np.tril(LU, -1) + np.eye(n), np.triu(LU)
    b = rng.standard_normal(n)
    z = np.zeros(n)
    z[perm] = np.linalg.solve(U, np.linalg.solve(L, b[perm]))
    assert np.abs(Gx @ z - b).max() <= 1e-12 * np.abs(b).max()
    assert np.allclose(z, np.linalg.solve(Gx.toarray(), b), rtol=0, atol=1e-9 * np.abs(z).max())


# --------------------------------------------------------------------- P15 structure pins
def _line_net(n_b, edges, gen_bus, ref_bus):
    Yff, Yft, Ytf, Ytt = pi_model(np.zeros(len(edges)), np.full(len(edges), 0.1), np.zeros(len(edges)),
                                  np.ones(len(edges)), np.zeros(len(edges)))
    e = np.array(edges, dtype=np.int32)
    return dict(n_b=n_b, n_l=len(edges), n_g=len(gen_bus), line_from=e[:, 0], line_to=e[:, 1],
                Y_ff=Yff, Y_ft=Yft, Y_tf=Ytf, Y_tt=Ytt, Y_sh=np.zeros(n_b, complex),
                gen_bus=np.array(gen_bus, np.int32), ref_bus=ref_bus, p_d=np.zeros(n_b), q_d=np.zeros(n_b),
                F_max=np.ones(len(edges)), c_quad=np.ones(len(gen_bus)), c_lin=np.ones(len(gen_bus)))


def test_md_ordering_hand_cases():
    """R18's written rule worked by hand: minimum current degree on the bus
    graph without the reference bus, ties to the lowest bus index, eliminated
    buses join their neighbours into a clique.
    Path 0-1-2-3-4 (ref 4): degrees 1,2,2,1 → 0 (tie with 3), then 1, 2, 3.
    Star centre 2, leaves 0,1,3,4 (ref 0): 1, 3, then 2 (tie with 4), 4.
    Ring 0..4 + ref 5 on bus 0: all degree 2 → 0; its neighbours 1, 4 join;
    all degree 2 again → 1, then 2, 3, 4."""
    cases = [(_line_net(5, [(0, 1), (1, 2), (2, 3), (3, 4)], [4], 4), [0, 1, 2, 3]),
             (_line_net(5, [(2, 0), (2, 1), (2, 3), (2, 4)], [0], 0), [1, 3, 2, 4]),
             (_line_net(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (5, 0)], [5], 5), [0, 1, 2, 3, 4])]
    for net, want in cases:
        part = O.partition(net)
        assert O.md_ordering(net, part).tolist() == want


@pytest.mark.parametrize("name", ["case9", "rich8", "case118"])
def test_patterns_match_numeric_jacobians(name):
    """The structural (topological, R19) CSR patterns of G_x, G_u and A contain
    exactly the nonzeros of the numeric Jacobians at a generic point (no
    structural zero is dropped, no spurious entry): patterns by graph walks vs
    values by closed-form derivatives."""
    if name == "case9":
        net, pt = case9()
    elif name == "rich8":
        net, pt = rich_small()
    else:
        net, pt = table1_grid(name)
    part = O.partition(net)
    rng = np.random.default_rng(9)   # a generic point (case9's is flat: r = 0 transformers give exact zeros)
    pt = dict(pt, v=pt["v"] + 0.05 * rng.uniform(size=net["n_b"]),
              theta=pt["theta"] + 0.1 * rng.uniform(size=net["n_b"]))
    pt["theta"][net["ref_bus"]] = 0.0
    Gx, Gu, A = O.jacobians(net, part, pt)
    (px, ix), (pu, iu) = O.gx_gu_patterns(net, part)
    pa, ia = O.a_pattern(net, part)
    for M, ptr, idx in ((Gx, px, ix), (Gu, pu, iu), (A, pa, ia)):
        D = np.asarray(sp.csr_matrix(M).toarray())
        P = np.zeros(D.shape, dtype=bool)
        P[np.repeat(np.arange(D.shape[0]), np.diff(ptr)), idx] = True
        assert np.array_equal(P, D != 0)


# --------------------------------------------------------------------- P13 Cholesky
def test_cholesky_pins():
    """P13: LLᵀ = K to c·n·ε, matches LAPACK; I → I; diag(1,−1) → info = 2."""
    rng = np.random.default_rng(2)
    B = rng.standard_normal((40, 40))
    K = B @ B.T + 40 * np.eye(40)
    L, info = O.cholesky(K)
    assert info == 0
    assert np.max(np.abs(L @ L.T - K)) <= 40 * 2.2e-16 * np.abs(K).max() * 10
    assert np.allclose(L, np.linalg.cholesky(K), atol=1e-12)
    b = rng.standard_normal(40)
    assert np.allclose(O.chol_solve(L, b), np.linalg.solve(K, b), atol=1e-12)
    assert np.allclose(O.cholesky(np.eye(5))[0], np.eye(5)) and O.cholesky(np.eye(5))[1] == 0
    assert O.cholesky(np.diag([1.0, -1.0]))[1] == 2
    assert O.cholesky(np.diag([1.0, np.nan]))[1] == 2


# --------------------------------------------------------------------- P15 structure
def _tree_net(n):
    rng = np.random.default_rng(n)
    parent = [int(rng.integers(0, i)) for i in range(1, n)]
    lf = np.array(parent, np.int32)
    lt = np.arange(1, n, dtype=np.int32)
    Y = -1j * np.ones(n - 1) * 10
    return dict(n_b=n, n_l=n - 1, n_g=2, line_from=lf, line_to=lt, Y_ff=-Y, Y_ft=Y, Y_tf=Y, Y_tt=-Y,
                Y_sh=np.zeros(n, complex), gen_bus=np.array([0, n - 1], np.int32), ref_bus=0,
                p_d=np.zeros(n), q_d=np.zeros(n), F_max=np.ones(n - 1), c_quad=np.ones(2), c_lin=np.ones(2))


def test_min_degree_on_tree_has_no_fill():
    """Minimum degree on a tree is a perfect elimination order (leaves first):
    the symbolic LU has no fill beyond G_x's own pattern."""
    net = _tree_net(30)
    part = O.partition(net)
    (px, ix), _ = O.gx_gu_patterns(net, part)
    order = O.md_ordering(net, part)
    perm, blk = O.permutation(part, order)
    F = O.symbolic_lu(px, ix, perm)
    assert F.sum() == len(ix)


@pytest.mark.parametrize("name", ["case9", "rich8", "case118"])
def test_symbolic_fill_matches_numeric_lu(name):
    """The Boolean fill equals the nonzero pattern of a numeric no-pivot LU of a
    random matrix with G_x's pattern (no accidental cancellation a.s.)."""
    if name == "case9":
        net, _ = case9()
    elif name == "rich8":
        net, _ = rich_small()
    else:
        net, _ = table1_grid("case118")
    part = O.partition(net)
    (px, ix), _ = O.gx_gu_patterns(net, part)
    perm, blk = O.permutation(part, O.md_ordering(net, part))
    F = O.symbolic_lu(px, ix, perm)
    n = part["n_x"]
    rng = np.random.default_rng(4)
    A = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(px))
    A[rows, ix] = rng.uniform(0.5, 1.5, size=len(ix))
    A[np.arange(n), np.arange(n)] += n
    inv = np.argsort(perm)
    Ap = A[np.ix_(perm, perm)]
    for k in range(n):       # Doolittle, no pivoting
        Ap[k + 1:, k] /= Ap[k, k]
        Ap[k + 1:, k + 1:] -= np.outer(Ap[k + 1:, k], Ap[k, k + 1:])
    assert np.array_equal(np.abs(Ap) > 1e-300, F)
    # levels: every dependency sits at a strictly lower level (P15)
    levL, levU = O.block_levels(F, blk)
    owner = np.repeat(np.arange(len(blk) - 1), np.diff(blk))
    r, c = np.nonzero(F)
    lo = owner[c] < owner[r]
    assert np.all(levL[owner[r][lo]] > levL[owner[c][lo]])
    up = owner[c] > owner[r]
    assert np.all(levU[owner[r][up]] > levU[owner[c][up]])
    # level count = longest path by an independent memoised DFS
    deps = {b: set() for b in range(len(blk) - 1)}
    for a, b in zip(owner[r][lo], owner[c][lo]):
        deps[a].add(b)
    memo = {}

    def depth(b):
        if b not in memo:
            memo[b] = 0 if not deps[b] else 1 + max(depth(d) for d in deps[b])
        return memo[b]

    assert max(depth(b) for b in deps) == levL.max()
