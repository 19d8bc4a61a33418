"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (NumPy/SciPy, IEEE fp64)
of what the batched reduced-Hessian hot path computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with the CUDA
path (``paper_2203_11875_b200``) and imports nothing from it; both sides take
their inputs from the seeded generators in ``synth/``.

Formulation (deliberately different from the GPU's ψ-basis chain):
every quantity is a sum of *polar terms*  T(a,b,c) = conj(c)·v_a v_b e^{j(θ_a-θ_b)}
 * bus injections  s_i = Σ_j T(i,j,Y_bus[i,j])
 * line flows      s_f = T(f,f,Y_ff)+T(f,t,Y_ft),
                   s_t = T(t,t,Y_tt)+T(t,f,Y_tf)             (PAPER.md L79–88 with R1)
and each term's value, gradient and Hessian is written in closed form.  The
bus terms are grouped by Y_bus entries (parallel lines and shunts merged),
the GPU groups by line.  The reduction follows the naive-sensitivity route
S = -G_x^{-1} G_u that the paper rejects, so it shares
no arithmetic order with the GPU's batched adjoint-adjoint route.

Readings of the paper: R1 conj in s_f/s_t, R8 implicit
p_ref in the objective, R9 Σ_u in K_cond, R11 G_uᵀΨ, R14 K carries Σ_x,
R18 static symmetric bus-level minimum-degree ordering, R21 one generator per
generator bus.  Parity status: every function below is pinned by a
``-m "not gpu"`` test (tests/test_oracle_*.py); none is "parity unpinned".
"""
from __future__ import annotations

import heapq
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


# ----------------------------------------------------------------------------
# Partition (PAPER.md L204–272 reduced-space OPF; L450–545 formalism)
# ----------------------------------------------------------------------------
class TopologyError(ValueError):
    """No/invalid reference bus, ≠1 generator on a generator bus (R21), bad index."""


def partition(net):
    """State/control/constraint index maps of SURVEY §8.0.

    x = [θ_i : i ≠ r0 ascending ; v_i : i ∈ PQ ascending]   (p_ref, q implicit)
    u = [v_i : i ∈ B_g ascending ; p_g : g ≠ g_r ascending]
    g rows = x rows: row of θ_i is P_i, row of v_i is Q_i
    r rows = [P_r0 ; Q_r0 ; Q_i : i ∈ PV ascending]         (eq. implicitcons)
    h rows = [H^f_ℓ : F_ℓ > 0 ; H^t_ℓ : F_ℓ > 0]           (eq. linelimitsvec)
    """
    n_b, n_g = int(net["n_b"]), int(net["n_g"])
    gen_bus = np.asarray(net["gen_bus"], dtype=np.int64)
    r0 = int(net["ref_bus"])
    if not (0 <= r0 < n_b):
        raise TopologyError("reference bus out of range")
    if np.any(gen_bus < 0) or np.any(gen_bus >= n_b):
        raise TopologyError("generator bus out of range")
    cnt = np.bincount(gen_bus, minlength=n_b)
    if cnt[r0] != 1:
        raise TopologyError("reference bus must host exactly one generator")
    if np.any(cnt > 1):
        raise TopologyError("more than one generator on a bus (R21)")
    is_gen = cnt > 0
    g_r = int(np.nonzero(gen_bus == r0)[0][0])
    x_th = -np.ones(n_b, dtype=np.int64)
    x_v = -np.ones(n_b, dtype=np.int64)
    u_v = -np.ones(n_b, dtype=np.int64)
    u_p = -np.ones(n_g, dtype=np.int64)
    k = 0
    for i in range(n_b):
        if i != r0:
            x_th[i] = k
            k += 1
    for i in range(n_b):
        if not is_gen[i]:
            x_v[i] = k
            k += 1
    n_x = k
    k = 0
    for i in range(n_b):
        if is_gen[i]:
            u_v[i] = k
            k += 1
    for g in range(n_g):
        if g != g_r:
            u_p[g] = k
            k += 1
    n_u = k
    r_rows = [(r0, 0), (r0, 1)] + [(i, 1) for i in range(n_b) if is_gen[i] and i != r0]
    F = np.asarray(net["F_max"])
    lim = [l for l in range(int(net["n_l"])) if F[l] > 0]
    h_rows = [(l, 0) for l in lim] + [(l, 1) for l in lim]
    return dict(n_b=n_b, n_g=n_g, r0=r0, g_r=g_r, is_gen=is_gen, x_th=x_th, x_v=x_v,
                u_v=u_v, u_p=u_p, n_x=n_x, n_u=n_u, r_rows=r_rows, h_rows=h_rows,
                n_r=len(r_rows), n_h=len(h_rows), m=len(r_rows) + len(h_rows))


def z_index(part):
    """Index of each bus variable in z = [u; x] (PAPER.md L527–544 ordering [u, x]); -1 = fixed θ_ref."""
    n_u = part["n_u"]
    zv = np.where(part["u_v"] >= 0, part["u_v"], n_u + part["x_v"])
    zth = np.where(part["x_th"] >= 0, n_u + part["x_th"], -1)
    return zv, zth


# ----------------------------------------------------------------------------
# O1 admittance matrix
# ----------------------------------------------------------------------------
def ybus(net):
    """Dense complex Y_bus = C_fᵀY_f + C_tᵀY_t + diag(Y_sh), with
    Y_f = diag(Y_ff)C_f + diag(Y_ft)C_t and Y_t = diag(Y_tf)C_f + diag(Y_tt)C_t."""
    n_b, n_l = int(net["n_b"]), int(net["n_l"])
    Cf = np.zeros((n_l, n_b))
    Ct = np.zeros((n_l, n_b))
    Cf[np.arange(n_l), net["line_from"]] = 1.0
    Ct[np.arange(n_l), net["line_to"]] = 1.0
    Yf = np.diag(net["Y_ff"]) @ Cf + np.diag(net["Y_ft"]) @ Ct
    Yt = np.diag(net["Y_tf"]) @ Cf + np.diag(net["Y_tt"]) @ Ct
    return Cf.T @ Yf + Ct.T @ Yt + np.diag(net["Y_sh"])


def ybus_entries(net, dense_max=3000):
    """Nonzero entries (i, j, Y_ij) of Y_bus in row-major order, topological
    pattern (an entry exists iff i = j or a line joins i and j; R19), values
    summed over parallel lines exactly as the dense product above.  Above
    dense_max buses the same product runs in sparse storage (pinned against
    the dense branch by tests/test_oracle_pins.py)."""
    n_b = int(net["n_b"])
    f = np.asarray(net["line_from"], dtype=np.int64)
    t = np.asarray(net["line_to"], dtype=np.int64)
    key = np.unique(np.concatenate([np.arange(n_b) * n_b + np.arange(n_b), f * n_b + t, t * n_b + f]))
    ii, jj = key // n_b, key % n_b
    if n_b <= dense_max:
        Y = ybus(net)
        return ii, jj, Y[ii, jj]
    # same formula with sparse storage (the dense product does not fit in memory at 9k buses)
    n_l = int(net["n_l"])
    rows = np.arange(n_l)
    Cf = sp.csr_matrix((np.ones(n_l), (rows, f)), shape=(n_l, n_b))
    Ct = sp.csr_matrix((np.ones(n_l), (rows, t)), shape=(n_l, n_b))
    Yf = sp.diags(net["Y_ff"]) @ Cf + sp.diags(net["Y_ft"]) @ Ct
    Yt = sp.diags(net["Y_tf"]) @ Cf + sp.diags(net["Y_tt"]) @ Ct
    Y = (Cf.T @ Yf + Ct.T @ Yt + sp.diags(net["Y_sh"])).tocsr()
    return ii, jj, np.asarray(Y[ii, jj]).ravel()


# ----------------------------------------------------------------------------
# O2/O3 function values (eq. powerflow, eq. powerflowvec,
# eq. power_inj_line L83–88 with R1, eq. linelimitsvec)
# ----------------------------------------------------------------------------
def injections(net, v, theta):
    """p_i^inj, q_i^inj by the explicit sum over j of eq. powerflow (L59–60),
    for every pair with a Y_bus entry."""
    n_b = int(net["n_b"])
    ii, jj, Y = ybus_entries(net)
    p = np.zeros(n_b)
    q = np.zeros(n_b)
    for k in range(len(ii)):
        i, j = ii[k], jj[k]
        g, b = Y[k].real, Y[k].imag
        t = theta[i] - theta[j]
        p[i] += v[i] * v[j] * (g * np.cos(t) + b * np.sin(t))
        q[i] += v[i] * v[j] * (g * np.sin(t) - b * np.cos(t))
    return p, q


def balance(net, point):
    """G(v,θ,p_g,q_g) = [p^inj − C_g p_g + p_d ; q^inj − C_g q_g + q_d] (eq. powerflowvec)."""
    p, q = injections(net, point["v"], point["theta"])
    n_b = int(net["n_b"])
    cgp = np.zeros(n_b)
    cgq = np.zeros(n_b)
    np.add.at(cgp, net["gen_bus"], point["p_g"])
    np.add.at(cgq, net["gen_bus"], point["q_g"])
    return np.concatenate([p - cgp + point["p_d"], q - cgq + point["q_d"]])


def line_flows(net, v, theta):
    """Complex s_f = (C_f V)⊙conj(Y_f V), s_t = (C_t V)⊙conj(Y_t V) (R1: the
    conjugate the print drops, consistent with Kirchhoff L45)."""
    V = v * np.exp(1j * theta)
    f, t = net["line_from"], net["line_to"]
    sf = V[f] * np.conj(net["Y_ff"] * V[f] + net["Y_ft"] * V[t])
    st = V[t] * np.conj(net["Y_tf"] * V[f] + net["Y_tt"] * V[t])
    return sf, st


def constraints(net, point):
    """(G [2n_b], H [2n_ℓ] = [|s_f|²; |s_t|²], s_flow [4][n_ℓ] = s_p^f, s_q^f, s_p^t, s_q^t)."""
    G = balance(net, point)
    sf, st = line_flows(net, point["v"], point["theta"])
    H = np.concatenate([(sf * np.conj(sf)).real, (st * np.conj(st)).real])
    s = np.stack([sf.real, sf.imag, st.real, st.imag])
    return G, H, s


# ----------------------------------------------------------------------------
# Polar terms: closed-form value / gradient / Hessian
# ----------------------------------------------------------------------------
def _terms_local(a, b, c, v, theta):
    """For terms T = conj(c) v_a v_b e^{jφ}, φ = θ_a − θ_b (vectorised over terms).
    Returns Re T, Im T, their gradients (K,4) and Hessians (K,4,4) w.r.t. the
    local variables (v_a, v_b, θ_a, θ_b).  With Rc = c_r cos φ + c_i sin φ and
    Ic = c_r sin φ − c_i cos φ:  Re T = v_a v_b Rc, Im T = v_a v_b Ic."""
    cr, ci = c.real, c.imag
    va, vb = v[a], v[b]
    phi = theta[a] - theta[b]
    cs, sn = np.cos(phi), np.sin(phi)
    Rc = cr * cs + ci * sn
    Ic = cr * sn - ci * cs
    R = va * vb * Rc
    I = va * vb * Ic
    K = len(a)
    gR = np.stack([vb * Rc, va * Rc, -va * vb * Ic, va * vb * Ic], axis=1)
    gI = np.stack([vb * Ic, va * Ic, va * vb * Rc, -va * vb * Rc], axis=1)
    HR = np.zeros((K, 4, 4))
    HI = np.zeros((K, 4, 4))
    # ∂²/∂v_a∂v_b
    HR[:, 0, 1] = HR[:, 1, 0] = Rc
    HI[:, 0, 1] = HI[:, 1, 0] = Ic
    # ∂²/∂v_a∂θ_a, ∂v_a∂θ_b, ∂v_b∂θ_a, ∂v_b∂θ_b
    HR[:, 0, 2] = HR[:, 2, 0] = -vb * Ic
    HR[:, 0, 3] = HR[:, 3, 0] = vb * Ic
    HR[:, 1, 2] = HR[:, 2, 1] = -va * Ic
    HR[:, 1, 3] = HR[:, 3, 1] = va * Ic
    HI[:, 0, 2] = HI[:, 2, 0] = vb * Rc
    HI[:, 0, 3] = HI[:, 3, 0] = -vb * Rc
    HI[:, 1, 2] = HI[:, 2, 1] = va * Rc
    HI[:, 1, 3] = HI[:, 3, 1] = -va * Rc
    # ∂²/∂θ²
    HR[:, 2, 2] = HR[:, 3, 3] = -R
    HR[:, 2, 3] = HR[:, 3, 2] = R
    HI[:, 2, 2] = HI[:, 3, 3] = -I
    HI[:, 2, 3] = HI[:, 3, 2] = I
    return R, I, gR, gI, HR, HI


def _local_z(a, b, zv, zth):
    return np.stack([zv[a], zv[b], zth[a], zth[b]], axis=1)


def _bus_terms(net):
    ii, jj, Y = ybus_entries(net)
    return ii, jj, Y


def _line_terms(net):
    """Terms of the line flows: end e=0 (from): T(f,f,Y_ff)+T(f,t,Y_ft);
    end e=1 (to): T(t,t,Y_tt)+T(t,f,Y_tf).  Returns (a, b, c, line, end)."""
    n_l = int(net["n_l"])
    f, t = np.asarray(net["line_from"]), np.asarray(net["line_to"])
    L = np.arange(n_l)
    a = np.concatenate([f, f, t, t])
    b = np.concatenate([f, t, t, f])
    c = np.concatenate([net["Y_ff"], net["Y_ft"], net["Y_tt"], net["Y_tf"]])
    line = np.concatenate([L, L, L, L])
    end = np.concatenate([np.zeros(2 * n_l, int), np.ones(2 * n_l, int)])
    return a, b, c, line, end


def _coo_rows(rows, cols, vals, shape):
    keep = cols >= 0
    return sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=shape)


# ----------------------------------------------------------------------------
# O4 first derivatives (G = [G_u G_x], A = [A_u A_x])
# ----------------------------------------------------------------------------
def bus_jacobian(net, part, v, theta):
    """∂[p^inj; q^inj]/∂z, z = [u; x], sparse (2n_b × (n_u+n_x))."""
    n_b, n_z = part["n_b"], part["n_u"] + part["n_x"]
    zv, zth = z_index(part)
    a, b, c = _bus_terms(net)
    _, _, gR, gI, _, _ = _terms_local(a, b, c, v, theta)
    zl = _local_z(a, b, zv, zth)
    rows = np.repeat(a, 4)
    JP = _coo_rows(rows, zl.ravel(), gR.ravel(), (n_b, n_z))
    JQ = _coo_rows(rows, zl.ravel(), gI.ravel(), (n_b, n_z))
    return sp.vstack([JP, JQ]).tocsr()


def line_jacobian(net, part, v, theta):
    """∂[s_p^f; s_q^f; s_p^t; s_q^t]/∂z, sparse (4n_ℓ × n_z), row blocks as in s_flow."""
    n_l, n_z = int(net["n_l"]), part["n_u"] + part["n_x"]
    zv, zth = z_index(part)
    a, b, c, line, end = _line_terms(net)
    _, _, gR, gI, _, _ = _terms_local(a, b, c, v, theta)
    zl = _local_z(a, b, zv, zth)
    rowP = np.repeat(line + 2 * n_l * end, 4)
    rowQ = np.repeat(line + n_l + 2 * n_l * end, 4)
    J = _coo_rows(np.concatenate([rowP, rowQ]), np.concatenate([zl.ravel(), zl.ravel()]),
                  np.concatenate([gR.ravel(), gI.ravel()]), (4 * n_l, n_z))
    return J


def jacobians(net, part, point):
    """G_x (n_x×n_x), G_u (n_x×n_u), A (m × (n_u+n_x)) at the point.

    g rows: P_i − C_g p_g + p_d (i≠r0), Q_i − C_g q_g + q_d (i∈PQ) — the p_g
    of a non-reference generator enters its bus's P row with −1 (eq. powerflowvec).
    A rows: r = injections (R7) and h = |s|², ∇h = 2(s_p∇s_p + s_q∇s_q)."""
    v, th = point["v"], point["theta"]
    n_u, n_x, n_b = part["n_u"], part["n_x"], part["n_b"]
    JB = bus_jacobian(net, part, v, th)
    # rows of g in x order
    grow = np.empty(n_x, dtype=np.int64)
    for i in range(n_b):
        if part["x_th"][i] >= 0:
            grow[part["x_th"][i]] = i
        if part["x_v"][i] >= 0:
            grow[part["x_v"][i]] = n_b + i
    Gz = JB[grow, :].tolil()
    gb = np.asarray(net["gen_bus"])
    for g in range(part["n_g"]):
        if part["u_p"][g] >= 0:
            Gz[part["x_th"][gb[g]], part["u_p"][g]] += -1.0
    Gz = Gz.tocsr()
    Gu = Gz[:, :n_u]
    Gx = Gz[:, n_u:]
    # A rows
    rrows = np.array([i + n_b * t for (i, t) in part["r_rows"]], dtype=np.int64)
    Ar = JB[rrows, :]
    n_l = int(net["n_l"])
    JL = line_jacobian(net, part, v, th)
    sf, st = line_flows(net, v, th)
    # one row per h row (l, e): 2 (s_p ∇s_p + s_q ∇s_q) of that line end
    hl = np.array([l for (l, e) in part["h_rows"]], dtype=np.int64)
    he = np.array([e for (l, e) in part["h_rows"]], dtype=np.int64)
    if len(hl):
        s_h = np.where(he == 0, sf[hl], st[hl])
        rp = hl + 2 * n_l * he
        rq = hl + n_l + 2 * n_l * he
        Ah = 2.0 * (sp.diags(s_h.real) @ JL[rp, :] + sp.diags(s_h.imag) @ JL[rq, :])
    else:
        Ah = sp.csr_matrix((0, n_u + n_x))
    A = sp.vstack([Ar, Ah]).tocsr()
    return Gx.tocsr(), Gu.tocsr(), A


def objective_gradient(net, part, point):
    """∇_z f with f = Σ_{g≠g_r}(c1 p_g² + c2 p_g) + c1_r p_ref² + c2_r p_ref,
    p_ref = P^inj_r0(v,θ) + p^d_r0 (implicit p_ref L220–223; R8)."""
    n_u, n_x = part["n_u"], part["n_x"]
    gr = part["g_r"]
    p, _ = injections(net, point["v"], point["theta"])
    pref = p[part["r0"]] + point["p_d"][part["r0"]]
    JB = bus_jacobian(net, part, point["v"], point["theta"])
    grad = (2 * net["c_quad"][gr] * pref + net["c_lin"][gr]) * JB[part["r0"], :].toarray().ravel()
    for g in range(part["n_g"]):
        if part["u_p"][g] >= 0:
            grad[part["u_p"][g]] += 2 * net["c_quad"][g] * point["p_g"][g] + net["c_lin"][g]
    return grad


def objective(net, part, point):
    p, _ = injections(net, point["v"], point["theta"])
    pref = p[part["r0"]] + point["p_d"][part["r0"]]
    f = 0.0
    for g in range(part["n_g"]):
        pg = pref if g == part["g_r"] else point["p_g"][g]
        f += net["c_quad"][g] * pg * pg + net["c_lin"][g] * pg
    return f


# ----------------------------------------------------------------------------
# O5 second derivatives: W = ∇²_z L, L = f + λᵀg + yᵀ[r; h]
# ----------------------------------------------------------------------------
def bus_multipliers(net, part, point, lam, y):
    """μ^P_i, μ^Q_i: weight of ∇²p_i^inj, ∇²q_i^inj in W.  λ on g rows, y_r on
    r rows, plus (2c1 p_ref + c2)_{g_r} on P_r0 from the implicit p_ref (R8)."""
    n_b = part["n_b"]
    muP = np.zeros(n_b)
    muQ = np.zeros(n_b)
    for i in range(n_b):
        if part["x_th"][i] >= 0:
            muP[i] += lam[part["x_th"][i]]
        if part["x_v"][i] >= 0:
            muQ[i] += lam[part["x_v"][i]]
    for k, (i, t) in enumerate(part["r_rows"]):
        if t == 0:
            muP[i] += y[k]
        else:
            muQ[i] += y[k]
    p, _ = injections(net, point["v"], point["theta"])
    r0, gr = part["r0"], part["g_r"]
    pref = p[r0] + point["p_d"][r0]
    muP[r0] += 2 * net["c_quad"][gr] * pref + net["c_lin"][gr]
    return muP, muQ


def lagrangian_hessian(net, part, point, lam, y):
    """W (n_z × n_z, sparse) = Σ_i μ^P_i∇²p_i + μ^Q_i∇²q_i
       + 2c1_{g_r}∇p_r0∇p_r0ᵀ                                 (R8)
       + Σ_h y_h·2(∇s_p∇s_pᵀ + ∇s_q∇s_qᵀ + s_p∇²s_p + s_q∇²s_q)
       + diag(2c1_g) on p_g, g ≠ g_r."""
    v, th = point["v"], point["theta"]
    n_u, n_x = part["n_u"], part["n_x"]
    n_z = n_u + n_x
    zv, zth = z_index(part)
    muP, muQ = bus_multipliers(net, part, point, lam, y)
    rows, cols, vals = [], [], []

    def add_local(zl, H):
        r = np.repeat(zl, 4, axis=1).ravel()
        c = np.tile(zl, (1, 4)).ravel()
        keep = (r >= 0) & (c >= 0)
        rows.append(r[keep])
        cols.append(c[keep])
        vals.append(H.reshape(len(zl), 16).ravel()[keep])

    a, b, c = _bus_terms(net)
    _, _, _, _, HR, HI = _terms_local(a, b, c, v, th)
    add_local(_local_z(a, b, zv, zth), muP[a][:, None, None] * HR + muQ[a][:, None, None] * HI)

    n_l = int(net["n_l"])
    la, lb, lc, line, end = _line_terms(net)
    _, _, _, _, LHR, LHI = _terms_local(la, lb, lc, v, th)
    sf, st = line_flows(net, v, th)
    yh_end = np.zeros((2, n_l))
    for k, (l, e) in enumerate(part["h_rows"]):
        yh_end[e, l] += y[part["n_r"] + k]
    s_end = np.stack([sf, st])
    w = yh_end[end, line]
    sp_, sq_ = s_end[end, line].real, s_end[end, line].imag
    add_local(_local_z(la, lb, zv, zth), (2 * w * sp_)[:, None, None] * LHR + (2 * w * sq_)[:, None, None] * LHI)
    W = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n_z, n_z))
    # Gauss–Newton part of y_h·h:  2 y_h (∇s_p∇s_pᵀ + ∇s_q∇s_qᵀ)
    JL = line_jacobian(net, part, v, th)
    Dp = np.zeros(4 * n_l)
    for e in (0, 1):
        Dp[2 * n_l * e: 2 * n_l * e + n_l] = 2 * yh_end[e]
        Dp[2 * n_l * e + n_l: 2 * n_l * (e + 1)] = 2 * yh_end[e]
    W = W + JL.T @ sp.diags(Dp) @ JL
    # objective curvature through p_ref (rank one) and on explicit p_g
    JB = bus_jacobian(net, part, v, th)
    gP = JB[part["r0"], :]
    W = W + 2 * net["c_quad"][part["g_r"]] * (gP.T @ gP)
    d = np.zeros(n_z)
    for g in range(part["n_g"]):
        if part["u_p"][g] >= 0:
            d[part["u_p"][g]] += 2 * net["c_quad"][g]
    return (W + sp.diags(d)).tocsr()


def kkt_K(net, part, point, lam, y, sigma_s=None, sigma_x=None):
    """K = W + AᵀΣ_sA + blkdiag(0_u, Σ_x) ordered [u; x] (R14)."""
    n_u, n_x = part["n_u"], part["n_x"]
    W = lagrangian_hessian(net, part, point, lam, y)
    _, _, A = jacobians(net, part, point)
    K = W
    if sigma_s is not None:
        K = K + A.T @ sp.diags(sigma_s) @ A
    if sigma_x is not None:
        K = K + sp.diags(np.concatenate([np.zeros(n_u), sigma_x]))
    return K.tocsr()


def kkt_K_from(W, A, sigma_s, sigma_x, n_u):
    """K = W + AᵀΣ_sA + blkdiag(0_u, Σ_x) from given W and A (same as kkt_K)."""
    K = sp.csr_matrix(W)
    if sigma_s is not None:
        K = K + sp.csr_matrix(A).T @ sp.diags(sigma_s) @ sp.csr_matrix(A)
    if sigma_x is not None:
        K = K + sp.diags(np.concatenate([np.zeros(n_u), sigma_x]))
    return K.tocsr()


# ----------------------------------------------------------------------------
# O7 / O7' reductions (PAPER.md eq. algo:reduction L1156–1172; L1180–1235)
# ----------------------------------------------------------------------------
def _blocks(K, n_u):
    K = sp.csr_matrix(K)
    return K[:n_u, :n_u], K[:n_u, n_u:], K[n_u:, :n_u], K[n_u:, n_u:]


def sensitivity(Gx, Gu):
    """S = −G_x^{-1}G_u (dense n_x × n_u; the naive route of L1180)."""
    lu = spla.splu(sp.csc_matrix(Gx))
    return -lu.solve(np.asarray(sp.csr_matrix(Gu).toarray()))


def reduce_naive(K, Gx, Gu):
    """O7: K̂ = [I; S]ᵀ K [I; S] = K_uu + K_uxS + SᵀK_xu + SᵀK_xxS."""
    n_u = Gu.shape[1]
    Kuu, Kux, Kxu, Kxx = _blocks(K, n_u)
    S = sensitivity(Gx, Gu)
    KxxS = Kxx @ S
    return Kuu.toarray() + Kux @ S + (Kxu.T @ S).T + S.T @ KxxS


def reduce_adjoint(K, Gx, Gu, V):
    """O7': the paper's three steps for K̂V (L1203–1222), dense, with R11:
    Z = −G_x^{-1}(G_uV); [H_u; H_x] = K[V; Z]; Ψ = G_x^{-T}H_x; K̂V = H_u − G_uᵀΨ."""
    n_u = Gu.shape[1]
    Gxd = np.asarray(sp.csr_matrix(Gx).toarray())
    Z = -np.linalg.solve(Gxd, Gu @ V)
    H = K @ np.vstack([V, Z])
    Hu, Hx = H[:n_u], H[n_u:]
    Psi = np.linalg.solve(Gxd.T, Hx)
    return Hu - Gu.T @ Psi


# ----------------------------------------------------------------------------
# O8 dense Cholesky (PAPER.md L784–787 with R9, L1339–1342; Theorem 3)
# ----------------------------------------------------------------------------
def cholesky(Kc):
    """Textbook column Cholesky without pivoting.  Returns (L, info):
    info = 0, or j+1 for the first column whose pivot is ≤ 0 or non-finite."""
    A = np.array(Kc, dtype=np.float64, copy=True)
    n = A.shape[0]
    L = np.zeros_like(A)
    for j in range(n):
        d = A[j, j] - L[j, :j] @ L[j, :j]
        if not (d > 0.0) or not np.isfinite(d):
            return L, j + 1
        L[j, j] = np.sqrt(d)
        L[j + 1:, j] = (A[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L, 0


def regularized_cholesky(Kc0, delta_init, delta_first, growth, delta_max):
    """NEXT-3, the paper's inertia correction: factorize
    K_cond + δ_w I with δ_w = delta_init; while the Cholesky fails, δ_w ←
    delta_first (from 0) or growth·δ_w, up to delta_max.  Success certifies
    the inertia of K_aug (Theorem 3).
    Returns (δ_w of the last trial, trials, info, L)."""
    n = Kc0.shape[0]
    delta, trials = delta_init, 1
    L, info = cholesky(Kc0 + delta * np.eye(n))
    while info:
        nd = delta_first if delta == 0.0 else delta * growth
        if nd > delta_max:
            break
        delta, trials = nd, trials + 1
        L, info = cholesky(Kc0 + delta * np.eye(n))
    return delta, trials, info, L


def chol_solve(L, b):
    """Solve L Lᵀ p = b by forward then backward substitution."""
    n = L.shape[0]
    b = np.array(b, dtype=np.float64, copy=True)
    y = np.zeros_like(b)
    for i in range(n):
        y[i] = (b[i] - L[i, :i] @ y[:i]) / L[i, i]
    p = np.zeros_like(b)
    for i in range(n - 1, -1, -1):
        p[i] = (y[i] - L[i + 1:, i] @ p[i + 1:]) / L[i, i]
    return p


def condensed(Khat, sigma_u, delta_w):
    """K_cond = K̂ + diag(Σ_u) + δ_w I (Theorem 2 with R9; regularisation L1341)."""
    n = Khat.shape[0]
    Kc = np.array(Khat, copy=True)
    if sigma_u is not None:
        Kc[np.diag_indices(n)] += sigma_u
    Kc[np.diag_indices(n)] += delta_w
    return Kc


# ----------------------------------------------------------------------------
# O6 Newton power flow (Algorithm 2 projection L1063; tolerance L1427–1429)
# ----------------------------------------------------------------------------
def g_residual(net, part, point):
    """g(x,u): the G rows selected by the x partition."""
    Gfull = balance(net, point)
    n_b = part["n_b"]
    out = np.empty(part["n_x"])
    for i in range(n_b):
        if part["x_th"][i] >= 0:
            out[part["x_th"][i]] = Gfull[i]
        if part["x_v"][i] >= 0:
            out[part["x_v"][i]] = Gfull[n_b + i]
    return out


def get_x(part, point):
    x = np.empty(part["n_x"])
    for i in range(part["n_b"]):
        if part["x_th"][i] >= 0:
            x[part["x_th"][i]] = point["theta"][i]
        if part["x_v"][i] >= 0:
            x[part["x_v"][i]] = point["v"][i]
    return x


def set_x(part, point, x):
    pt = dict(point)
    v, th = point["v"].copy(), point["theta"].copy()
    for i in range(part["n_b"]):
        if part["x_th"][i] >= 0:
            th[i] = x[part["x_th"][i]]
        if part["x_v"][i] >= 0:
            v[i] = x[part["x_v"][i]]
    pt["v"], pt["theta"] = v, th
    return pt


def get_u(part, point):
    u = np.empty(part["n_u"])
    for i in range(part["n_b"]):
        if part["u_v"][i] >= 0:
            u[part["u_v"][i]] = point["v"][i]
    for g in range(part["n_g"]):
        if part["u_p"][g] >= 0:
            u[part["u_p"][g]] = point["p_g"][g]
    return u


def set_u(part, point, u):
    pt = dict(point)
    v, pg = point["v"].copy(), point["p_g"].copy()
    for i in range(part["n_b"]):
        if part["u_v"][i] >= 0:
            v[i] = u[part["u_v"][i]]
    for g in range(part["n_g"]):
        if part["u_p"][g] >= 0:
            pg[g] = u[part["u_p"][g]]
    pt["v"], pt["p_g"] = v, pg
    return pt


def newton(net, part, point, tol=1e-12, maxit=20):
    """x ← x − G_x^{-1} g(x,u) with dense LU (partial pivoting, LAPACK) until
    ‖g‖∞ ≤ tol.  Returns (point, iterations, residual history)."""
    pt = dict(point)
    hist = []
    for it in range(maxit + 1):
        gres = g_residual(net, part, pt)
        hist.append(np.max(np.abs(gres)))
        if hist[-1] <= tol:
            return pt, it, hist
        Gx, _, _ = jacobians(net, part, pt)
        dx = np.linalg.solve(Gx.toarray(), gres)
        pt = set_x(part, pt, get_x(part, pt) - dx)
    raise RuntimeError("Newton did not converge: %s" % hist[-3:])


def adjoint_multipliers(net, part, point, y):
    """λ solving G_xᵀλ = −∇_x(f + y_rᵀr + y_hᵀh) (Algorithm 2 adjoint step, L1064)."""
    Gx, _, A = jacobians(net, part, point)
    n_u = part["n_u"]
    grad = objective_gradient(net, part, point) + A.T @ y
    return spla.splu(sp.csc_matrix(Gx)).solve(-grad[n_u:], trans="T")


def reduced_gradient(net, part, point, y):
    """Algorithm 2's adjoint step and the reduced gradient (Theorem 'Reduced
    derivatives'): with ∇ℓ = ∇_z(f + y_rᵀr + y_hᵀh),
    λ = −G_x⁻ᵀ∇_xℓ and ∇_uℓ_r = ∇_uℓ − G_uᵀG_x⁻ᵀ∇_xℓ = ∇_uℓ + G_uᵀλ.
    Returns (λ, ∇_uℓ_r)."""
    Gx, Gu, A = jacobians(net, part, point)
    n_u = part["n_u"]
    grad = objective_gradient(net, part, point) + A.T @ y
    lam = -spla.splu(sp.csc_matrix(Gx)).solve(grad[n_u:], trans="T")
    return lam, grad[:n_u] + Gu.T @ lam


def reduced_value(net, part, point, y, u):
    """φ(u) = f(x(u),u) + yᵀ[r; h](x(u),u), x(u) by Newton (the reduced
    Lagrangian's smooth part, Theorem 'Reduced derivatives' L967–990)."""
    pt = set_u(part, point, u)
    pt, _, _ = newton(net, part, pt, tol=1e-14)
    p, q = injections(net, pt["v"], pt["theta"])
    r = np.array([p[i] if t == 0 else q[i] for (i, t) in part["r_rows"]])
    sf, st = line_flows(net, pt["v"], pt["theta"])
    h = np.array([abs(sf[l]) ** 2 if e == 0 else abs(st[l]) ** 2 for (l, e) in part["h_rows"]])
    return objective(net, part, pt) + y @ np.concatenate([r, h])


# ----------------------------------------------------------------------------
# O9 augmented KKT (PAPER.md eq. kktmatrix:normal L626–634), case9 only
# ----------------------------------------------------------------------------
def kaug(W, Gx, Gu, A, sigma_u, sigma_x, sigma_s):
    """Dense K_aug with blocks ordered (p_u, p_x, p_s, p_λ, p_y)."""
    n_x, n_u = Gu.shape
    m = A.shape[0]
    W = np.asarray(sp.csr_matrix(W).toarray())
    A = np.asarray(sp.csr_matrix(A).toarray())
    Gu = np.asarray(sp.csr_matrix(Gu).toarray())
    Gx = np.asarray(sp.csr_matrix(Gx).toarray())
    Au, Ax = A[:, :n_u], A[:, n_u:]
    n = n_u + n_x + m + n_x + m
    K = np.zeros((n, n))
    iu, ix, is_, il, iy = 0, n_u, n_u + n_x, n_u + n_x + m, n_u + n_x + m + n_x
    K[iu:ix, iu:ix] = W[:n_u, :n_u] + np.diag(sigma_u)
    K[iu:ix, ix:is_] = W[:n_u, n_u:]
    K[ix:is_, iu:ix] = W[n_u:, :n_u]
    K[ix:is_, ix:is_] = W[n_u:, n_u:] + np.diag(sigma_x)
    K[is_:il, is_:il] = np.diag(sigma_s)
    K[is_:il, iy:] = -np.eye(m)
    K[iy:, is_:il] = -np.eye(m)
    K[iu:ix, il:iy] = Gu.T
    K[ix:is_, il:iy] = Gx.T
    K[il:iy, iu:ix] = Gu
    K[il:iy, ix:is_] = Gx
    K[iu:ix, iy:] = Au.T
    K[ix:is_, iy:] = Ax.T
    K[iy:, iu:ix] = Au
    K[iy:, ix:is_] = Ax
    return K


# ----------------------------------------------------------------------------
# NEXT-1: condensed right-hand side and step recovery (Theorem 1 P:L671–719,
# Theorem 2, Algorithm 1), dense, in the paper's order
# and notation, with reading R10 (the signs of the r̂₂ terms).
# W is the Lagrangian Hessian ∇²ℒ (lagrangian_hessian: no Σ, no AᵀΣ_sA).
# The right-hand side r = (r₁, r₂, r₃, r₄, r₅) of eq. kktmatrix:normal is
# ordered like kaug's blocks (p_u, p_x, p_s, p_λ, p_y): K_aug p = −r.
# ----------------------------------------------------------------------------
def split_kkt(vec, n_u, n_x, m):
    o = np.cumsum([0, n_u, n_x, m, n_x, m])
    return [np.asarray(vec[o[k]:o[k + 1]], dtype=np.float64) for k in range(5)]


def condensed_rhs(W, Gx, Gu, A, sigma_x, sigma_s, r):
    """Theorem 1: r̂₁ = r₁ − G_uᵀG_x⁻ᵀr₂ − (W_ux − G_uᵀG_x⁻ᵀ(W_xx+Σ_x))G_x⁻¹r₄,
    r̂₂ = r₃, r̂₃ = r₅ − A_xG_x⁻¹r₄, Â_u = A_u − A_xG_x⁻¹G_u; Theorem 2 (R10):
    K_cond p_u = −(r̂₁ + Â_uᵀΣ_s r̂₃ + Â_uᵀ r̂₂).  Returns (b, (r̂₁, r̂₂, r̂₃), Â_u)."""
    Gx = np.asarray(sp.csr_matrix(Gx).toarray())
    Gu = np.asarray(sp.csr_matrix(Gu).toarray())
    A = np.asarray(sp.csr_matrix(A).toarray())
    W = np.asarray(sp.csr_matrix(W).toarray())
    n_x, n_u = Gu.shape
    m = A.shape[0]
    r1, r2, r3, r4, r5 = split_kkt(r, n_u, n_x, m)
    Wux, Wxx = W[:n_u, n_u:], W[n_u:, n_u:] + np.diag(sigma_x)
    Au, Ax = A[:, :n_u], A[:, n_u:]
    Gx_inv_r4 = np.linalg.solve(Gx, r4)
    rh1 = r1 - Gu.T @ np.linalg.solve(Gx.T, r2) - (Wux - Gu.T @ np.linalg.solve(Gx.T, Wxx)) @ Gx_inv_r4
    rh2 = r3
    rh3 = r5 - Ax @ Gx_inv_r4
    Ahat = Au - Ax @ np.linalg.solve(Gx, Gu)
    b = -(rh1 + Ahat.T @ (sigma_s * rh3) + Ahat.T @ rh2)
    return b, (rh1, rh2, rh3), Ahat


def recover_step(W, Gx, Gu, A, sigma_x, sigma_s, r, p_u, lu=None):
    """Algorithm 1's dual, slack, state and adjoint steps (Theorem 1 recovery,
    Theorem 2 with R10): p_y = Σ_s(Â_u p_u + r̂₃ + Σ_s⁻¹r̂₂), p_s = Σ_s⁻¹(p_y − r̂₂),
    p_x = −G_x⁻¹(r₄ + G_u p_u), p_λ = −G_x⁻ᵀ(r₂ + A_xᵀp_y + W_xu p_u + (W_xx+Σ_x)p_x).
    Returns the step ordered (p_u, p_x, p_s, p_λ, p_y).  lu: None = dense
    LAPACK solves with G_x, or a SparseLU (an independent factorization, for
    the measured noise floor of R20) for the p_x and p_λ solves."""
    _, (rh1, rh2, rh3), Ahat = condensed_rhs(W, Gx, Gu, A, sigma_x, sigma_s, r)
    if lu is not None:
        solve = lambda b: lu.solve(b)                  # noqa: E731
        solve_t = lambda b: lu.solve(b, trans="T")     # noqa: E731
    Gx = np.asarray(sp.csr_matrix(Gx).toarray())
    if lu is None:
        solve = lambda b: np.linalg.solve(Gx, b)       # noqa: E731
        solve_t = lambda b: np.linalg.solve(Gx.T, b)   # noqa: E731
    Gu = np.asarray(sp.csr_matrix(Gu).toarray())
    A = np.asarray(sp.csr_matrix(A).toarray())
    W = np.asarray(sp.csr_matrix(W).toarray())
    n_x, n_u = Gu.shape
    m = A.shape[0]
    r1, r2, r3, r4, r5 = split_kkt(r, n_u, n_x, m)
    Wxu, Wxx = W[n_u:, :n_u], W[n_u:, n_u:] + np.diag(sigma_x)
    Ax = A[:, n_u:]
    p_y = sigma_s * (Ahat @ p_u + rh3 + rh2 / sigma_s)
    p_s = (p_y - rh2) / sigma_s
    p_x = -solve(r4 + Gu @ p_u)
    p_l = -solve_t(r2 + Ax.T @ p_y + Wxu @ p_u + Wxx @ p_x)
    return np.concatenate([p_u, p_x, p_s, p_l, p_y])


def gauss_jordan_inverse(M):
    """Plain Gauss–Jordan with partial pivoting (for the Schur pin P10)."""
    n = M.shape[0]
    A = np.hstack([np.array(M, dtype=np.float64), np.eye(n)])
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        A[[k, p]] = A[[p, k]]
        A[k] /= A[k, k]
        for i in range(n):
            if i != k:
                A[i] -= A[i, k] * A[k]
    return A[:, n:]


def jacobi_eigenvalues(M, sweeps=60, tol=1e-13):
    """Cyclic Jacobi eigenvalues of a symmetric matrix (inertia, P11):
    rotate rows/columns p, q to annihilate A[p, q] until the off-diagonal
    norm is negligible."""
    A = np.array(M, dtype=np.float64, copy=True)
    n = A.shape[0]
    scale = max(1.0, np.abs(A).max())
    for _ in range(sweeps):
        off = np.sqrt(max(np.sum(A * A) - np.sum(np.diag(A) ** 2), 0.0))
        if off < tol * scale:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if abs(apq) < 1e-300:
                    continue
                tau = (A[q, q] - A[p, p]) / (2 * apq)
                t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + np.hypot(1.0, tau))
                c = 1 / np.sqrt(1 + t * t)
                s = t * c
                Ap, Aq = A[:, p].copy(), A[:, q].copy()
                A[:, p] = c * Ap - s * Aq
                A[:, q] = s * Ap + c * Aq
                Ap, Aq = A[p, :].copy(), A[q, :].copy()
                A[p, :] = c * Ap - s * Aq
                A[q, :] = s * Ap + c * Aq
    return np.diag(A)


# ----------------------------------------------------------------------------
# O10 structure (R18, R19): patterns,
# ordering, symbolic LU and level sets, written independently of the library.
# ----------------------------------------------------------------------------
def bus_adjacency(net):
    n_b = int(net["n_b"])
    adj = [set() for _ in range(n_b)]
    for f, t in zip(net["line_from"], net["line_to"]):
        f, t = int(f), int(t)
        if f != t:
            adj[f].add(t)
            adj[t].add(f)
    return adj


def gx_gu_patterns(net, part):
    """Topological CSR patterns (sorted int32 columns) of G_x and G_u (R19)."""
    adj = bus_adjacency(net)
    n_b = part["n_b"]
    x_th, x_v, u_v, u_p = part["x_th"], part["x_v"], part["u_v"], part["u_p"]
    rows_x = [[] for _ in range(part["n_x"])]
    rows_u = [[] for _ in range(part["n_x"])]
    for i in range(n_b):
        for r in (x_th[i], x_v[i]):
            if r < 0:
                continue
            for j in sorted(adj[i] | {i}):
                for c in (x_th[j], x_v[j]):
                    if c >= 0:
                        rows_x[r].append(c)
                if u_v[j] >= 0:
                    rows_u[r].append(u_v[j])
    gb = np.asarray(net["gen_bus"])
    for g in range(part["n_g"]):
        if u_p[g] >= 0:
            rows_u[x_th[gb[g]]].append(u_p[g])

    def csr(rows):
        ptr = np.zeros(len(rows) + 1, dtype=np.int32)
        idx = []
        for k, r in enumerate(rows):
            r = sorted(set(r))
            idx += r
            ptr[k + 1] = ptr[k] + len(r)
        return ptr, np.array(idx, dtype=np.int32)

    return csr(rows_x), csr(rows_u)


def md_ordering(net, part):
    """R18 written rule: exact minimum degree on the elimination graph of the
    buses that carry state variables (all but r0); the bus of minimum current
    degree is eliminated next, ties to the lowest bus index; eliminating a bus
    joins its remaining neighbours into a clique.  Returns the bus order."""
    n_b, r0 = part["n_b"], part["r0"]
    adj = bus_adjacency(net)
    g = {i: set(a) - {r0} for i, a in enumerate(adj) if i != r0}
    heap = [(len(nb), i) for i, nb in g.items()]
    heapq.heapify(heap)
    order, done = [], set()
    while heap:
        d, i = heapq.heappop(heap)
        if i in done or d != len(g[i]):
            continue
        order.append(i)
        done.add(i)
        nb = g.pop(i)
        for a in nb:
            g[a].discard(i)
            g[a] |= (nb - {a})
        for a in nb:
            heapq.heappush(heap, (len(g[a]), a))
    return np.array(order, dtype=np.int32)


def permutation(part, bus_order):
    """perm[k] = x index placed at position k: for each bus in order, θ then v."""
    perm = []
    blk = [0]
    for i in bus_order:
        for c in (part["x_th"][i], part["x_v"][i]):
            if c >= 0:
                perm.append(c)
        blk.append(len(perm))
    return np.array(perm, dtype=np.int32), np.array(blk, dtype=np.int32)


def symbolic_lu(ptr, idx, perm):
    """Dense Boolean elimination of P G_x Pᵀ (no numerical pivoting).  Returns
    the boolean filled pattern F (strict lower = L, upper incl. diagonal = U)."""
    n = len(perm)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    F = np.zeros((n, n), dtype=bool)
    for r in range(n):
        F[inv[r], inv[idx[ptr[r]:ptr[r + 1]]]] = True
    for k in range(n):
        rows = np.nonzero(F[k + 1:, k])[0] + k + 1
        if len(rows):
            F[np.ix_(rows, np.arange(k + 1, n))] |= F[k, k + 1:][None, :]
    return F


def block_levels(F, blk):
    """Level of each diagonal block (bus) in the forward (L) and backward (U)
    triangular-solve DAGs: 0 for sources, else 1 + max over blocks it reads
    (longest path, computed by Kahn's topological sweep).  Returns
    (lev_L, lev_U) per block."""
    nblk = len(blk) - 1
    owner = np.empty(blk[-1], dtype=np.int64)
    for b in range(nblk):
        owner[blk[b]:blk[b + 1]] = b
    depL = [set() for _ in range(nblk)]
    depU = [set() for _ in range(nblk)]
    rr, cc = np.nonzero(F)
    for r, c in zip(rr, cc):
        br, bc = owner[r], owner[c]
        if bc < br:
            depL[br].add(bc)
        elif bc > br:
            depU[br].add(bc)

    def kahn(dep):
        indeg = np.array([len(d) for d in dep])
        users = [[] for _ in range(nblk)]
        for b, d in enumerate(dep):
            for a in d:
                users[a].append(b)
        lev = np.zeros(nblk, dtype=np.int64)
        frontier = [b for b in range(nblk) if indeg[b] == 0]
        while frontier:
            nxt = []
            for a in frontier:
                for b in users[a]:
                    lev[b] = max(lev[b], lev[a] + 1)
                    indeg[b] -= 1
                    if indeg[b] == 0:
                        nxt.append(b)
            frontier = nxt
        return lev

    return kahn(depL), kahn(depU)


def level_sets(lev):
    """(level_ptr, level_blocks): blocks grouped by level, ascending within a level."""
    nl = int(lev.max()) + 1 if len(lev) else 0
    ptr = np.zeros(nl + 1, dtype=np.int32)
    blocks = []
    for l in range(nl):
        b = np.nonzero(lev == l)[0]
        blocks += list(b)
        ptr[l + 1] = ptr[l] + len(b)
    return ptr, np.array(blocks, dtype=np.int32)


def a_pattern(net, part):
    """Topological CSR pattern of A = ∂[r; h]/∂[u; x] (R19): an r row of bus i
    depends on the variables of i and its neighbours, an h row of line ℓ on
    the variables of its two end buses."""
    adj = bus_adjacency(net)
    zv, zth = z_index(part)
    rows = []
    for (i, t) in part["r_rows"]:
        cols = set()
        for j in adj[i] | {i}:
            cols.add(int(zv[j]))
            if zth[j] >= 0:
                cols.add(int(zth[j]))
        rows.append(sorted(cols))
    for (l, e) in part["h_rows"]:
        cols = set()
        for j in (int(net["line_from"][l]), int(net["line_to"][l])):
            cols.add(int(zv[j]))
            if zth[j] >= 0:
                cols.add(int(zth[j]))
        rows.append(sorted(cols))
    ptr = np.zeros(len(rows) + 1, dtype=np.int32)
    for k, r in enumerate(rows):
        ptr[k + 1] = ptr[k] + len(r)
    return ptr, np.array([c for r in rows for c in r], dtype=np.int32)


def static_lu(Gx, perm, rel=1e-12):
    """R18 numeric refactorization rule, written out: dense LU of P G_x Pᵀ
    (P from the R18 ordering) with NO pivoting, right-looking.  Pivot k fails
    iff u_kk is non-finite, zero, or |u_kk| < rel · max_j |(P G_x Pᵀ)_kj|; the
    first failure stops the factorization.  Returns (info, LU): info = 0 or
    k+1; LU holds L (unit, strict lower) and U (upper) of the rows done."""
    A = np.asarray(sp.csr_matrix(Gx).toarray(), dtype=np.float64)[np.ix_(perm, perm)]
    n = A.shape[0]
    rowmax = np.abs(A).max(axis=1) if n else np.zeros(0)
    for k in range(n):
        d = A[k, k]
        if not np.isfinite(d) or d == 0.0 or abs(d) < rel * rowmax[k]:
            return k + 1, A
        A[k + 1:, k] /= d
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    return 0, A


def filled_csr(F):
    """CSR (ptr, idx) of a boolean filled pattern."""
    ptr = np.zeros(F.shape[0] + 1, dtype=np.int32)
    idx = []
    for r in range(F.shape[0]):
        c = np.nonzero(F[r])[0]
        idx.append(c)
        ptr[r + 1] = ptr[r] + len(c)
    return ptr, np.concatenate(idx).astype(np.int32) if idx else np.zeros(0, np.int32)


class SparseLU:
    """A sparse LU of G_x used as a solve primitive (SuperLU), in one of three
    independent variants (for the measured noise floor of R20):
      "colamd": SuperLU defaults — COLAMD column ordering, partial pivoting;
      "mmd":    minimum degree on AᵀA+A, static diagonal pivots;
      "static": the R18 rule itself — P G_x Pᵀ with the given bus-level
                ordering perm, natural order inside SuperLU, diagonal pivots
                (no numerical pivoting), i.e. the algorithm the GPU runs."""

    def __init__(self, Gx, kind="colamd", perm=None):
        A = sp.csc_matrix(Gx)
        self.perm = None
        if kind == "colamd":
            self.lu = spla.splu(A)
        elif kind == "mmd":
            self.lu = spla.splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                                options=dict(SymmetricMode=True))
        elif kind == "static":
            self.perm = np.asarray(perm)
            Ap = sp.csc_matrix(A[self.perm][:, self.perm])
            self.lu = spla.splu(Ap, permc_spec="NATURAL", diag_pivot_thresh=0.0,
                                options=dict(SymmetricMode=True))
            n = len(self.perm)
            assert np.array_equal(self.lu.perm_r, np.arange(n)) and np.array_equal(self.lu.perm_c, np.arange(n))
        else:
            raise ValueError(kind)

    def solve(self, B, trans="N"):
        B = np.asarray(B, dtype=np.float64)
        if self.perm is None:
            return self.lu.solve(B, trans=trans)
        X = np.empty_like(B)
        X[self.perm] = self.lu.solve(B[self.perm], trans=trans)   # (P G_x Pᵀ)⁻¹ and its transpose
        return X


def reduce_columns(K, Gx, Gu, cols, kind="colamd", perm=None):
    """O7' for selected unit directions (full-size parity): the three steps of
    PAPER.md L1203–1222 with R11 for V = I[:, cols], with a sparse LU of G_x
    (SparseLU `kind`) as the solve primitive."""
    n_u = Gu.shape[1]
    V = np.zeros((n_u, len(cols)))
    V[cols, np.arange(len(cols))] = 1.0
    lu = SparseLU(Gx, kind, perm)
    Gu = sp.csr_matrix(Gu)
    Z = -lu.solve(np.asarray((Gu @ V)))
    H = sp.csr_matrix(K) @ np.vstack([V, Z])
    Hu, Hx = H[:n_u], H[n_u:]
    Psi = lu.solve(np.asarray(Hx), trans="T")
    return Hu - Gu.T @ Psi
