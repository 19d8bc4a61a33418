"""NEXT-4 — the linearize-then-reduce interior-point driver (LinRed, Algorithm 1,
P:L868–895) with a filter line search, on top of the C-ABI.

This is the role MadNLP plays in the paper: the outer IPM
logic — barrier parameter, fraction to the boundary, filter line search, the
O(n) vector updates of the iterate — runs on the host, while every piece of
KKT linear algebra of an iteration runs in libpf.so's kernels:

  pf_eval_constraints  f, g, r, h at the iterate (A2/A3)
  pf_jacobian          G_x, G_u, A and the LU of G_x (A4/A5)
  pf_reduced_hessian_batch   K̂ (all n_u HVPs, A6/A7)
  pf_condensed_rhs     Theorem 1/2's right-hand side (NEXT-1, R10)
  pf_condensed_kkt_solve_reg K_cond p_u = b inside the δ_w loop (A9 + NEXT-3)
  pf_recover_step      p_x, p_s, p_λ, p_y (NEXT-1)

Problem (P:L472–495 with the slack form of K_aug, eq. kktmatrix:normal as
printed at P:L626–634):  min f(x,u)  s.t.  g(x,u) = 0,  c(x,u) − s = 0,
lo ≤ (u, x, s) ≤ up, with c = [r; h] (r = injections at
[P_ref; Q_ref; Q_PV], h = |s_flow|² at limited line ends).  OPF bounds
(MATPOWER convention): v ∈ [v_lo, v_hi] at every bus (u at generator buses,
x elsewhere), p_g ∈ [p_lo, p_hi] for g ≠ g_ref (u), p_ref ∈ [p_lo, p_hi]
and q_g ∈ [q_lo, q_hi] through r (loads shift the bounds, R7), h ≤ F_max².
Barrier subproblem residuals (two-sided bounds, primal-dual Σ = z_L/(w−lo) +
z_U/(up−w), R16):
  r₁ = ∇_u f + G_uᵀλ + A_uᵀy − μ/(u−lo) + μ/(up−u),  r₂ likewise for x,
  r₃ = −y − μ/(s−lo) + μ/(up−s),  r₄ = g,  r₅ = c − s.
Filter line search after Wächter & Biegler (the paper's MadNLP/Ipopt
default): θ = ‖(g, c − s)‖₁, φ = f − μ Σ log(bound distances), switching
condition + Armijo on φ, filter augmentation, fraction-to-boundary
τ = max(0.99, 1 − μ); Fiacco–McCormick barrier updates
μ ← max(tol/10, min(κ_μ μ, μ^1.5)); convergence when the scaled optimality
error ≤ tol (the paper's 1e-8).  No restoration phase: a line search
that collapses below α_min stops with status "line search failed".
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .pf import Network


class LinRedIPM:
    """One network, one scenario.  bounds: dict with v_lo, v_hi [n_b],
    p_lo, p_hi, q_lo, q_hi [n_g] (p.u.)."""

    def __init__(self, net, bounds, device=0, tol=1e-8, max_iter=200, mu0=0.1, verbose=False):
        import torch
        self.torch = torch
        self.net = net
        self.b = {k: np.asarray(v, dtype=np.float64) for k, v in bounds.items()}
        self.tol, self.max_iter, self.mu0, self.verbose = tol, max_iter, mu0, verbose
        tmp = Network(net, max_batch=1, max_scen=1, device=-1)
        n_u = tmp.dims["n_u"]
        tmp.close()
        self.h = Network(net, max_batch=n_u, max_scen=1, device=device)
        d = self.h.dims
        self.d = d
        self.dev = torch.device("cuda", device)
        n_b, n_g, n_l = d["n_b"], d["n_g"], d["n_l"]
        self.n_b, self.n_g, self.n_l = n_b, n_g, n_l
        self.n_u, self.n_x, self.m, self.n_r, self.n_h = d["n_u"], d["n_x"], d["m"], d["n_r"], d["n_h"]
        st = self.h.structure
        self.x_th, self.x_v, self.u_v, self.u_p = st("x_theta"), st("x_v"), st("u_v"), st("u_p")
        self.gx = (st("gx_ptr"), st("gx_idx"))
        self.gu = (st("gu_ptr"), st("gu_idx"))
        self.ap = (st("a_ptr"), st("a_idx"))
        gen_bus = np.asarray(net["gen_bus"])
        self.gen_bus = gen_bus
        self.r0, self.g_r = d["ref_bus"], d["ref_gen"]
        pv = [i for i in range(n_b) if self.u_v[i] >= 0 and i != self.r0]
        # r rows: P_ref, Q_ref, Q_i for PV buses ascending; their bus and kind
        self.r_bus = np.array([self.r0, self.r0] + pv, dtype=np.int64)
        self.r_isq = np.array([0, 1] + [1] * len(pv), dtype=bool)
        F = np.asarray(net["F_max"], dtype=np.float64)
        self.lim = np.nonzero(F > 0)[0]
        self.p_d, self.q_d = np.asarray(net["p_d"], np.float64), np.asarray(net["q_d"], np.float64)
        self.c1, self.c2 = np.asarray(net["c_quad"], np.float64), np.asarray(net["c_lin"], np.float64)
        self._bounds(F)

    # ------------------------------------------------------------------ layout
    def _bounds(self, F):
        b, n_b = self.b, self.n_b
        lo_u, up_u = np.full(self.n_u, -np.inf), np.full(self.n_u, np.inf)
        lo_x, up_x = np.full(self.n_x, -np.inf), np.full(self.n_x, np.inf)
        for i in range(n_b):
            if self.u_v[i] >= 0:
                lo_u[self.u_v[i]], up_u[self.u_v[i]] = b["v_lo"][i], b["v_hi"][i]
            if self.x_v[i] >= 0:
                lo_x[self.x_v[i]], up_x[self.x_v[i]] = b["v_lo"][i], b["v_hi"][i]
        for g in range(self.n_g):
            if self.u_p[g] >= 0:
                lo_u[self.u_p[g]], up_u[self.u_p[g]] = b["p_lo"][g], b["p_hi"][g]
        gen_of = {int(bus): g for g, bus in enumerate(self.gen_bus)}
        lo_s, up_s = np.full(self.m, -np.inf), np.full(self.m, np.inf)
        for k, (i, isq) in enumerate(zip(self.r_bus, self.r_isq)):
            g = gen_of[int(i)]
            if isq:   # Q_inj = q_g − q_d (R7)
                lo_s[k], up_s[k] = b["q_lo"][g] - self.q_d[i], b["q_hi"][g] - self.q_d[i]
            else:     # P_inj,ref = p_ref − p_d
                lo_s[k], up_s[k] = b["p_lo"][g] - self.p_d[i], b["p_hi"][g] - self.p_d[i]
        nl = len(self.lim)
        up_s[self.n_r:self.n_r + nl] = F[self.lim] ** 2
        up_s[self.n_r + nl:] = F[self.lim] ** 2
        self.lo = np.concatenate([lo_u, lo_x, lo_s])
        self.up = np.concatenate([up_u, up_x, up_s])
        self.hasl, self.hasu = np.isfinite(self.lo), np.isfinite(self.up)

    def _to_bus(self, u, x, p_g_ref=0.0):
        """(v, θ, p_g) of the iterate; the reference generator's p_g slot is p_g_ref."""
        v, th, pg = np.zeros(self.n_b), np.zeros(self.n_b), np.zeros(self.n_g)
        for i in range(self.n_b):
            if self.x_th[i] >= 0:
                th[i] = x[self.x_th[i]]
            if self.x_v[i] >= 0:
                v[i] = x[self.x_v[i]]
            if self.u_v[i] >= 0:
                v[i] = u[self.u_v[i]]
        for g in range(self.n_g):
            pg[g] = u[self.u_p[g]] if self.u_p[g] >= 0 else p_g_ref
        return v, th, pg

    def _dv(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)[None]), device=self.dev)

    # ------------------------------------------------------------------ functions (through the C-ABI)
    def evaluate(self, w):
        """f, g, c and the p_ref of the iterate w = (u, x, s)."""
        torch = self.torch
        u, x = w[:self.n_u], w[self.n_u:self.n_u + self.n_x]
        v, th, pg = self._to_bus(u, x)
        G = torch.empty(1, 2 * self.n_b, dtype=torch.float64, device=self.dev)
        H = torch.empty(1, 2 * self.n_l, dtype=torch.float64, device=self.dev)
        # q_g = 0 and the reference p_g = 0: G then carries the injections plus loads at r rows
        self.h.pf_eval_constraints(1, self._dv(v), self._dv(th), self._dv(pg), self._dv(np.zeros(self.n_g)),
                                   self._dv(self.p_d), self._dv(self.q_d), G, H)
        G, H = G[0].cpu().numpy(), H[0].cpu().numpy()
        g = np.empty(self.n_x)
        for i in range(self.n_b):
            if self.x_th[i] >= 0:
                g[self.x_th[i]] = G[i]
            if self.x_v[i] >= 0:
                g[self.x_v[i]] = G[self.n_b + i]
        Pinj = G[:self.n_b] - self.p_d
        Qinj = G[self.n_b:] - self.q_d
        r = np.where(self.r_isq, Qinj[self.r_bus], Pinj[self.r_bus])
        c = np.concatenate([r, H[self.lim], H[self.n_l + self.lim]])
        p_ref = Pinj[self.r0] + self.p_d[self.r0]
        f = self.c1[self.g_r] * p_ref ** 2 + self.c2[self.g_r] * p_ref
        for gg in range(self.n_g):
            if self.u_p[gg] >= 0:
                f += self.c1[gg] * pg[gg] ** 2 + self.c2[gg] * pg[gg]
        return f, g, c, p_ref

    def derivatives(self, w, v_dev, th_dev, p_ref):
        """G_x, G_u, A (host CSR copies of the device Jacobians) and ∇f over z = [u; x]."""
        torch = self.torch
        d = self.d
        Gx = torch.empty(1, d["nnz_gx"], dtype=torch.float64, device=self.dev)
        Gu = torch.empty(1, d["nnz_gu"], dtype=torch.float64, device=self.dev)
        A = torch.empty(1, d["nnz_a"], dtype=torch.float64, device=self.dev)
        info = torch.empty(1, dtype=torch.int32, device=self.dev)
        self.h.pf_jacobian(1, v_dev, th_dev, Gx, Gu, A, info)
        if int(info.item()) != 0:
            raise RuntimeError("singular G_x at the iterate (R18 pivot %d)" % int(info.item()))
        csr = lambda vals, pi, shape: sp.csr_matrix((vals[0].cpu().numpy(), pi[1], pi[0]), shape=shape)  # noqa
        Gxm = csr(Gx, self.gx, (self.n_x, self.n_x))
        Gum = csr(Gu, self.gu, (self.n_x, self.n_u))
        Am = csr(A, self.ap, (self.m, self.n_u + self.n_x))
        u = w[:self.n_u]
        gf = (2 * self.c1[self.g_r] * p_ref + self.c2[self.g_r]) * Am.getrow(0).toarray().ravel()  # R8: ∇p_ref = A row P_ref
        for gg in range(self.n_g):
            if self.u_p[gg] >= 0:
                gf[self.u_p[gg]] += 2 * self.c1[gg] * u[self.u_p[gg]] + self.c2[gg]
        return Gxm, Gum, Am, gf

    # ------------------------------------------------------------------ IPM pieces
    def _slacks(self, w):
        dl = np.where(self.hasl, w - self.lo, 1.0)
        du = np.where(self.hasu, self.up - w, 1.0)
        return dl, du

    def barrier(self, f, w, mu):
        dl, du = self._slacks(w)
        return f - mu * (np.sum(np.log(dl[self.hasl])) + np.sum(np.log(du[self.hasu])))

    def _interior(self, w):
        """Push a starting point strictly inside its bounds (Ipopt's κ₁ = κ₂ = 1e-2 rule)."""
        lo = np.where(self.hasl, self.lo, 0.0)
        up = np.where(self.hasu, self.up, 0.0)
        both = self.hasl & self.hasu
        width = np.where(both, up - lo, np.inf)
        pl = np.minimum(1e-2 * np.maximum(1, np.abs(lo)), 1e-2 * width)
        pu = np.minimum(1e-2 * np.maximum(1, np.abs(up)), 1e-2 * width)
        w = np.where(self.hasl, np.maximum(w, lo + pl), w)
        return np.where(self.hasu, np.minimum(w, up - pu), w)

    def solve(self, v0=None, theta0=None, p_g0=None):
        torch = self.torch
        n_u, n_x, m = self.n_u, self.n_x, self.m
        nz = n_u + n_x
        b = self.b
        v0 = np.ones(self.n_b) if v0 is None else np.asarray(v0, np.float64)
        theta0 = np.zeros(self.n_b) if theta0 is None else np.asarray(theta0, np.float64)
        p_g0 = 0.5 * (b["p_lo"] + b["p_hi"]) if p_g0 is None else np.asarray(p_g0, np.float64)
        u = np.zeros(n_u)
        x = np.zeros(n_x)
        for i in range(self.n_b):
            if self.u_v[i] >= 0:
                u[self.u_v[i]] = v0[i]
            if self.x_th[i] >= 0:
                x[self.x_th[i]] = theta0[i]
            if self.x_v[i] >= 0:
                x[self.x_v[i]] = v0[i]
        for g in range(self.n_g):
            if self.u_p[g] >= 0:
                u[self.u_p[g]] = p_g0[g]
        w = np.concatenate([u, x, np.zeros(m)])
        f, g, c, p_ref = self.evaluate(w)
        w[nz:] = c
        w = self._interior(w)
        mu = self.mu0
        lam, y = np.zeros(n_x), np.zeros(m)
        dl, du = self._slacks(w)
        zl = np.where(self.hasl, mu / dl, 0.0)
        zu = np.where(self.hasu, mu / du, 0.0)
        f, g, c, p_ref = self.evaluate(w)
        theta = np.abs(g).sum() + np.abs(c - w[nz:]).sum()
        th_max, th_min = 1e4 * max(1.0, theta), 1e-4 * max(1.0, theta)
        filt = []
        hist = []
        status = "max_iter"
        delta_prev = 0.0
        for it in range(self.max_iter + 1):
            u, x, s = w[:n_u], w[n_u:nz], w[nz:]
            v, th, _ = self._to_bus(u, x)
            v_dev, th_dev = self._dv(v), self._dv(th)
            Gx, Gu, A, gf = self.derivatives(w, v_dev, th_dev, p_ref)
            dl, du = self._slacks(w)
            # optimality error (Ipopt's scaled E_μ)
            grad_z = gf + np.concatenate([Gu.T @ lam, Gx.T @ lam]) + A.T @ y
            dual_z = grad_z - zl[:nz] + zu[:nz]
            dual_s = -y - zl[nz:] + zu[nz:]
            ncomp = int(self.hasl.sum() + self.hasu.sum())
            s_d = max(100.0, (np.abs(lam).sum() + np.abs(y).sum() + zl.sum() + zu.sum()) / max(1, n_x + m + ncomp)) / 100
            s_c = max(100.0, (zl.sum() + zu.sum()) / max(1, ncomp)) / 100

            def err(mu_):
                comp = max(np.max(np.abs(np.where(self.hasl, zl * dl - mu_, 0.0))),
                           np.max(np.abs(np.where(self.hasu, zu * du - mu_, 0.0))))
                return max(max(np.abs(dual_z).max(), np.abs(dual_s).max()) / s_d,
                           max(np.abs(g).max(), np.abs(c - s).max()), comp / s_c)

            e0 = err(0.0)
            hist.append(dict(it=it, f=f, mu=mu, inf_pr=max(np.abs(g).max(), np.abs(c - s).max()),
                             inf_du=max(np.abs(dual_z).max(), np.abs(dual_s).max()), err=e0, delta_w=delta_prev))
            if self.verbose:
                print("%3d f=%.8e mu=%.1e pr=%.2e du=%.2e err=%.2e" % (it, f, mu, hist[-1]["inf_pr"], hist[-1]["inf_du"], e0))
            if e0 <= self.tol:
                status = "converged"
                break
            if it == self.max_iter:
                break
            while err(mu) <= 10.0 * mu and mu > self.tol / 10:   # barrier subproblem solved: decrease μ
                mu = max(self.tol / 10, min(0.2 * mu, mu ** 1.5))
                filt = []
            # ---------------- the LinRed step (Algorithm 1) on the device
            sig = np.where(self.hasl, zl / dl, 0.0) + np.where(self.hasu, zu / du, 0.0)
            bar = np.where(self.hasl, mu / dl, 0.0) - np.where(self.hasu, mu / du, 0.0)
            r1 = grad_z[:n_u] - bar[:n_u]
            r2 = grad_z[n_u:] - bar[n_u:nz]
            r3 = -y - bar[nz:]
            r = np.concatenate([r1, r2, r3, g, c - s])
            d_lam, d_y = self._dv(lam), self._dv(y)
            d_ss, d_sx, d_pd = self._dv(sig[nz:]), self._dv(sig[n_u:nz]), self._dv(self.p_d)
            KV = torch.empty(1, n_u, n_u, dtype=torch.float64, device=self.dev)
            self.h.pf_reduced_hessian_batch(1, v_dev, th_dev, d_lam, d_y, KV, sigma_s=d_ss, sigma_x=d_sx, p_d=d_pd)
            rd = self._dv(r)
            bvec = self.h.pf_condensed_rhs(1, v_dev, th_dev, d_lam, d_y, rd, sigma_s=d_ss, sigma_x=d_sx, p_d=d_pd)
            # δ_w loop (NEXT-3, Ipopt's schedule): 0 first; then 1e-4 ×100, or δ_last/3 ×8 once one was needed
            first = 1e-4 if delta_prev == 0.0 else max(1e-20, delta_prev / 3)
            delta, trials, info = self.h.pf_condensed_kkt_solve_reg(1, KV, self._dv(sig[:n_u]), 0.0, first,
                                                                    100.0 if delta_prev == 0.0 else 8.0, 1e40,
                                                                    rhs=bvec, nrhs=1)
            if info[0] != 0:
                status = "regularization failed"
                break
            delta_prev = float(delta[0])
            p = self.h.pf_recover_step(1, v_dev, th_dev, d_lam, d_y, rd, bvec, sigma_s=d_ss, sigma_x=d_sx,
                                       p_d=d_pd)[0].cpu().numpy()
            o = np.cumsum([0, n_u, n_x, m, n_x, m])
            pw = np.concatenate([p[o[0]:o[1]], p[o[1]:o[2]], p[o[2]:o[3]]])
            plam, py = p[o[3]:o[4]], p[o[4]:o[5]]
            pzl = np.where(self.hasl, (mu - zl * dl - zl * pw) / dl, 0.0)
            pzu = np.where(self.hasu, (mu - zu * du + zu * pw) / du, 0.0)
            # ---------------- fraction to the boundary
            tau = max(0.99, 1.0 - mu)

            def max_step(val, dval, mask):
                neg = mask & (dval < 0)
                return min(1.0, float(np.min(-tau * val[neg] / dval[neg]))) if np.any(neg) else 1.0

            a_max = min(max_step(dl, pw, self.hasl), max_step(du, -pw, self.hasu))
            a_z = min(max_step(zl, pzl, self.hasl), max_step(zu, pzu, self.hasu))
            # ---------------- filter line search
            phi = self.barrier(f, w, mu)
            gphi = np.concatenate([gf, np.zeros(m)]) - bar
            dphi = float(gphi @ pw)
            alpha, accepted = a_max, False
            a_min = 1e-12
            while alpha >= a_min:
                wt = w + alpha * pw
                ft, gt, ct, pref_t = self.evaluate(wt)
                tht = np.abs(gt).sum() + np.abs(ct - wt[nz:]).sum()
                phit = self.barrier(ft, wt, mu) if np.all(self._slacks(wt)[0][self.hasl] > 0) and \
                    np.all(self._slacks(wt)[1][self.hasu] > 0) else np.inf
                if tht <= th_max and np.isfinite(phit) and not any(tht >= ft_ and phit >= fp_ for ft_, fp_ in filt):
                    switching = dphi < 0 and alpha * (-dphi) ** 2.3 > theta ** 1.1 and theta <= th_min
                    if switching:
                        ok = phit <= phi + 1e-4 * alpha * dphi
                    else:
                        ok = tht <= (1 - 1e-5) * theta or phit <= phi - 1e-5 * theta
                    if ok:
                        if not (switching and phit <= phi + 1e-4 * alpha * dphi):
                            filt.append(((1 - 1e-5) * theta, phi - 1e-5 * theta))
                        accepted = True
                        break
                alpha *= 0.5
            if not accepted:
                status = "line search failed"
                break
            w = wt
            f, g, c, p_ref = ft, gt, ct, pref_t
            theta = tht
            lam = lam + alpha * plam
            y = y + alpha * py
            zl = zl + a_z * pzl
            zu = zu + a_z * pzu
            # keep the bound multipliers near the primal-dual central path (Ipopt's κ_Σ = 1e10 safeguard)
            dl, du = self._slacks(w)
            zl = np.where(self.hasl, np.clip(zl, mu / (1e10 * dl), 1e10 * mu / dl), 0.0)
            zu = np.where(self.hasu, np.clip(zu, mu / (1e10 * du), 1e10 * mu / du), 0.0)
        u, x, s = w[:n_u], w[n_u:nz], w[nz:]
        v, th, pg = self._to_bus(u, x, p_g_ref=p_ref)
        return dict(status=status, iterations=len(hist) - 1, objective=f, v=v, theta=th, p_g=pg, p_ref=p_ref,
                    lam=lam, y=y, s=s, z_l=zl, z_u=zu, history=hist)

    def close(self):
        self.h.close()
