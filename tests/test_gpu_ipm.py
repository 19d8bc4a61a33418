"""NEXT-4 — the LinRed IPM driver (Algorithm 1 with a filter line search,
paper_2203_11875_b200/ipm.py) end to end on the device.

* case9 (MATPOWER data, hand-embedded): the optimum is the published
  MATPOWER/WSCC OPF solution, 5296.69 $/h with P_g = (89.80, 134.32, 94.19) MW
  (external values, not from this code base), reached at the paper's 1e-8
  tolerance;
* case118-shaped synthetic grid (seeded bounds, synth.grid.opf_bounds): no
  published optimum, so the converged point is pinned by the ORACLE's
  first-order conditions — its independent Jacobians, objective gradient
  (implicit p_ref, R8) and power-flow residual — ∇f + G_zᵀλ + A_zᵀy − z_L + z_U
  = 0, g = 0, c(x,u) = s, bounds and complementarity."""
import numpy as np
import pytest

from oracle import pf_oracle as O
from synth import case9
from synth.case9 import case9_bounds
from synth.grid import opf_bounds, table1_grid
from tests import golden_data
from tests.gpu_common import record

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ipm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2203_11875_b200 import _build
    _build.build()
    from paper_2203_11875_b200 import ipm as m
    return m


def _oracle_kkt(net, res, solver):
    """First-order optimality of the returned point by the oracle's derivatives."""
    part = O.partition(net)
    pt = dict(v=res["v"], theta=res["theta"], p_g=res["p_g"], q_g=np.zeros(net["n_g"]),
              p_d=np.asarray(net["p_d"]), q_d=np.asarray(net["q_d"]))
    Gx, Gu, A = O.jacobians(net, part, pt)
    grad = O.objective_gradient(net, part, pt)
    n_u, n_x = part["n_u"], part["n_x"]
    lam, y = res["lam"], res["y"]
    dual = grad + np.concatenate([Gu.T @ lam, Gx.T @ lam]) + A.T @ y - res["z_l"][:n_u + n_x] + res["z_u"][:n_u + n_x]
    g = O.g_residual(net, part, pt)
    _, H, _ = O.constraints(net, pt)
    p, q = O.injections(net, pt["v"], pt["theta"])
    r = np.array([p[i] if t == 0 else q[i] for (i, t) in part["r_rows"]])
    h = np.array([H[l] if e == 0 else H[net["n_l"] + l] for (l, e) in part["h_rows"]])
    cs = np.concatenate([r, h]) - res["s"]
    w = np.concatenate([np.zeros(n_u + n_x), res["s"]])
    scale = max(1.0, np.abs(grad).max())
    return dict(dual=float(np.abs(dual).max() / scale), g=float(np.abs(g).max()), c_minus_s=float(np.abs(cs).max()))


def test_ipm_case9_matpower_optimum(ipm):
    net, pt = case9()
    b, c0 = case9_bounds()
    s = ipm.LinRedIPM(net, b, tol=1e-8)
    res = s.solve(v0=pt["v"], p_g0=pt["p_g"])
    s.close()
    assert res["status"] == "converged", res["status"]
    g = golden_data.keyed("case9_opf.txt")
    assert abs(res["objective"] + c0 - g["objective_usd_per_h"][0]) <= 0.01, res["objective"] + c0
    assert np.allclose(res["p_g"] * 100, g["p_g_mw"], atol=0.01), res["p_g"] * 100
    k = _oracle_kkt(net, res, s)
    assert k["dual"] <= 1e-7 and k["g"] <= 1e-9 and k["c_minus_s"] <= 1e-9, k
    record("ipm", case="case9", iterations=res["iterations"], objective=res["objective"] + c0, **k,
           delta_w=[h["delta_w"] for h in res["history"]])


def test_ipm_case118_synthetic_kkt(ipm):
    net, pt = table1_grid("case118")
    b = opf_bounds(net)
    s = ipm.LinRedIPM(net, b, tol=1e-8, max_iter=150)
    res = s.solve()
    s.close()
    assert res["status"] == "converged", (res["status"], res["history"][-3:])
    k = _oracle_kkt(net, res, s)
    assert k["dual"] <= 1e-7 and k["g"] <= 1e-9 and k["c_minus_s"] <= 1e-9, k
    lo, up = s.lo, s.up
    w = np.concatenate([np.zeros(s.n_u + s.n_x), res["s"]])
    assert np.all(res["v"] >= 0.9 - 1e-9) and np.all(res["v"] <= 1.1 + 1e-9)
    record("ipm", case="case118", iterations=res["iterations"], objective=res["objective"], **k)
