"""MATPOWER case9 (WSCC 9-bus), hand-embedded.

The reference ships no case files; BASELINE.json configs[0]
asks for a hand-embedded case9.  Data recalled from MATPOWER's public
``case9.m``; pinned in tests by the textbook power-flow
solution.  Zero-based bus numbering; bus 0 is the reference.
"""
import numpy as np

from .grid import pi_model, counts

BASE_MVA = 100.0
# from, to, r, x, b, rateA (MW)
_BRANCH = [
    (1, 4, 0.0, 0.0576, 0.0, 250),
    (4, 5, 0.017, 0.092, 0.158, 250),
    (5, 6, 0.039, 0.17, 0.358, 150),
    (3, 6, 0.0, 0.0586, 0.0, 300),
    (6, 7, 0.0119, 0.1008, 0.209, 150),
    (7, 8, 0.0085, 0.072, 0.149, 250),
    (8, 2, 0.0, 0.0625, 0.0, 250),
    (8, 9, 0.032, 0.161, 0.306, 250),
    (9, 4, 0.01, 0.085, 0.176, 250),
]
# bus, Pg (MW), Vg, c2 ($/MW^2h), c1 ($/MWh)
_GEN = [
    (1, 72.3, 1.04, 0.11, 5.0),
    (2, 163.0, 1.025, 0.085, 1.2),
    (3, 85.0, 1.025, 0.1225, 1.0),
]
# OPF data of case9.m: Pmin, Pmax, Qmin, Qmax (MW, MVAr), constant cost c0 ($/h); Vmin, Vmax
_GEN_LIM = [(10.0, 250.0, -300.0, 300.0, 150.0), (10.0, 300.0, -300.0, 300.0, 600.0),
            (10.0, 270.0, -300.0, 300.0, 335.0)]
_VLIM = (0.9, 1.1)
_LOAD = {5: (90.0, 30.0), 7: (100.0, 35.0), 9: (125.0, 50.0)}


def case9():
    """Return (net, point0): the network in the ABI's input contract and the
    case-file starting point (Vg at generator buses, flat elsewhere)."""
    br = np.array(_BRANCH, dtype=np.float64)
    lf = (br[:, 0] - 1).astype(np.int32)
    lt = (br[:, 1] - 1).astype(np.int32)
    n_l = len(br)
    Yff, Yft, Ytf, Ytt = pi_model(br[:, 2], br[:, 3], br[:, 4], np.ones(n_l), np.zeros(n_l))
    n_b = 9
    gen_bus = np.array([g[0] - 1 for g in _GEN], dtype=np.int32)
    p_d = np.zeros(n_b)
    q_d = np.zeros(n_b)
    for bus, (p, q) in _LOAD.items():
        p_d[bus - 1] = p / BASE_MVA
        q_d[bus - 1] = q / BASE_MVA
    c_quad = np.array([g[3] for g in _GEN]) * BASE_MVA ** 2
    c_lin = np.array([g[4] for g in _GEN]) * BASE_MVA
    net = dict(n_b=n_b, n_l=n_l, n_g=3, line_from=lf, line_to=lt,
               Y_ff=Yff, Y_ft=Yft, Y_tf=Ytf, Y_tt=Ytt, Y_sh=np.zeros(n_b, dtype=np.complex128),
               gen_bus=gen_bus, ref_bus=0, p_d=p_d, q_d=q_d, F_max=br[:, 5] / BASE_MVA,
               c_quad=c_quad, c_lin=c_lin, seed=9)
    v = np.ones(n_b)
    v[gen_bus] = [g[2] for g in _GEN]
    point = dict(v=v, theta=np.zeros(n_b), p_g=np.array([g[1] for g in _GEN]) / BASE_MVA,
                 q_g=np.zeros(3), p_d=p_d.copy(), q_d=q_d.copy())
    return net, point


def case9_multipliers(seed=9):
    """IPM-like multipliers for case9 in the ABI layout (same rules as grid)."""
    from .grid import _multipliers
    net, _ = case9()
    cnt = counts(9, net["gen_bus"], net["F_max"])
    return _multipliers(np.random.default_rng(seed), 9, 3, cnt, 9)


def case9_bounds():
    """OPF bounds of MATPOWER case9 in p.u. (NEXT-4), and the constant cost
    Σ c0 = 1085 $/h the objective f omits (MATPOWER's optimum 5296.69 $/h
    includes it)."""
    lim = np.array(_GEN_LIM)
    b = dict(v_lo=np.full(9, _VLIM[0]), v_hi=np.full(9, _VLIM[1]),
             p_lo=lim[:, 0] / BASE_MVA, p_hi=lim[:, 1] / BASE_MVA,
             q_lo=lim[:, 2] / BASE_MVA, q_hi=lim[:, 3] / BASE_MVA)
    return b, float(lim[:, 4].sum())
