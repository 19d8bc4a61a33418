"""Small seeded test networks (built only from synth/, no method arithmetic)."""
import numpy as np

from synth import case9, make_grid
from synth.grid import pi_model


def two_bus():
    """lossless line x = 0.1 between ref/gen bus 0 and PQ bus 1."""
    Yff, Yft, Ytf, Ytt = pi_model(np.array([0.0]), np.array([0.1]), np.array([0.0]),
                                  np.array([1.0]), np.array([0.0]))
    net = dict(n_b=2, n_l=1, n_g=1, line_from=np.array([0], np.int32), line_to=np.array([1], np.int32),
               Y_ff=Yff, Y_ft=Yft, Y_tf=Ytf, Y_tt=Ytt, Y_sh=np.zeros(2, complex),
               gen_bus=np.array([0], np.int32), ref_bus=0,
               p_d=np.array([0.0, 0.5]), q_d=np.array([0.0, 0.0]), F_max=np.array([5.0]),
               c_quad=np.array([1000.0]), c_lin=np.array([2000.0]), seed=2)
    point = dict(v=np.array([1.0, 1.0]), theta=np.zeros(2), p_g=np.array([0.0]), q_g=np.array([0.0]),
                 p_d=net["p_d"].copy(), q_d=net["q_d"].copy())
    return net, point


def rich_small(seed=5, n_b=8, n_l=13, n_g=3):
    """A small grid that exercises every line type: transformers (tap), a
    phase shifter (Y_ft ≠ Y_tf), a parallel line and bus shunts."""
    net, point = make_grid(n_b, n_l, n_g, seed, parallel_frac=0.08, tr_frac=0.3,
                           ps_frac=0.5, shunt_frac=0.5)
    assert np.any(np.abs(net["Y_ft"] - net["Y_tf"]) > 1e-9), "needs a phase shifter"
    pairs = set()
    par = False
    for f, t in zip(net["line_from"], net["line_to"]):
        k = (min(f, t), max(f, t))
        par |= k in pairs
        pairs.add(k)
    assert par, "needs a parallel line"
    return net, point


def all_small():
    n9, p9 = case9()
    from synth.case9 import case9_multipliers
    p9.update(case9_multipliers())
    return [("case9", n9, p9), ("rich8", *rich_small())]
