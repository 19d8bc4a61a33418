"""LinRed IPM (NEXT-4, Algorithm 1) on the Table-1-shaped synthetic grids: iterations, status and
wall time per iteration (host loop over the C-ABI).  python tools/ipm_scale.py case1354 case2869 case9241"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_11875_b200 import _build  # noqa: E402

_build.build()
from paper_2203_11875_b200.ipm import LinRedIPM  # noqa: E402
from synth.grid import opf_bounds, opf_feasible, table1_grid  # noqa: E402
from synth.grid import pi_model  # noqa: E402,F401

for name in sys.argv[1:]:
    net, pt = table1_grid(name)
    b = opf_bounds(net)
    if os.environ.get("IPM_FEASIBLE", "1") == "1":
        # loosen the limits the synthetic point violates (flows |s| at both ends from the π model)
        V = pt["v"] * np.exp(1j * pt["theta"])
        f, t = net["line_from"], net["line_to"]
        i_f = net["Y_ff"] * V[f] + net["Y_ft"] * V[t]
        i_t = net["Y_tf"] * V[f] + net["Y_tt"] * V[t]
        pt = dict(pt, s_abs=np.maximum(np.abs(V[f] * np.conj(i_f)), np.abs(V[t] * np.conj(i_t))))
        net, b = opf_feasible(net, pt)
    s = LinRedIPM(net, b, tol=1e-8, max_iter=int(os.environ.get("IPM_MAX_ITER", 300)))
    t0 = time.perf_counter()
    # start: the grid's synthetic operating point (power-flow feasible), or a flat start
    res = s.solve() if os.environ.get("IPM_FLAT") else s.solve(v0=pt["v"], theta0=pt["theta"], p_g0=pt["p_g"])
    dt = time.perf_counter() - t0
    s.close()
    rec = {"case": name, "status": res["status"], "iterations": res["iterations"], "objective": res["objective"],
           "wall_s": dt, "ms_per_iteration": 1e3 * dt / max(1, res["iterations"]),
           "delta_w_max": max(h["delta_w"] for h in res["history"])}
    print(json.dumps(rec), flush=True)
