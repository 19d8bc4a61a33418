import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2203_11875_b200 as pkg
from oracle import pf_oracle as O
from synth.grid import make_grid
for nb, nl, ng in [(12000, 16400, 1150), (13600, 18600, 1300)]:
    net, pt = make_grid(nb, nl, ng, 21)
    part = O.partition(net)
    p, q = O.injections(net, pt["v"], pt["theta"])
    gb = net["gen_bus"]
    star = dict(pt, p_d=np.where(part["is_gen"], 0.0, -p), q_d=np.where(part["is_gen"], 0.0, -q), p_g=p[gb].copy(), q_g=q[gb].copy())
    d = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float64)[None].copy(), device="cuda")
    for eps in (0.0, 1e-4, 1e-3, 1e-2):
        rng = np.random.default_rng(5)
        h = pkg.Network(net, max_batch=1, max_scen=1)
        v0 = d(np.where(part["is_gen"], star["v"], star["v"] + eps * rng.standard_normal(nb)))
        th0 = d(star["theta"] + 2 * eps * rng.standard_normal(nb) * (np.arange(nb) != net["ref_bus"]))
        it, res, info = h.pf_power_flow(1, v0, th0, d(star["p_g"]), d(star["q_g"]), d(star["p_d"]), d(star["q_d"]), tol=1e-10, max_iter=20)
        print(nb, part["n_x"], eps, it, res, info, flush=True)
        h.close()
