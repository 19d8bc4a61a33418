"""Debug helper: case9 K̂ parity for each tile width (run on the GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import pf_oracle as O
from synth import case9
from synth.case9 import case9_multipliers
import paper_2203_11875_b200 as pkg

net, pt = case9()
part = O.partition(net)
pt, _, _ = O.newton(net, part, pt)
pt.update(case9_multipliers())
Gx, Gu, A = O.jacobians(net, part, pt)
K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
Kh = O.reduce_naive(K, Gx, Gu)
dev = lambda a: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)[None]), device="cuda")  # noqa
h = pkg.Network(net, max_batch=5, max_scen=1)
print("tile_cols", h.dims["tile_cols"])
v, th = dev(pt["v"]), dev(pt["theta"])
h.pf_jacobian(1, v, th)
KV = torch.empty(1, 5, 5, dtype=torch.float64, device="cuda")
h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"]), dev(pt["y"]), KV, sigma_s=dev(pt["sigma_s"]),
                           sigma_x=dev(pt["sigma_x"]), N=5, p_d=dev(pt["p_d"]))
torch.cuda.synchronize()
G = KV[0].cpu().numpy().T
print("rel err", np.abs(G - Kh).max() / np.abs(Kh).max())
