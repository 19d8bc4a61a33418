"""Per-phase timing of the k_fwd / k_adj sweeps of CTA (0, 0) (debug build with
-DPF_SWEEP_TRACE; run on a GPU box): python tools/sweep_trace.py build/libpf_swtrace.so [grid] [scenarios]
Slots: 0 = k_fwd L (reach), 1 = k_fwd U, 2 = k_adj Uᵀ, 3 = k_adj Lᵀ (ancestors)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PF_LIB"] = sys.argv[1]
import torch  # noqa: E402

import paper_2203_11875_b200 as pkg  # noqa: E402
from synth import make_scenario  # noqa: E402
from synth.grid import table1_grid  # noqa: E402

grid = sys.argv[2] if len(sys.argv) > 2 else "case9241"
S = int(sys.argv[3]) if len(sys.argv) > 3 else 8
net, pt = table1_grid(grid)
pts = [pt] + [make_scenario(net, pt, s) for s in range(1, S)]
from oracle import pf_oracle as O  # noqa: E402  (only for n_u)
n_u = O.partition(net)["n_u"]
h = pkg.Network(net, max_batch=n_u, max_scen=S)
lib = pkg.load_library()
tr = torch.zeros(4 * 512, dtype=torch.int64, device="cuda")
lib.pf_debug_set_sweep_trace(ctypes.c_void_p(tr.data_ptr()))
dev = lambda k: torch.as_tensor(np.stack([p[k] for p in pts]), device="cuda")  # noqa: E731
v, th = dev("v"), dev("theta")
h.pf_jacobian(S, v, th)
KV = torch.empty(S, n_u, n_u, dtype=torch.float64, device="cuda")
for _ in range(3):
    h.pf_reduced_hessian_batch(S, v, th, dev("lam"), dev("y"), KV, sigma_s=dev("sigma_s"), sigma_x=dev("sigma_x"),
                               N=n_u, p_d=dev("p_d"))
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.float64).reshape(4, 512)
names = ["k_fwd L(reach)", "k_fwd U", "k_adj U^T", "k_adj L^T(anc)"]
for k in range(4):
    r = t[k]
    t0 = r[0]
    if t0 == 0:
        continue
    tot = (r[511] - t0) / 1e3
    bot = [(r[1 + i] - t0) / 1e3 for i in range(8) if r[1 + i] > 0]
    levs = [(i, (r[64 + i])) for i in range(128) if r[64 + i] > 0]
    print("%-16s total %8.1f us" % (names[k], tot))
    if bot:
        print("   team bottom-phase end (us from sweep start, UPPER: from the top phase's end too):",
              " ".join("%.0f" % b for b in bot))
    if levs:
        prev = t0 if k in (1, 3) else max(r[1:9].max(), t0)
        d = []
        for i, x in levs:
            d.append((i, (x - prev) / 1e3))
            prev = x
        print("   levels: %d, sum %.1f us; per level: %s" % (len(d), sum(x for _, x in d),
              " ".join("%d:%.1f" % (i, x) for i, x in d)))
