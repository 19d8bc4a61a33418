"""Per-level k_lu timing (debug build with -DPF_LU_TRACE; run on a GPU box):
python tools/lu_trace.py build/libpf_lutrace.so [grid] [scenarios]"""
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
h = pkg.Network(net, max_batch=64, max_scen=S)
lib = pkg.load_library()
nlev = h.dims["n_levels_l"]
tr = torch.zeros(1024 + 8 * (nlev + 2), dtype=torch.int64, device="cuda")
lib.pf_debug_set_lu_trace(ctypes.c_void_p(tr.data_ptr()))
dev = lambda k: torch.as_tensor(np.stack([p[k] for p in pts]), device="cuda")  # noqa: E731
v, th = dev("v"), dev("theta")
for _ in range(3):
    h.pf_jacobian(S, v, th)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.float64)
dt = np.diff(t[: nlev + 1]) / 1e3
lp = np.asarray(h.structure("level_l_ptr"))
cnt = np.diff(lp)
ph = t[1024:1024 + 8 * nlev].reshape(nlev, 8)
print("CTA 0 warp 0, per level: load | stage | chain | store+pair | done -> cluster.sync done (us)")
for l in range(0, nlev, 3):
    r = ph[l]
    if r[0] > 0 and t[l + 1] > 0:
        d = lambda a, b: (r[b] - r[a]) / 1e3 if r[a] > 0 and r[b] > 0 else float("nan")
        print("  lev %3d  %6.2f %6.2f %6.2f %6.2f  sync %6.2f" % (l, d(0, 1), d(1, 2), d(2, 3) if r[2] > 0 else d(1, 3), d(3, 4), (t[l + 1] - r[5]) / 1e3 if r[5] > 0 else float("nan")))
print("k_lu levels: total %.1f us over %d levels" % (dt.sum(), nlev))
order = np.argsort(-dt)[:15]
for l in sorted(order):
    print("  level %3d  blocks %5d  %8.1f us" % (l, cnt[l], dt[l]))
big = cnt >= 64
print("wide levels (>=64 blocks): %d, %.1f us; narrow: %d, %.1f us" % (big.sum(), dt[big].sum(), (~big).sum(), dt[~big].sum()))
