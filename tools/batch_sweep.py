"""Batch-size sweep of the reduced-Hessian assembly (the Fig. 2b
pattern of P:L1306–1313): the full K̂ of one scenario assembled in ⌈n_u/N⌉
calls of pf_reduced_hessian_batch with N directions each, CUDA-event timed
(L2 flushed before each assembly).  Prints one JSON object.
    python tools/batch_sweep.py [grid ...]"""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11875_b200 as pkg  # noqa: E402
from synth.grid import table1_grid  # noqa: E402

grids = sys.argv[1:] or ["case118", "case1354"]
out = {"what": "full K̂ of one scenario in ceil(n_u/N) calls; HVP/s = n_u / time", "results": {}}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for g in grids:
    net, pt = table1_grid(g)
    tmp = pkg.Network(net, max_batch=1, max_scen=1, device=-1)
    n_u = tmp.dims["n_u"]
    tmp.close()
    dev = lambda k: torch.as_tensor(np.asarray(pt[k], dtype=np.float64)[None], device="cuda")  # noqa: E731
    res = {}
    for N in sorted({1, 8, 32, 64, 128, 256, n_u}):
        if N > n_u:
            continue
        h = pkg.Network(net, max_batch=N, max_scen=1)
        v, th = dev("v"), dev("theta")
        h.pf_jacobian(1, v, th)
        KV = torch.empty(1, N, n_u, dtype=torch.float64, device="cuda")
        args = dict(sigma_s=dev("sigma_s"), sigma_x=dev("sigma_x"), p_d=dev("p_d"))
        lam, y = dev("lam"), dev("y")

        def assemble():
            for c0 in range(0, n_u, N):
                nn = min(N, n_u - c0)
                h.pf_reduced_hessian_batch(1, v, th, lam, y, KV[:, :nn], col0=c0, N=nn, **args)

        assemble()
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assemble()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        res[str(N)] = {"ms": ms, "calls": -(-n_u // N), "hvp_per_s": n_u / (ms / 1e3), "tile_cols": h.dims["tile_cols"]}
        h.close()
    out["results"][g] = {"n_u": n_u, "by_N": res}
print(json.dumps(out))
