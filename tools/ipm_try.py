import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2203_11875_b200 import _build; _build.build()
from paper_2203_11875_b200.ipm import LinRedIPM
from synth import case9
from synth.case9 import case9_bounds
net, pt = case9()
b, c0 = case9_bounds()
ipm = LinRedIPM(net, b, verbose=True, max_iter=100)
res = ipm.solve(v0=pt["v"], p_g0=pt["p_g"])
print(res["status"], res["iterations"], res["objective"] + c0, res["p_g"] * 100, res["p_ref"] * 100)
