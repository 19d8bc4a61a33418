import sys, os
sys.path.insert(0, "/root/repo")
from paper_2203_11875_b200.ipm import LinRedIPM
from synth.grid import opf_bounds, table1_grid
net, _ = table1_grid(sys.argv[1])
s = LinRedIPM(net, opf_bounds(net), tol=1e-8, max_iter=300)
res = s.solve()
for h in res["history"][-8:]: print(h)
print(res["status"])
