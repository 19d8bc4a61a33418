"""Summarise a tools/chol_bench.cu task trace: span, busy fraction, per-kind
durations, and the diagonal-task chain (the DAG's critical path)."""
import collections
import sys

import numpy as np

rows = [l.strip().split(",") for l in open(sys.argv[1]).readlines()[1:]]
a = np.array([[float(x) for x in r] for r in rows], dtype=np.float64)
tk, kind, s, i, j, sm, t0, t1, m0, m1, m2, m3 = a.T
T0 = t0.min()
mk = [np.where((m >= t0) & (m <= t1), (m - T0) / 1e3, np.nan) for m in (m0, m1, m2, m3)]
t0, t1 = (t0 - T0) / 1e3, (t1 - T0) / 1e3  # µs
span = t1.max()
nsm = len(set(sm))
print("tasks %d  span %.1f us  SMs %d  busy %.1f%% of (CTAs=%d x span)" % (
    len(a), span, nsm, 100 * (t1 - t0).sum() / (span * len(set(zip(sm))) * 2), 2 * nsm))
names = {1: "tile", 2: "fwd", 3: "bwd"}
for k in (1, 2, 3):
    m = kind == k
    if m.any():
        d = t1[m] - t0[m]
        print("%-5s n=%5d  mean %7.2f us  max %7.2f  sum %9.1f us  last end %.1f" % (names[k], m.sum(), d.mean(),
              d.max(), d.sum(), t1[m].max()))
m = (kind == 1) & (i == j)
print("diag tiles: mean %.2f us" % (t1[m] - t0[m]).mean())
for lab, mm in (("diag", m), ("offdiag", (kind == 1) & (i > j))):
    ph = [np.nanmean(mk[0][mm] - t0[mm]), np.nanmean(mk[1][mm] - mk[0][mm]), np.nanmean(mk[2][mm] - mk[1][mm]),
          np.nanmean(mk[3][mm] - mk[2][mm]), np.nanmean(t1[mm] - mk[3][mm])]
    print("  %-8s phases (us): gemm %.2f | epilogue %.2f | tri %.2f | write %.2f | release %.2f" % (lab, *ph))
m1 = (kind == 1) & (i == j + 1)
print("subdiag tiles: mean %.2f us" % (t1[m1] - t0[m1]).mean())
# chain of scenario 0: diag(j) end -> diag(j+1) end
for sc in (0,):
    de = {int(jj): (t0v, t1v) for jj, t0v, t1v in zip(j[m & (s == sc)], t0[m & (s == sc)], t1[m & (s == sc)])}
    se = {int(jj): (t0v, t1v) for jj, t0v, t1v in zip(j[m1 & (s == sc)], t0[m1 & (s == sc)], t1[m1 & (s == sc)])}
    print("scenario %d: j, diag start/end, subdiag start/end (us)" % sc)
    for jj in sorted(de)[:: max(1, len(de) // 12)]:
        print("  %3d  %8.1f %8.1f   %s" % (jj, de[jj][0], de[jj][1], "%8.1f %8.1f" % se[jj] if jj in se else ""))
# utilisation over time (fraction of CTA slots busy) in 10 bins
bins = np.linspace(0, span, 11)
occ = []
for b0, b1 in zip(bins[:-1], bins[1:]):
    ov = np.clip(np.minimum(t1, b1) - np.maximum(t0, b0), 0, None).sum()
    occ.append(ov / ((b1 - b0) * 2 * nsm))
print("busy by decile:", " ".join("%.2f" % o for o in occ))
