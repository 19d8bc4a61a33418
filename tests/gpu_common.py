"""Shared helpers of the GPU parity tests: stack seeded scenarios on the
device, compute the matching oracle quantities, the per-column K̂ gates of
R20 and the parity records written to $PF_PARITY_OUT (JSON lines)."""
import json
import os

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import pf_oracle as O


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def stack(points, key):
    return np.stack([np.asarray(p[key], dtype=np.float64) for p in points])


def dev(a, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or torch.float64, device="cuda")


def csr_dense(ptr, idx, val, shape):
    rows = np.repeat(np.arange(shape[0]), np.diff(ptr))
    D = np.zeros(shape)
    np.add.at(D, (rows, idx), val)
    return D


def oracle_khat(net, pt):
    part = O.partition(net)
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
    return O.reduce_naive(K, Gx, Gu), part


# ---------------------------------------------------------------- R20 per-column gates
TOL = 1e-10      # BASELINE.json north_star: relative 1e-10 in FP64
FLOOR_MULT = 3.0  # a column's gate: max(1e-10, FLOOR_MULT × the largest per-column route discrepancy)


def col_errs(got_cols, ref):
    """Per-column normwise error ‖a_j − b_j‖∞ / ‖b_j‖∞ (R20).  got_cols[j] is
    column j (the KV slab layout), ref is the matrix (columns = axis 1)."""
    a = np.asarray(got_cols, dtype=np.float64).T
    b = np.asarray(ref, dtype=np.float64)
    den = np.abs(b).max(axis=0)
    den[den == 0] = 1.0
    return np.abs(a - b).max(axis=0) / den


def oracle_routes(net, pt, cols=None):
    """Oracle routes of K̂ (columns `cols`, default all), three independent LU codes:
      naive  — O7, the naive sensitivity route, SuperLU COLAMD + partial pivoting;
      mmd    — O7′, the 3-step adjoint route, SuperLU minimum degree on AᵀA+A, diagonal pivots;
      static — O7′ with the R18 static-pivot LU (the bus-level minimum-degree
               ordering, no numerical pivoting): the algorithm the GPU runs;
      lapack — O7′ with a dense LAPACK LU (partial pivoting), where n_x ≤ 6000.
    floor[j] = the largest per-column discrepancy of the other routes from
    naive: how far correct implementations land apart on column j (R20;
    κ(G_x)·ε-level — up to ~3e-10 per column at 1354/2869 while the
    whole-matrix discrepancy stays ≤ 1e-12).  Returns (naive, static, floor, G_x)."""
    import scipy.linalg as sl
    part = O.partition(net)
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
    n_u, n_x = part["n_u"], part["n_x"]
    cols = np.arange(n_u) if cols is None else np.asarray(cols)
    naive = O.reduce_naive(K, Gx, Gu)[:, cols]
    perm, _ = O.permutation(part, O.md_ordering(net, part))
    static = O.reduce_columns(K, Gx, Gu, cols, kind="static", perm=perm)
    floor = np.maximum(col_errs(O.reduce_columns(K, Gx, Gu, cols, kind="mmd").T, naive), col_errs(static.T, naive))
    if n_x <= 6000:
        lu = sl.lu_factor(Gx.toarray())
        V = np.zeros((n_u, len(cols)))
        V[cols, np.arange(len(cols))] = 1.0
        Gud = Gu.toarray()
        H = K @ np.vstack([V, -sl.lu_solve(lu, Gud @ V)])
        lap = H[:n_u] - Gud.T @ sl.lu_solve(lu, H[n_u:], trans=1)
        floor = np.maximum(floor, col_errs(lap.T, naive))
    return naive, static, floor, Gx


def column_gates(floor):
    """Every column's gate: max(1e-10, FLOOR_MULT × max_j floor_j).  A per-column
    floor is one sample of the route-to-route scatter, not a bound for another
    implementation (the GPU also rounds K·d differently: per-line blocks vs
    the oracle's Y_bus-entry grouping), so the gate uses the matrix-wide
    largest measured scatter, applied to each column's own relative error."""
    return np.full(floor.shape, max(TOL, FLOOR_MULT * float(floor.max())))


def check_columns(got_cols, naive, floor, what="", static=None):
    """Assert the per-column gates against the naive oracle and (when given)
    the oracle running the same algorithm (R18 static pivots); return the
    summary for the parity record."""
    e = col_errs(got_cols, naive)
    tol = column_gates(floor)
    bad = np.nonzero(e > tol)[0]
    assert len(bad) == 0, "%s: %d columns over the gate %.3g, worst col %d err %.3g (floor max %.3g)" % (
        what, len(bad), tol[0], bad[np.argmax(e[bad])], e[bad].max(), floor.max())
    out = {"cols": int(len(e)), "gate": float(tol[0]), "col_err_max": float(e.max()),
           "col_err_median": float(np.median(e)), "col_err_p99": float(np.quantile(e, 0.99)),
           "cols_err_gt_1e-10": int((e > TOL).sum()), "floor_max": float(floor.max()),
           "floor_median": float(np.median(floor)), "cols_floor_gt_1e-10": int((floor > TOL).sum())}
    if static is not None:
        es = col_errs(got_cols, static)
        assert np.all(es <= tol), "%s: vs the static-pivot oracle route, col %d err %.3g gate %.3g" % (
            what, np.argmax(es), es.max(), tol[0])
        out.update({"vs_static_route_col_err_max": float(es.max()),
                    "vs_static_route_col_err_median": float(np.median(es))})
    return out


def cond1_sparse(A):
    """cond₁(A) with Hager/Higham's 1-norm estimate of ‖A⁻¹‖₁ (SuperLU solves)."""
    A = sp.csc_matrix(A)
    lu = spla.splu(A)
    n = A.shape[0]
    op = spla.LinearOperator((n, n), matvec=lambda x: lu.solve(np.asarray(x, dtype=np.float64).ravel()),
                             rmatvec=lambda x: lu.solve(np.asarray(x, dtype=np.float64).ravel(), trans="T"),
                             dtype=np.float64)
    return float(spla.norm(A, 1) * spla.onenormest(op))


def cond2_spd(M):
    w = np.linalg.eigvalsh(0.5 * (M + M.T))
    return float(w[-1] / w[0]) if w[0] > 0 else float("inf")


def record(name, **kw):
    """Append one parity record (JSON line) to $PF_PARITY_OUT."""
    path = os.environ.get("PF_PARITY_OUT", os.path.join(os.path.dirname(os.path.dirname(__file__)),
                                                        "gpurun_out", "parity_r02.jsonl"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps(dict(test=name, **kw)) + "\n")
