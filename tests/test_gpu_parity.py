"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle,
element by element on the same seeded inputs.

Tolerances (R20, BASELINE.json north_star "relative 1e-10 in FP64"):
* G, H, s, G_x, G_u, A, the Cholesky factor and solves: normwise per output
  array, max|a−b| / max|b| ≤ 1e-10;
* K̂: per COLUMN, ‖a_j − b_j‖∞/‖b_j‖∞ ≤ max(1e-10, 3 × the largest per-column
  scatter among correct oracle routes with independent LU codes) — O7 (SuperLU
  COLAMD + partial pivoting) vs O7′ with minimum-degree diagonal pivots, with
  the R18 static-pivot LU (the GPU's algorithm) and with dense LAPACK
  (tests/gpu_common.oracle_routes / column_gates) — against both O7 and the
  R18 route; every column's error goes into the parity record;
* bit-exact for integer outputs (info) and for batch / tile / partition
  invariance.
Every K̂ check appends its per-column statistics, cond₁(G_x) and cond(K_cond)
to $PF_PARITY_OUT (profiles/r02_parity.jsonl is a copy)."""
import os

import numpy as np
import pytest

from oracle import pf_oracle as O
from synth import case9, make_grid, make_scenario
from synth.case9 import case9_multipliers
from synth.grid import TABLE1, table1_grid
from tests.gpu_common import (TOL, check_columns, col_errs, cond1_sparse, cond2_spd, csr_dense, dev,
                              oracle_khat, oracle_routes, record, rel_err, stack)
from tests.nets import rich_small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pfmod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2203_11875_b200 import _build
    _build.build()
    import paper_2203_11875_b200 as m
    return m


def _case9_point():
    net, pt = case9()
    part = O.partition(net)
    pt, _, _ = O.newton(net, part, pt)      # case9 at its textbook operating point
    pt.update(case9_multipliers())
    return net, pt


def _nolimit_grid():
    """case118-shaped grid with 30% of the lines unlimited (F_max = 0: no h rows, R23)."""
    n_b, n_l, n_g = TABLE1["case118"]
    net, pt = make_grid(n_b, n_l, n_g, 118, nolimit_frac=0.3)
    assert (net["F_max"] <= 0).sum() > 10
    return net, pt


def _cases(names):
    out = []
    for name in names:
        if name == "case9":
            net, pt = _case9_point()
            pts = [pt]
        elif name == "rich8":
            net, pt = rich_small()
            pts = [pt]
        elif name == "nolimit118":
            net, pt = _nolimit_grid()
            pts = [pt, make_scenario(net, pt, 1)]
        else:
            net, pt = table1_grid(name)
            pts = [pt, make_scenario(net, pt, 1)]
        out.append((name, net, pts))
    return out


MEDIUM = ["case9", "rich8", "case118", "nolimit118", "case1354"]


@pytest.mark.parametrize("name,net,pts", _cases(MEDIUM))
def test_eval_constraints(pfmod, name, net, pts):
    import torch
    S = len(pts)
    h = pfmod.Network(net, max_batch=8, max_scen=S)
    G = torch.empty(S, 2 * net["n_b"], dtype=torch.float64, device="cuda")
    H = torch.empty(S, 2 * net["n_l"], dtype=torch.float64, device="cuda")
    sf = torch.empty(S, 4, net["n_l"], dtype=torch.float64, device="cuda")
    h.pf_eval_constraints(S, dev(stack(pts, "v")), dev(stack(pts, "theta")), dev(stack(pts, "p_g")),
                          dev(stack(pts, "q_g")), dev(stack(pts, "p_d")), dev(stack(pts, "q_d")), G, H, sf)
    torch.cuda.synchronize()
    for s, pt in enumerate(pts):
        Go, Ho, so = O.constraints(net, pt)
        assert rel_err(G[s].cpu().numpy(), Go) <= TOL
        assert rel_err(H[s].cpu().numpy(), Ho) <= TOL
        assert rel_err(sf[s].cpu().numpy(), so) <= TOL
    # NULL loads = the base loads given at build time
    G2 = torch.empty_like(G)
    h.pf_eval_constraints(S, dev(stack(pts, "v")), dev(stack(pts, "theta")), dev(stack(pts, "p_g")),
                          dev(stack(pts, "q_g")), None, None, G2)
    pt0 = dict(pts[0], p_d=net["p_d"], q_d=net["q_d"])
    assert rel_err(G2[0].cpu().numpy(), O.constraints(net, pt0)[0]) <= TOL
    h.close()


@pytest.mark.parametrize("name,net,pts", _cases(MEDIUM))
def test_jacobian_values(pfmod, name, net, pts):
    import torch
    S = len(pts)
    h = pfmod.Network(net, max_batch=8, max_scen=S)
    d = h.dims
    part = O.partition(net)
    assert d["n_h"] == part["n_h"] and d["m"] == part["m"]
    Gx = torch.empty(S, d["nnz_gx"], dtype=torch.float64, device="cuda")
    Gu = torch.empty(S, d["nnz_gu"], dtype=torch.float64, device="cuda")
    A = torch.empty(S, d["nnz_a"], dtype=torch.float64, device="cuda")
    info = torch.full((S,), -7, dtype=torch.int32, device="cuda")
    h.pf_jacobian(S, dev(stack(pts, "v")), dev(stack(pts, "theta")), Gx, Gu, A, info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * S
    for s, pt in enumerate(pts):
        Gxo, Guo, Ao = O.jacobians(net, part, pt)
        gx = csr_dense(h.structure("gx_ptr"), h.structure("gx_idx"), Gx[s].cpu().numpy(), Gxo.shape)
        gu = csr_dense(h.structure("gu_ptr"), h.structure("gu_idx"), Gu[s].cpu().numpy(), Guo.shape)
        a = csr_dense(h.structure("a_ptr"), h.structure("a_idx"), A[s].cpu().numpy(), Ao.shape)
        assert rel_err(gx, Gxo.toarray()) <= TOL
        assert rel_err(gu, Guo.toarray()) <= TOL
        assert rel_err(a, Ao.toarray()) <= TOL
    h.close()


def _run_khat(pfmod, h, net, pts, N=None, col0=0, V=None, chunks=None):
    import torch
    S = len(pts)
    d = h.dims
    n_u = d["n_u"]
    v, th = dev(stack(pts, "v")), dev(stack(pts, "theta"))
    info = torch.empty(S, dtype=torch.int32, device="cuda")
    h.pf_jacobian(S, v, th, info=info)
    args = dict(sigma_s=dev(stack(pts, "sigma_s")), sigma_x=dev(stack(pts, "sigma_x")), p_d=dev(stack(pts, "p_d")))
    lam, y = dev(stack(pts, "lam")), dev(stack(pts, "y"))
    if chunks is None:
        N = n_u if N is None else N
        KV = torch.empty(S, N, n_u, dtype=torch.float64, device="cuda")
        h.pf_reduced_hessian_batch(S, v, th, lam, y, KV, V=V, col0=col0, N=N, **args)
        torch.cuda.synchronize()
        return KV.cpu().numpy(), info.cpu().numpy()
    out = np.zeros((S, n_u, n_u))
    for c0 in range(0, n_u, chunks):
        n = min(chunks, n_u - c0)
        KV = torch.empty(S, n, n_u, dtype=torch.float64, device="cuda")
        h.pf_reduced_hessian_batch(S, v, th, lam, y, KV, col0=c0, N=n, **args)
        out[:, c0:c0 + n] = KV.cpu().numpy()
    torch.cuda.synchronize()
    return out, info.cpu().numpy()


def _check_khat(name, KVs, net, pt, s=0, extra=None):
    """Per-column gates of K̂ (unsymmetrised and symmetrised, R21) + P12, and a
    parity record with the noise floor and cond₁(G_x)."""
    if os.environ.get("PF_DUMP_KHAT") and KVs.shape[0] <= 1100:   # gate studies (tools/)
        np.save(os.path.join(os.environ["PF_DUMP_KHAT"], "khat_%s_%d.npy" % (name, s)), KVs)
    naive, static, floor, Gx = oracle_routes(net, pt)
    st = check_columns(KVs, naive, floor, "%s scen %d" % (name, s), static)
    assert rel_err(KVs.T, naive) <= TOL, name
    sym = 0.5 * (KVs + KVs.T)
    assert rel_err(sym, 0.5 * (naive + naive.T)) <= TOL
    assert np.abs(KVs - KVs.T).max() <= 1e-12 * np.abs(KVs).max()   # P12
    st["whole_matrix_rel_err"] = float(rel_err(KVs.T, naive))
    st["cond1_Gx"] = cond1_sparse(Gx)
    record("khat", case=name, scenario=s, **st, **(extra or {}))
    return naive


@pytest.mark.parametrize("name,net,pts", _cases(MEDIUM))
def test_reduced_hessian_full(pfmod, name, net, pts):
    """Full K̂ (unit directions, one batch) vs the oracle, per column."""
    S = len(pts)
    part = O.partition(net)
    h = pfmod.Network(net, max_batch=part["n_u"], max_scen=S)
    KV, info = _run_khat(pfmod, h, net, pts)
    assert info.tolist() == [0] * S
    for s, pt in enumerate(pts):
        _check_khat(name, KV[s], net, pt, s, {"tile_cols": h.dims["tile_cols"]})
    h.close()


@pytest.mark.parametrize("name,net,pts", _cases(["rich8", "case118"]))
def test_reduced_hessian_dense_directions(pfmod, name, net, pts):
    """Generic HVPs: dense seeded V (A7.1 as a real SpMM), K̂V vs the oracle."""
    S = len(pts)
    part = O.partition(net)
    n_u = part["n_u"]
    N = min(13, n_u)
    rng = np.random.default_rng(7)
    Vs = rng.standard_normal((S, N, n_u))
    h = pfmod.Network(net, max_batch=N, max_scen=S)
    KV, _ = _run_khat(pfmod, h, net, pts, N=N, V=dev(Vs))
    for s, pt in enumerate(pts):
        Kh, _ = oracle_khat(net, pt)
        ref = Kh @ Vs[s].T
        assert rel_err(KV[s], ref.T) <= TOL
        assert col_errs(KV[s], ref).max() <= 1e-9
    h.close()


@pytest.mark.parametrize("name,net,pts", _cases(["case9", "case118"]))
def test_batch_invariance_bitwise(pfmod, name, net, pts):
    """Each column's arithmetic is independent of the batch: K̂ is
    bit-identical for N = n_u in one call and in chunks of 1, 3, 7."""
    part = O.partition(net)
    h = pfmod.Network(net, max_batch=part["n_u"], max_scen=len(pts))
    ref, _ = _run_khat(pfmod, h, net, pts)
    for ch in (1, 3, 7):
        out, _ = _run_khat(pfmod, h, net, pts, chunks=ch)
        assert np.array_equal(out, ref), ch
    h.close()


@pytest.mark.parametrize("name", ["case118", "case1354"])
def test_tile_width_invariance_bitwise(pfmod, name):
    """Every direction-tile width (8, 16, 32, 64 directions per CTA: teams of
    8/16/32 lanes, one or two directions per lane) runs the same arithmetic per
    direction, so K̂ is bit-identical across widths — for unit
    directions in aligned (sparse-RHS reach) and unaligned calls and for dense
    V — and matches the oracle per column; dense V is checked against the
    oracle at the bench's width 64."""
    net, pt = table1_grid(name)
    pts = [pt, make_scenario(net, pt, 1)]
    n_u = O.partition(net)["n_u"]
    outs = {}
    rng = np.random.default_rng(21)
    Vd = rng.standard_normal((len(pts), 70, n_u))
    for c in (8, 16, 32, 64):
        h = pfmod.Network(net, max_batch=n_u, max_scen=len(pts), tile_cols=c)
        assert h.dims["tile_cols"] == c
        full, _ = _run_khat(pfmod, h, net, pts)
        part, _ = _run_khat(pfmod, h, net, pts, N=70, col0=37)      # unaligned: full L sweep
        dense, _ = _run_khat(pfmod, h, net, pts, N=70, V=dev(Vd))  # dense directions
        outs[c] = (full, part, dense)
        h.close()
    for c in (16, 32, 64):
        for a, b in zip(outs[8], outs[c]):
            assert np.array_equal(a, b), c
    full = outs[64][0]
    assert np.array_equal(outs[64][1], full[:, 37:107])
    for s, p in enumerate(pts):
        naive = _check_khat(name, full[s], net, p, s, {"tile_cols": "8/16/32/64 (bitwise equal)"})
        ref = naive @ Vd[s].T
        assert rel_err(outs[64][2][s], ref.T) <= TOL
        e = col_errs(outs[64][2][s], ref)
        record("dense_V_C64", case=name, scenario=s, col_err_max=float(e.max()), col_err_median=float(np.median(e)))
        assert e.max() <= 1e-9


def test_direction_partition_emulated(pfmod):
    """bench.py's direction sharding (configs 3–4) for G ∈ {2, 4, 8}, run rank
    by rank on one GPU: each rank's tile-aligned slab (dist.column_partition)
    plus the all-gather's padding/concatenation (dist.assemble_columns) gives a
    K̂ bit-identical to the single call (§8(e) invariance)."""
    import torch
    from paper_2203_11875_b200.dist import assemble_columns, column_partition
    net, pt = table1_grid("case1354")
    pts = [pt]
    n_u = O.partition(net)["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=1, tile_cols=8)
    ref, _ = _run_khat(pfmod, h, net, pts)
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            col0, ncols, c = column_partition(n_u, G, r, h.dims["tile_cols"])
            slab = np.zeros((1, c, n_u))
            if ncols:
                slab[:, :ncols], _ = _run_khat(pfmod, h, net, pts, N=ncols, col0=col0)
            parts.append(torch.from_numpy(slab))
        full = assemble_columns(parts, n_u).numpy()
        assert np.array_equal(full, ref), G
    h.close()


def _kcond_delta(Khs, pts):
    lmins = [np.linalg.eigvalsh(Kh + np.diag(p["sigma_u"])).min() for Kh, p in zip(Khs, pts)]
    return max(0.0, -min(lmins)) * 1.5 + 1.0, lmins


@pytest.mark.parametrize("name", ["case118", "case1354"])
def test_condensed_kkt_solve(pfmod, name):
    """K_cond = sym(K̂) + diag(Σ_u) + δ_w I: L and the solve vs the oracle's
    textbook Cholesky; info for an indefinite shift equals the oracle's.
    case1354 (n_u = 519) exercises ragged tiles and deep tile-DAG chains."""
    import torch
    net, pt = table1_grid(name)
    pts = [pt, make_scenario(net, pt, 1)]
    S = 2
    part = O.partition(net)
    n_u = part["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    KV, _ = _run_khat(pfmod, h, net, pts)
    Khs = [0.5 * (KV[s] + KV[s].T) for s in range(S)]
    delta, lmins = _kcond_delta(Khs, pts)
    rng = np.random.default_rng(3)
    b = rng.standard_normal((S, 2, n_u))
    K = dev(KV.copy())
    rhs = dev(b.copy())
    info = torch.empty(S, dtype=torch.int32, device="cuda")
    h.pf_condensed_kkt_solve(S, K, dev(stack(pts, "sigma_u")), delta, rhs, 2, info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0, 0]
    Lg = K.cpu().numpy()
    for s in range(S):
        Kc = O.condensed(Khs[s], pts[s]["sigma_u"], delta)
        Lo, io = O.cholesky(Kc)
        assert io == 0
        L = Lg[s].T  # column-major → row-major
        assert np.array_equal(np.triu(L, 1), np.zeros_like(L))
        assert rel_err(L, Lo) <= TOL
        for r in range(2):
            po = O.chol_solve(Lo, b[s, r])
            assert rel_err(rhs[s, r].cpu().numpy(), po) <= TOL
        record("kcond", case=name, scenario=s, delta_w=delta, cond2_Kcond=cond2_spd(Kc),
               L_rel_err=float(rel_err(L, Lo)))
    # an indefinite shift: info = first failing column, as the oracle's
    lam_min = min(lmins)
    shift = -lam_min - 10.0
    K = dev(KV.copy())
    h.pf_condensed_kkt_solve(S, K, dev(stack(pts, "sigma_u")), shift, None, 0, info)
    torch.cuda.synchronize()
    for s in range(S):
        _, io = O.cholesky(O.condensed(0.5 * (KV[s] + KV[s].T), pts[s]["sigma_u"], shift))
        assert info[s].item() == io
    h.close()


@pytest.mark.parametrize("name", ["case118", "case1354"])
def test_condensed_kkt_high_condition(pfmod, name):
    """The paper's regime cond(K_cond) up to 1e13: δ_w just above
    the smallest PD shift (cond₂ ≥ 1e10).  The factor is unique (R21) but its
    forward error grows with cond, so the checks are R20's: info = 0 as the
    oracle's, backward error ‖K_cond p − b‖∞/(‖K_cond‖∞‖p‖∞ + ‖b‖∞) ≤ 4 n_u ε,
    ‖LLᵀ − K_cond‖/‖K_cond‖ ≤ 4 n_u ε, and L vs the oracle within cond·ε."""
    import torch
    net, pt = table1_grid(name)
    pts = [pt]
    part = O.partition(net)
    n_u = part["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=1)
    KV, _ = _run_khat(pfmod, h, net, pts)
    Kh = 0.5 * (KV[0] + KV[0].T)
    w = np.linalg.eigvalsh(Kh + np.diag(pt["sigma_u"]))
    delta = -w[0] + (w[-1] - w[0]) * 3e-11
    Kc = O.condensed(Kh, pt["sigma_u"], delta)
    c2 = cond2_spd(Kc)
    assert 1e9 <= c2 < 1e13, c2
    b = np.random.default_rng(8).standard_normal((1, 1, n_u))
    K, rhs = dev(KV.copy()), dev(b.copy())
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    h.pf_condensed_kkt_solve(1, K, dev(pt["sigma_u"][None]), delta, rhs, 1, info)
    torch.cuda.synchronize()
    Lo, io = O.cholesky(Kc)
    assert info.item() == io == 0
    L = K.cpu().numpy()[0].T
    p = rhs.cpu().numpy()[0, 0]
    eps = np.finfo(float).eps
    bwd = np.abs(Kc @ p - b[0, 0]).max() / (np.abs(Kc).sum(1).max() * np.abs(p).max() + np.abs(b).max())
    fac = np.abs(L @ L.T - Kc).max() / np.abs(Kc).max()
    assert bwd <= 4 * n_u * eps, bwd
    assert fac <= 4 * n_u * eps, fac
    lerr = rel_err(L, Lo)
    assert lerr <= max(TOL, c2 * eps), lerr
    record("kcond_high", case=name, delta_w=float(delta), cond2_Kcond=c2, backward_err=float(bwd),
           factor_residual=float(fac), L_rel_err=float(lerr))
    h.close()


def test_condensed_kkt_many_rhs_mixed_info(pfmod):
    """Three scenarios, six right-hand sides (more than one DAG run carries),
    one scenario made indefinite through Σ_u: its info is the oracle's first
    failing column and its right-hand sides stay untouched; the others solve."""
    import torch
    net, pt = table1_grid("case118")
    pts = [pt, make_scenario(net, pt, 1), make_scenario(net, pt, 2)]
    S, R = 3, 6
    n_u = O.partition(net)["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    KV, _ = _run_khat(pfmod, h, net, pts)
    Khs = [0.5 * (KV[s] + KV[s].T) for s in range(S)]
    sig = stack(pts, "sigma_u").copy()
    delta = max(0.0, -min(np.linalg.eigvalsh(Khs[s] + np.diag(sig[s])).min() for s in range(S))) * 1.5 + 1.0
    sig[1, 70] = -1e9
    rng = np.random.default_rng(5)
    b = rng.standard_normal((S, R, n_u))
    K, rhs = dev(KV.copy()), dev(b.copy())
    info = torch.empty(S, dtype=torch.int32, device="cuda")
    h.pf_condensed_kkt_solve(S, K, dev(sig), delta, rhs, R, info)
    torch.cuda.synchronize()
    got = rhs.cpu().numpy()
    Lg = K.cpu().numpy()
    for s in range(S):
        Lo, io = O.cholesky(O.condensed(Khs[s], sig[s], delta))
        assert info[s].item() == io, s
        if io:
            assert s == 1 and io == 71
            assert np.array_equal(got[s], b[s])
            continue
        assert rel_err(Lg[s].T, Lo) <= TOL
        for r in range(R):
            assert rel_err(got[s, r], O.chol_solve(Lo, b[s, r])) <= TOL, (s, r)
    h.close()


@pytest.mark.parametrize("n_scen", [1, 3])
def test_condensed_kkt_nonfinite_and_indefinite(pfmod, n_scen):
    """Degenerate inputs never fault: a NaN K̂, an all-zero K̂ (first pivot 0) and a
    negative-definite K̂ give info = 1 for every scenario, leave the right-hand
    sides untouched, and the handle stays usable for a regular solve after."""
    import torch
    net, pt = table1_grid("case1354")
    n_u = O.partition(net)["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=n_scen)
    b = np.random.default_rng(4).standard_normal((n_scen, 1, n_u))
    info = torch.empty(n_scen, dtype=torch.int32, device="cuda")
    for fill in (np.nan, 0.0, -1.0):
        Kbad = np.full((n_scen, n_u, n_u), fill) if fill != -1.0 else np.stack([-np.eye(n_u)] * n_scen)
        K, rhs = dev(Kbad), dev(b.copy())
        h.pf_condensed_kkt_solve(n_scen, K, None, 0.0, rhs, 1, info)
        torch.cuda.synchronize()
        assert info.cpu().tolist() == [1] * n_scen, fill
        assert np.array_equal(rhs.cpu().numpy(), b)
    A = np.random.default_rng(5).standard_normal((n_u, n_u))
    Kgood = np.stack([A @ A.T / n_u + np.eye(n_u)] * n_scen)
    K, rhs = dev(Kgood.copy()), dev(b.copy())
    h.pf_condensed_kkt_solve(n_scen, K, None, 0.0, rhs, 1, info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * n_scen
    Lo, _ = O.cholesky(Kgood[0])
    assert rel_err(rhs[0, 0].cpu().numpy(), O.chol_solve(Lo, b[0, 0])) <= TOL
    h.close()


@pytest.mark.parametrize("name", ["case118", "case300"])
def test_lu_singular_pivot_info(pfmod, name):
    """A5's failure contract (R18): a scenario with v_i = 0 at a PQ bus makes
    G_x's θ_i column vanish, so its static pivot is 0.  pf_jacobian's info is
    the oracle's first failing permuted pivot (k+1, from the oracle's own R18
    ordering and dense no-pivot LU); the regular scenario of the same call
    reports 0, and the handle works afterwards."""
    import torch
    net, pt = table1_grid(name)
    part = O.partition(net)
    pq = [i for i in range(net["n_b"]) if not part["is_gen"][i]]
    bad = dict(pt, v=pt["v"].copy())
    bad["v"][pq[len(pq) // 2]] = 0.0
    pts = [pt, bad, make_scenario(net, pt, 2)]
    perm, _ = O.permutation(part, O.md_ordering(net, part))
    want = []
    for p in pts:
        Gx, _, _ = O.jacobians(net, part, p)
        want.append(O.static_lu(Gx, perm)[0])
    assert want[0] == 0 and want[1] > 0 and want[2] == 0
    h = pfmod.Network(net, max_batch=8, max_scen=3)
    assert np.array_equal(h.structure("perm"), perm)
    info = torch.full((3,), -7, dtype=torch.int32, device="cuda")
    h.pf_jacobian(3, dev(stack(pts, "v")), dev(stack(pts, "theta")), info=info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == want
    record("lu_info", case=name, info=want)
    # the handle stays usable: the regular scenarios factorize and reduce
    KV, inf2 = _run_khat(pfmod, h, net, [pts[0]], N=8)
    assert inf2.tolist() == [0]
    assert np.all(np.isfinite(KV))
    h.close()


def test_capacity_and_argument_errors(pfmod):
    import torch
    net, pt = table1_grid("case118")
    h = pfmod.Network(net, max_batch=4, max_scen=1)
    KV = torch.empty(1, 8, h.dims["n_u"], dtype=torch.float64, device="cuda")
    v, th = dev(pt["v"][None]), dev(pt["theta"][None])
    with pytest.raises(pfmod.PFError) as e:   # reduction before any jacobian
        h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), KV[:, :4].contiguous(), N=4)
    assert e.value.status == 5
    h.pf_jacobian(1, v, th)
    with pytest.raises(pfmod.PFError) as e:
        h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), KV, N=8)
    assert e.value.status == 3
    with pytest.raises(pfmod.PFError) as e:
        h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), KV[:, :4].contiguous(),
                                   col0=h.dims["n_u"] - 2, N=4)
    assert e.value.status == 1
    # a different point than the last pf_jacobian's (same values, other arrays): refused
    with pytest.raises(pfmod.PFError) as e:
        h.pf_reduced_hessian_batch(1, v.clone(), th, dev(pt["lam"][None]), dev(pt["y"][None]),
                                   KV[:, :4].contiguous(), N=4)
    assert e.value.status == 5
    # NULL v/theta = the last pf_jacobian's point; more scenarios than it factorized: refused
    h.pf_reduced_hessian_batch(1, None, None, dev(pt["lam"][None]), dev(pt["y"][None]), KV[:, :4].contiguous(), N=4)
    # N = 0 is a no-op
    h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), KV[:, :0].contiguous(), N=0)
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(net, max_batch=4, max_scen=1, tile_cols=12)
    assert e.value.status == 1
    h.close()


@pytest.mark.slow
@pytest.mark.parametrize("name,S,tile", [("case9241", 8, 64), ("case9241", 4, 32), ("case2869", 8, 16),
                                         ("case2869", 2, 8)])
def test_full_size(pfmod, name, S, tile):
    """Full BASELINE sizes in the launch configuration the handle picks itself
    (case9241 × 8 scenarios: the bench's 64-direction tiles; × 4: 32; case2869
    × 8: 16; × 2: 8): all n_u directions of all scenarios in one call, the WHOLE
    K̂ of the first and last scenario vs the oracle per column, every scenario
    symmetric (P12) and finite, then the condensed-KKT Cholesky + solve of all
    scenarios at once vs the oracle's on those two."""
    import torch
    net, pt = table1_grid(name)
    pts = [pt] + [make_scenario(net, pt, s) for s in range(1, S)]
    checked = [0, S - 1]
    part = O.partition(net)
    n_u = part["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    assert h.dims["tile_cols"] == tile  # the width pick_tile_cols gives this launch shape
    KV, info = _run_khat(pfmod, h, net, pts)
    assert info.tolist() == [0] * S
    assert np.all(np.isfinite(KV))
    for s in range(S):
        assert np.abs(KV[s] - KV[s].T).max() <= 1e-12 * np.abs(KV[s]).max()
    Khs = {}
    for s in checked:
        Khs[s] = 0.5 * (KV[s] + KV[s].T)
        _check_khat(name, KV[s], net, pts[s], s, {"tile_cols": tile, "scenarios_in_call": S})
    delta = max(0.0, -min(np.linalg.eigvalsh(Khs[s] + np.diag(pts[s]["sigma_u"])).min() for s in checked)) * 1.5 + 1.0
    delta = max(delta, 1e6)  # every scenario PD (the bench's δ_w search lands at 1e6 on these points)
    b = np.random.default_rng(12).standard_normal((S, 1, n_u))
    K, rhs = dev(KV.copy()), dev(b.copy())
    info = torch.empty(S, dtype=torch.int32, device="cuda")
    h.pf_condensed_kkt_solve(S, K, dev(stack(pts, "sigma_u")), delta, rhs, 1, info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * S
    Lg = K.cpu().numpy()
    for s in checked:
        Kc = O.condensed(Khs[s], pts[s]["sigma_u"], delta)
        Lo, io = O.cholesky(Kc)
        assert io == 0
        assert rel_err(Lg[s].T, Lo) <= TOL, (name, s)
        assert rel_err(rhs[s, 0].cpu().numpy(), O.chol_solve(Lo, b[s, 0])) <= TOL, (name, s)
        record("kcond", case=name, scenario=s, delta_w=delta, cond2_Kcond=cond2_spd(Kc),
               L_rel_err=float(rel_err(Lg[s].T, Lo)))
    h.close()


def test_cuda_graph_capture_replay(pfmod):
    """The per-iteration device work — constraints, Jacobians + LU refactor, the full
    reduced Hessian (prep on the side stream, fork/join) and the condensed-KKT
    factor + solve — is CUDA-graph capturable: captured once with
    torch.cuda.graph and replayed, it reproduces the eager results bit for bit, also
    after the inputs change in place (a new point replayed through the same graph)."""
    import torch
    net, pt = table1_grid("case118")
    pts = [pt, make_scenario(net, pt, 1)]
    S, n_u = len(pts), O.partition(net)["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    inp = {k: dev(stack(pts, k)) for k in ("v", "theta", "p_g", "q_g", "p_d", "q_d", "lam", "y", "sigma_s",
                                           "sigma_x", "sigma_u")}
    G = torch.empty(S, 2 * net["n_b"], dtype=torch.float64, device="cuda")
    KV = torch.empty(S, n_u, n_u, dtype=torch.float64, device="cuda")
    rhs = torch.empty(S, n_u, dtype=torch.float64, device="cuda")
    info = torch.empty(S, dtype=torch.int32, device="cuda")

    def body():
        h.pf_eval_constraints(S, inp["v"], inp["theta"], inp["p_g"], inp["q_g"], inp["p_d"], inp["q_d"], G)
        h.pf_jacobian(S, inp["v"], inp["theta"])
        h.pf_reduced_hessian_batch(S, inp["v"], inp["theta"], inp["lam"], inp["y"], KV, sigma_s=inp["sigma_s"],
                                   sigma_x=inp["sigma_x"], N=n_u, p_d=inp["p_d"])
        rhs.fill_(1.0)
        h.pf_condensed_kkt_solve(S, KV, inp["sigma_u"], 1e6, rhs=rhs, nrhs=1, info=info)

    def eager():
        body()
        torch.cuda.synchronize()
        return G.clone(), KV.clone(), rhs.clone(), info.clone()

    ref = eager()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()  # warm-up on the capture stream (lazy attributes, allocator)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for X in (G, KV, rhs):
        X.zero_()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip((G, KV, rhs, info), ref):
        assert torch.equal(a, b)
    # a new point through the same graph (inputs updated in place) equals an eager call
    inp["v"].mul_(1.001)
    inp["theta"].mul_(0.999)
    g.replay()
    torch.cuda.synchronize()
    got = (G.clone(), KV.clone(), rhs.clone(), info.clone())
    ref2 = eager()
    for a, b in zip(got, ref2):
        assert torch.equal(a, b)
    assert not torch.equal(ref2[1], ref[1])
    h.close()


def test_lu_row_workspace_capacity_error(pfmod):
    """k_lu keeps a dense workspace of the longest filled-LU row per warp in SMEM; a
    network whose longest row does not fit (a 1,500-leaf star around a PQ hub, the
    generator / reference at a leaf: the hub's rows span every other state, 3,000
    entries) is refused at build with PF_ERR_CAPACITY and a message naming the row
    length — not a CUDA launch failure at the first pf_jacobian."""
    from synth.grid import pi_model
    nl = 1500
    n_b = nl + 1
    r = np.full(nl, 0.01)
    x = np.full(nl, 0.1)
    Yff, Yft, Ytf, Ytt = pi_model(r, x, np.zeros(nl), np.ones(nl), np.zeros(nl))
    net = dict(n_b=n_b, n_l=nl, n_g=1, line_from=np.zeros(nl, np.int32), line_to=np.arange(1, n_b, dtype=np.int32),
               Y_ff=Yff, Y_ft=Yft, Y_tf=Ytf, Y_tt=Ytt, Y_sh=np.zeros(n_b, complex), gen_bus=np.array([1], np.int32),
               ref_bus=1, p_d=np.full(n_b, 0.001), q_d=np.zeros(n_b), F_max=np.ones(nl),
               c_quad=np.array([1.0]), c_lin=np.array([1.0]), seed=3)
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(net, max_batch=1, max_scen=1)
    assert e.value.status == 3  # PF_ERR_CAPACITY
    assert "SMEM" in str(e.value) and "3000" in str(e.value)
