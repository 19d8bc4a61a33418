"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle,
element by element on the same seeded inputs.  Tolerance:
normwise max|a−b| / max|b| ≤ 1e-10 per output array (R20, BASELINE.json
north_star), bit-exact for integer outputs (info) and for batch invariance."""
import numpy as np
import pytest

from oracle import pf_oracle as O
from synth import case9, make_scenario
from synth.case9 import case9_multipliers
from synth.grid import table1_grid
from tests.gpu_common import csr_dense, dev, oracle_khat, rel_err, stack
from tests.nets import rich_small

pytestmark = pytest.mark.gpu
TOL = 1e-10


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


def _cases(names):
    out = []
    for name in names:
        if name == "case9":
            net, pt = _case9_point()
            pts = [pt]
        elif name == "rich8":
            net, pt = rich_small()
            pts = [pt]
        else:
            net, pt = table1_grid(name)
            pts = [pt, make_scenario(net, pt, 1)]
        out.append((name, net, pts))
    return out


SMALL = ["case9", "rich8", "case118"]
MEDIUM = ["case9", "rich8", "case118", "case1354"]


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
    Gx = torch.empty(S, d["nnz_gx"], dtype=torch.float64, device="cuda")
    Gu = torch.empty(S, d["nnz_gu"], dtype=torch.float64, device="cuda")
    A = torch.empty(S, d["nnz_a"], dtype=torch.float64, device="cuda")
    info = torch.full((S,), -7, dtype=torch.int32, device="cuda")
    h.pf_jacobian(S, dev(stack(pts, "v")), dev(stack(pts, "theta")), Gx, Gu, A, info)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * S
    part = O.partition(net)
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


@pytest.mark.parametrize("name,net,pts", _cases(MEDIUM))
def test_reduced_hessian_full(pfmod, name, net, pts):
    """Full K̂ (unit directions, one batch) vs the naive-sensitivity oracle."""
    S = len(pts)
    part = O.partition(net)
    h = pfmod.Network(net, max_batch=part["n_u"], max_scen=S)
    KV, info = _run_khat(pfmod, h, net, pts)
    assert info.tolist() == [0] * S
    for s, pt in enumerate(pts):
        Kh, _ = oracle_khat(net, pt)
        # KV[s][j] is column j of K̂ (column-major): compare unsymmetrised (R21)
        assert rel_err(KV[s].T, Kh) <= TOL, name
        sym = 0.5 * (KV[s] + KV[s].T)
        assert rel_err(sym, 0.5 * (Kh + Kh.T)) <= TOL
        assert np.abs(KV[s] - KV[s].T).max() <= 1e-12 * np.abs(KV[s]).max()   # P12
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
        assert rel_err(KV[s], (Kh @ Vs[s].T).T) <= TOL
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
def test_tile_width_invariance_bitwise(pfmod, name, monkeypatch):
    """64-direction tiles (two directions per lane, the bench's launch shape) and
    8-direction tiles (teams of 8 lanes) run the same arithmetic per direction,
    so K̂ is bit-identical across tile widths, for unit directions
    in aligned (sparse-RHS reach) and unaligned calls and for dense V, and it
    matches the oracle."""
    import torch
    net, pt = table1_grid(name)
    pts = [pt, make_scenario(net, pt, 1)]
    n_u = O.partition(net)["n_u"]
    outs = {}
    rng = np.random.default_rng(21)
    Vd = rng.standard_normal((len(pts), 70, n_u))
    for c in ("8", "64"):
        monkeypatch.setenv("PF_TILE_COLS", c)
        h = pfmod.Network(net, max_batch=n_u, max_scen=len(pts))
        assert h.dims["tile_cols"] == int(c)
        full, _ = _run_khat(pfmod, h, net, pts)
        part, _ = _run_khat(pfmod, h, net, pts, N=70, col0=37)      # unaligned: full L sweep
        dense, _ = _run_khat(pfmod, h, net, pts, N=70, V=dev(Vd))  # dense directions
        outs[c] = (full, part, dense)
        h.close()
    for a, b in zip(outs["8"], outs["64"]):
        assert np.array_equal(a, b)
    full = outs["64"][0]
    assert np.array_equal(outs["64"][1], full[:, 37:107])
    for s, p in enumerate(pts):
        assert rel_err(full[s].T, oracle_khat(net, p)[0]) <= TOL


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
    lmins = [np.linalg.eigvalsh(Kh + np.diag(p["sigma_u"])).min() for Kh, p in zip(Khs, pts)]
    delta = max(0.0, -min(lmins)) * 1.5 + 1.0
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
    # N = 0 is a no-op
    h.pf_reduced_hessian_batch(1, v, th, dev(pt["lam"][None]), dev(pt["y"][None]), KV[:, :0].contiguous(), N=0)
    h.close()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["case2869", "case9241"])
def test_full_size_sampled_columns(pfmod, name):
    """Full BASELINE sizes in the bench's launch configuration — case9241: the 8
    scenarios of config 5 in one call with all n_u directions (64-direction
    tiles, sparse-RHS reach, subtree schedules), case2869: 2 scenarios —
    sampled columns vs the oracle's adjoint route computed one column at a time
    (SuperLU solves) on the first and last scenario, then the condensed-KKT
    Cholesky + solve of all scenarios at once vs the oracle's on those two."""
    import torch
    net, pt = table1_grid(name)
    S = 8 if name == "case9241" else 2
    pts = [pt] + [make_scenario(net, pt, s) for s in range(1, S)]
    checked = [0, S - 1]
    part = O.partition(net)
    n_u = part["n_u"]
    h = pfmod.Network(net, max_batch=n_u, max_scen=S)
    if name == "case9241":
        assert h.dims["tile_cols"] == 64  # the bench's tile width
    KV, info = _run_khat(pfmod, h, net, pts)
    assert info.tolist() == [0] * S
    assert np.all(np.isfinite(KV))
    rng = np.random.default_rng(11)
    cols = np.unique(np.concatenate([[0, n_u - 1, part["n_u"] // 2], rng.choice(n_u, 5, replace=False)]))
    for s in checked:
        p = pts[s]
        Gx, Gu, A = O.jacobians(net, part, p)
        K = O.kkt_K(net, part, p, p["lam"], p["y"], p["sigma_s"], p["sigma_x"])
        ref = O.reduce_columns(K, Gx, Gu, cols)
        got = KV[s][cols].T
        assert rel_err(got, ref) <= TOL, (name, s)
    # the condensed-KKT Cholesky + solve at full size (bench launch: all scenarios at once)
    Khs = {s: 0.5 * (KV[s] + KV[s].T) for s in checked}
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
        Lo, io = O.cholesky(O.condensed(Khs[s], pts[s]["sigma_u"], delta))
        assert io == 0
        assert rel_err(Lg[s].T, Lo) <= TOL, (name, s)
        assert rel_err(rhs[s, 0].cpu().numpy(), O.chol_solve(Lo, b[s, 0])) <= TOL, (name, s)
    h.close()
