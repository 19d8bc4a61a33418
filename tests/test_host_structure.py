"""CPU-only checks of the native library: it loads, exports every symbol
include/pf.h declares, and its host structural analysis (A1: partition,
patterns, R18 ordering, symbolic LU, level sets) is bit-exact with the
oracle's independent structural routines (R19)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pf_oracle as O
from synth import case9
from synth.grid import table1_grid
from tests.nets import rich_small

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pfmod():
    from paper_2203_11875_b200 import _build
    _build.build()
    import paper_2203_11875_b200 as m
    m.load_library()
    return m


def test_library_exports_every_header_symbol(pfmod):
    hdr = open(os.path.join(ROOT, "include", "pf.h")).read()
    declared = sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", hdr)))
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2203_11875_b200", "libpf.so"))
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(pfmod.SYMBOLS)


def _nets():
    out = [("case9",) + case9(), ("rich8",) + rich_small(), ("rich8b",) + rich_small(11)]
    out.append(("case118",) + table1_grid("case118"))
    out.append(("case300",) + table1_grid("case300"))
    out.append(("case1354",) + table1_grid("case1354"))
    out.append(("case2869",) + table1_grid("case2869"))   # the benchmarked shapes (configs 3 and 4/5)
    out.append(("case9241",) + table1_grid("case9241"))
    return out


@pytest.mark.parametrize("name,net,pt", _nets())
def test_structure_bit_exact(pfmod, name, net, pt):
    h = pfmod.Network(net, max_batch=8, max_scen=1, device=-1)
    part = O.partition(net)
    d = h.dims
    assert (d["n_x"], d["n_u"], d["m"], d["n_r"], d["n_h"]) == (part["n_x"], part["n_u"], part["m"], part["n_r"], part["n_h"])
    for k, key in (("x_theta", "x_th"), ("x_v", "x_v"), ("u_v", "u_v"), ("u_p", "u_p")):
        assert np.array_equal(h.structure(k), part[key]), k
    (px, ix), (pu, iu) = O.gx_gu_patterns(net, part)
    assert np.array_equal(h.structure("gx_ptr"), px) and np.array_equal(h.structure("gx_idx"), ix)
    assert np.array_equal(h.structure("gu_ptr"), pu) and np.array_equal(h.structure("gu_idx"), iu)
    pa, ia = O.a_pattern(net, part)
    assert np.array_equal(h.structure("a_ptr"), pa) and np.array_equal(h.structure("a_idx"), ia)
    order = O.md_ordering(net, part)
    assert np.array_equal(h.structure("bus_order"), order)
    perm, blk = O.permutation(part, order)
    assert np.array_equal(h.structure("perm"), perm) and np.array_equal(h.structure("block_ptr"), blk)
    F = O.symbolic_lu(px, ix, perm)
    lp, li = O.filled_csr(F)
    assert np.array_equal(h.structure("lu_ptr"), lp) and np.array_equal(h.structure("lu_idx"), li)
    levL, levU = O.block_levels(F, blk)
    for lev, tag in ((levL, "l"), (levU, "u")):
        ptr, blocks = O.level_sets(lev)
        assert np.array_equal(h.structure("level_%s_ptr" % tag), ptr)
        assert np.array_equal(h.structure("level_%s_blk" % tag), blocks)
    h.close()


def test_topology_errors(pfmod):
    net, _ = case9()
    bad = dict(net, gen_bus=np.array([0, 1, 1], np.int32))
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(bad, 5, 1, device=-1)
    assert e.value.status == 2
    bad = dict(net, ref_bus=4)
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(bad, 5, 1, device=-1)
    assert e.value.status == 2
    lf = net["line_from"].copy()
    lf[0] = net["line_to"][0]
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(dict(net, line_from=lf), 5, 1, device=-1)
    assert e.value.status == 2
    # disconnected: drop bus 0's only line by re-routing it to bus 8 (0 isolated)
    lf = net["line_from"].copy()
    lf[0] = 8
    with pytest.raises(pfmod.PFError) as e:
        pfmod.Network(dict(net, line_from=lf), 5, 1, device=-1)
    assert e.value.status == 2


def test_host_only_handle_refuses_compute(pfmod):
    net, _ = case9()
    h = pfmod.Network(net, 5, 1, device=-1)
    lib = pfmod.load_library()
    st = lib.pf_jacobian(h._h, 1, ctypes.c_void_p(8), ctypes.c_void_p(8), None, None, None, None, None)
    assert st == 5
    h.close()


@pytest.mark.parametrize("name,net,pt", _nets())
def test_lu_schedule(pfmod, name, net, pt):
    """k_lu's schedule (A5) against the oracle's own symbolic LU: the dense front is the set of
    rows of levels >= front_level (the lowest cut with at most 96 rows) and is closed upwards
    (no row outside it has a pivot inside it); the bottom subtree lists cover every block below
    lu_cut_level exactly once, and every block a listed block depends on (an L pivot's block)
    comes earlier in the same pair's list; each level's LU order is a permutation of the level."""
    h = pfmod.Network(net, max_batch=8, max_scen=1, device=-1)
    part = O.partition(net)
    d = h.dims
    (px, ix), _ = O.gx_gu_patterns(net, part)
    perm, blk = O.permutation(part, O.md_ordering(net, part))
    F = O.symbolic_lu(px, ix, perm)
    lp, li = O.filled_csr(F)
    levL, _ = O.block_levels(F, blk)
    levL = np.asarray(levL)
    nblk = len(blk) - 1
    row_blk = np.repeat(np.arange(nblk), np.diff(blk))
    row_lev = levL[row_blk]
    n_x = len(lp) - 1
    fl = d["front_level"]
    front = h.structure("front_row")
    assert np.array_equal(front, np.nonzero(row_lev >= fl)[0])
    assert d["front_rows"] == len(front) <= 96
    if fl > 0:
        assert (row_lev >= fl - 1).sum() > 96, "the cut is not the lowest one"
    infront = np.zeros(n_x, bool)
    infront[front] = True
    for r in np.nonzero(~infront)[0]:
        piv = li[lp[r]:lp[r + 1]]
        assert not infront[piv[piv < r]].any(), "row %d outside the front has a front pivot" % r
    # bottom subtree lists
    cut = d["lu_cut_level"]
    assert 0 <= cut <= fl
    ptr = h.structure("lu_subtree_ptr")
    lst = h.structure("lu_subtree_blk")
    assert d["lu_pairs"] == len(ptr) - 1 and ptr[0] == 0 and ptr[-1] == len(lst)
    assert np.array_equal(np.sort(lst), np.nonzero(levL < cut)[0])
    deps = [set() for _ in range(nblk)]
    for r in range(n_x):
        piv = li[lp[r]:lp[r + 1]]
        for c in piv[piv < r]:
            if row_blk[c] != row_blk[r]:
                deps[row_blk[r]].add(int(row_blk[c]))
    for t in range(len(ptr) - 1):
        seen = set()
        for b in lst[ptr[t]:ptr[t + 1]]:
            assert deps[b] <= seen, "pair %d: block %d before its dependencies" % (t, b)
            seen.add(int(b))
    # per-level LU order: a permutation of each level set
    lptr = h.structure("level_l_ptr")
    lblk = h.structure("level_l_blk")
    lub = h.structure("lu_level_blk")
    for l in range(len(lptr) - 1):
        assert np.array_equal(np.sort(lub[lptr[l]:lptr[l + 1]]), np.sort(lblk[lptr[l]:lptr[l + 1]]))
    h.close()
