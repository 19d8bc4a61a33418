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
