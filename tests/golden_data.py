"""Loader for the text fixtures under tests/golden/ (values printed by the paper,
SPEC.md or the published case9 solutions; each file's header cites its source)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def table1():
    """{case: (n_b, n_l, n_g, n_x, n_u)} of PAPER.md Table 1 (L1275–1285)."""
    rows = _lines("table1_instances.tsv")
    assert rows[0] == ["case", "n_b", "n_l", "n_g", "n_x", "n_u"]
    return {r[0]: tuple(int(x) for x in r[1:]) for r in rows[1:]}


def keyed(name):
    """{key: [floats]} of a 'key v1 v2 …' fixture."""
    return {r[0]: [float(x) for x in r[1:]] for r in _lines(name)}


def complex_pair(s):
    re, im = s.split(",")
    return complex(float(re), float(im))


def spec_pi_model():
    out = {}
    for r in _lines("spec_pi_model.txt"):
        out[r[0]] = r[1:]
    return out
