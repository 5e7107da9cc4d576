"""Rule tables (host re-derivation shipped to the device) against the reference payloads
(moments of every payload and full arrays of a subset, recorded from
quadrature.reference_payload, quadrature.py:401-420, by tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import golden
from oracle import fraclap_oracle as O
from paper_1708_03912_b200 import quadrature as Q

T = Q.PairTopology
NAMES = {"identical": T.IDENTICAL, "common_edge": T.COMMON_EDGE, "common_vertex": T.COMMON_VERTEX,
         "edge_of_cell": T.EDGE_OF_CELL, "touching_edge": T.TOUCHING_EDGE, "disjoint": T.DISJOINT}


def _keys():
    try:
        G = golden("tables")
    except BaseException:
        return []
    return sorted(k[:-4] for k in G.files if k.endswith("/sha"))


def _parse(key):
    d, topo, k, s, van = key.split("/")
    return int(d), NAMES[topo], int(k), (0.5 if s == "x" else float(s)), int(van)


def _moments(p):
    """The moments make_golden.py recorded: count, sum w, and per coordinate sum w c, sum w c^2,
    min c, max c."""
    w = np.asarray(p["w"], float)
    mom = [len(w), w.sum()]
    for key in sorted(p):
        if key == "w":
            continue
        a = np.asarray(p[key], float).reshape(len(w), -1)
        for c in range(a.shape[1]):
            mom += [(w * a[:, c]).sum(), (w * a[:, c] ** 2).sum(), a[:, c].min(), a[:, c].max()]
    return np.array(mom)


@pytest.mark.parametrize("key", _keys())
def test_payload_moments(key):
    """Every payload the configurations can touch (re-derived as Duffy pieces in
    quadrature._rule) against the reference's: node count exact, moments within 1e-14."""
    G = golden("tables")
    d, topo, k, s, van = _parse(key)
    p = Q.payload(topo, max(k, 2), s, d, van)
    mom, want = _moments(p), G[key + "/mom"]
    assert mom.shape == want.shape and mom[0] == want[0], key
    assert np.all(np.abs(mom - want) <= 1e-14 * np.maximum(1.0, np.abs(want))), (key, np.abs(mom - want).max())


def _payload_keys():
    try:
        G = golden("payloads")
    except BaseException:
        return []
    return sorted({k.rsplit("/", 1)[0] for k in G.files})


@pytest.mark.parametrize("key", _payload_keys())
def test_payload_arrays(key):
    """Node by node against the reference's own arrays (tests/golden/payloads.npz): coordinates
    within 1e-14, weights within 1e-14 of the largest weight."""
    G = golden("payloads")
    d, topo, k, s, van = key.split("/")
    p = Q.payload(getattr(T, topo.upper()), int(k), float(s), int(d), int(van))
    for name in p:
        a, b = np.asarray(p[name], float), G[key + "/" + name]
        assert a.shape == b.shape, (key, name)
        scale = np.abs(b).max() if name == "w" else 1.0
        assert np.abs(a - b).max() <= 1e-14 * scale, (key, name, np.abs(a - b).max())


@pytest.mark.parametrize("key", _keys()[::3])
def test_oracle_rules_match_reference(key):
    """The oracle's independent (loop-based) restatement agrees with the reference moments."""
    G = golden("tables")
    d, topo, k, s, van = _parse(key)
    short = {T.IDENTICAL: "ident", T.COMMON_EDGE: "ce", T.COMMON_VERTEX: "cv", T.EDGE_OF_CELL: "eoc",
             T.TOUCHING_EDGE: "te"}
    if topo is T.DISJOINT:
        pytest.skip("disjoint product rule is the simplex rule squared")
    x, y, w = O.rule(short[topo], max(k, 2), s, d, van)
    mom = G[key + "/mom"]
    assert int(mom[0]) == len(w)
    assert abs(mom[1] - w.sum()) <= 1e-14 * max(1.0, abs(mom[1]))


def test_pack_tables_layout():
    dir_, data = Q.pack_tables(2, 0.5)
    d = dir_.reshape(Q.NTOPO, Q.KDIR, 2)
    assert d[Q.TOPO_CELL, 0, 1] == 16 and d[Q.TOPO_EDGE_GL, 0, 1] == 8
    assert d[3, 9, 1] == 81 and d[3, 10, 1] == 0           # 2D disjoint cap k <= 9
    assert d[1, 20, 1] == d[1, 16, 1] == 12 * 16 * 16       # CE uses min(k, 16)
    assert (d[..., 0] + d[..., 1]).max() * Q.NODE <= len(data)
    d1, _ = Q.pack_tables(1, 0.75)
    d1 = d1.reshape(Q.NTOPO, Q.KDIR, 2)
    assert d1[Q.TOPO_CELL, 0, 1] == 6 and d1[3, 32, 1] == 32 and d1[0, 0, 1] == 6


def test_gauss_legendre_exactness():
    # SPEC.md:134-140
    x, w = Q.gauss_legendre(8)
    assert abs((w * x ** 15).sum() - 1 / 16) < 1e-14
    x, w = Q.gauss_legendre(1)
    assert x[0] == 0.5 and w[0] == 1.0


def test_select_order_properties():
    # SPEC.md:148-156
    p = Q.OrderParams()
    k1 = Q.select_order(T.IDENTICAL, 0.1, 0.1, 0.0, 100, 0.5, p)
    k4 = Q.select_order(T.IDENTICAL, 0.1, 0.1, 0.0, 400, 0.5, p)
    assert k4 >= k1
    kb = Q.select_order(T.EDGE_OF_CELL, 0.1, 0.1, 0.0, 100, 0.5, p, boundary=True)
    assert kb <= k1
    far = Q.select_order(T.DISJOINT, 0.01, 0.01, 1e6, 100, 0.5, p)
    assert far == 2
    with pytest.raises(Q.QuadratureError):
        Q.select_order(T.DISJOINT, 0.1, 0.1, 0.0, 100, 0.5, p)
    assert Q.classify_pair([0, 1, 2], [0, 1, 2]) is T.IDENTICAL
    assert Q.classify_pair([0, 1, 2], [1, 2, 3]) is T.COMMON_EDGE
    assert Q.classify_pair([0, 1], [1, 2]) is T.COMMON_VERTEX
    assert Q.classify_pair([0, 1, 2], [3, 4, 5]) is T.DISJOINT
