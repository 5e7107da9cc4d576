"""Pin the CPU oracle (oracle/fraclap_oracle.py) to the reference's own outputs
(tests/golden/*.npz, produced by running the unmodified reference)."""
import hashlib

import numpy as np
import pytest

from conftest import golden, irregular_cases, irregular_mesh, make_mesh, small_cases, tiny_cases
from oracle import fraclap_oracle as O


def _fast(cases):
    return [c for c in cases if not (c[1] == "square2d" and c[2] >= 12)]


@pytest.mark.parametrize("key,kind,N,s", _fast(small_cases()))
def test_oracle_small_matrices(key, kind, N, s):
    from paper_1708_03912_b200 import mesh as M
    G = golden("small")
    mesh = make_mesh(kind, N)
    dm = M.DofMap(mesh, s)
    A = O.assemble_dense(mesh, dm, s)
    Ar = G[key + "/A"]
    assert np.abs(A - Ar).max() <= 1e-13 * np.abs(Ar).max()
    b = O.load_vector(mesh, dm)
    assert np.allclose(b, G[key + "/b"], rtol=1e-14, atol=1e-16)
    x, it, _, _ = O.pcg(A, b, tol=1e-10, max_iter=10 ** 5)
    assert it == int(G[key + "/iters"])
    assert np.linalg.norm(x - G[key + "/x"]) <= 1e-9 * np.linalg.norm(G[key + "/x"])


@pytest.mark.slow
@pytest.mark.parametrize("key,kind,N,s", [c for c in small_cases() if c not in _fast(small_cases())])
def test_oracle_small_matrices_2d12(key, kind, N, s):
    test_oracle_small_matrices(key, kind, N, s)


def test_oracle_c1_full():
    from paper_1708_03912_b200 import mesh as M
    G = golden("c1")
    mesh = make_mesh("uniform1d", 512)
    dm = M.DofMap(mesh, 0.25)
    assert dm.n == 513                                    # s < 1/2: every vertex (mesh.py:225)
    A = O.assemble_dense(mesh, dm, 0.25)
    assert np.abs(A - G["A"]).max() <= 1e-13 * np.abs(G["A"]).max()
    x, it, _, _ = O.pcg(A, G["b"], tol=1e-10, max_iter=10 ** 5)
    assert it == 25 == int(G["iters"])


def test_oracle_c2_rows():
    from paper_1708_03912_b200 import mesh as M
    G = golden("c2")
    mesh = make_mesh("graded1d", 8192)
    dm = M.DofMap(mesh, 0.75)
    rows = G["rows_idx"][:6]
    R = O.assemble_rows(mesh, dm, 0.75, rows)
    assert np.abs(R - G["rows"][:6]).max() <= 1e-13 * float(G["maxabs"])
    assert np.allclose(O.load_vector(mesh, dm), G["b"], rtol=1e-14, atol=1e-18)


@pytest.mark.slow
def test_oracle_c3_rows():
    from paper_1708_03912_b200 import mesh as M
    G = golden("c3")
    mesh = make_mesh("square2d", 64)
    dm = M.DofMap(mesh, 0.5)
    rows = G["rows_idx"][:4]
    R = O.assemble_rows(mesh, dm, 0.5, rows)
    assert np.abs(R - G["rows"][:4]).max() <= 1e-13 * float(G["maxabs"])


def test_oracle_orders_c1():
    """Per-pair orders of the oracle == the reference's (hash of the nc x nc order matrix)."""
    from dataclasses import replace
    from paper_1708_03912_b200 import mesh as M
    G = golden("c1")
    mesh = make_mesh("uniform1d", 512)
    dm = M.DofMap(mesh, 0.25)
    g = O.Geo(mesh, dm, 0.25)
    p = O.Params()
    nc = g.nc
    Kc = np.zeros((nc, nc), np.int8)
    Kt = np.zeros((nc, nc), np.int8)
    hi = replace(p, C_offset=p.C_offset - 4)
    for K in range(nc):
        keep = np.ones(nc, bool)
        keep[g.neigh(K)] = False
        src = np.nonzero(keep)[0]
        tgt = np.full(len(src), K)
        dist = g.dist(tgt, src)
        Kt[K, src] = O.order_far(g.h[tgt], g.h[src], np.maximum(dist, 1e-300), g.n, 0.25, 1, hi)
        up = src[src > K]
        t2 = np.full(len(up), K)
        Kc[K, up] = O.order_far(g.h[t2], g.h[up], np.maximum(g.dist(t2, up), 1e-300), g.n, 0.25, 1, p)
    assert hashlib.sha256(Kc.tobytes()).hexdigest() == str(G["cross_sha"])
    assert hashlib.sha256(Kt.tobytes()).hexdigest() == str(G["tail_sha"])


def test_normalisation_known_answers():
    # SPEC.md:212-215
    from paper_1708_03912_b200.assembly import normalisation
    assert abs(normalisation(1, 0.5) - 1 / np.pi) < 1e-15
    assert abs(normalisation(2, 0.5) - 1 / (2 * np.pi)) < 1e-15
    assert abs(O.normalisation(2, 0.5) - 1 / (2 * np.pi)) < 1e-15
    G = golden("tables")
    for d, s, c in G["normalisation"]:
        assert normalisation(int(d), s) == c
    with pytest.raises(ValueError):
        normalisation(1, 1.0)


@pytest.mark.parametrize("key,s", irregular_cases())
def test_oracle_irregular_meshes(key, s):
    """Jittered + relabelled 2D triangulations and shuffled random 1D partitions (the reference's
    own _finish_polygon_mesh orientation): full A, b and the CG solution."""
    from paper_1708_03912_b200 import mesh as M
    G = golden("irregular")
    mesh = irregular_mesh(key)
    dm = M.DofMap(mesh, s)
    A = O.assemble_dense(mesh, dm, s)
    Ar = G[key + "/A"]
    assert np.abs(A - Ar).max() <= 1e-13 * np.abs(Ar).max()
    b = O.load_vector(mesh, dm)
    assert np.allclose(b, G[key + "/b"], rtol=1e-14, atol=1e-16)


@pytest.mark.parametrize("key,kind,N,s", tiny_cases())
def test_oracle_tiny_and_generic_s(key, kind, N, s):
    """n = 1, 2 meshes and exponents outside {1/4, 1/2, 3/4} (the generic-power path)."""
    from paper_1708_03912_b200 import mesh as M
    G = golden("tiny")
    mesh = make_mesh(kind, N)
    dm = M.DofMap(mesh, s)
    A = O.assemble_dense(mesh, dm, s)
    Ar = G[key + "/A"]
    assert A.shape == Ar.shape
    assert np.abs(A - Ar).max() <= 1e-13 * np.abs(Ar).max()
