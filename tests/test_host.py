"""Host-side logic on CPU: mesh builders vs the reference's meshes, DofMap rule, load
vector, and the C ABI library (loads and exports every symbol the header declares)."""
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, make_mesh
from paper_1708_03912_b200 import mesh as M


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4a", "c5"])
def test_baseline_meshes_match_reference(name):
    G = golden("meshes")
    mesh, s = M.baseline_mesh(name)
    assert _sha(mesh.cells) == G[name + "/cells_sha"].tobytes()
    assert _sha(mesh.vertices) == G[name + "/verts_sha"].tobytes()
    assert _sha(mesh.boundary_edges) == G[name + "/bedges_sha"].tobytes()
    assert _sha(mesh.boundary_normals) == G[name + "/bnormals_sha"].tobytes()
    nv, nc, nb, n = G[name + "/counts"]
    assert (mesh.num_vertices, mesh.num_cells, len(mesh.boundary_edges), M.DofMap(mesh, s).n) == (nv, nc, nb, n)


def test_dof_rule():
    # mesh.py:225: s < 1/2 keeps the boundary vertices (c1: n = 513, not 511)
    mesh = M.build_interval_mesh(-1, 1, 512)
    assert M.DofMap(mesh, 0.25).n == 513
    assert M.DofMap(mesh, 0.5).n == 511
    sq = M.build_unit_square_mesh(128)
    assert M.DofMap(sq, 0.25).n == 16641 and M.DofMap(sq, 0.75).n == 16129
    with pytest.raises(ValueError):
        M.DofMap(mesh, 1.5)


def test_library_exports_header_symbols():
    from paper_1708_03912_b200 import _lib
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "fraclap_b200.h")).read()
    declared = set(re.findall(r"\b(fl_[a-z_0-9]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == declared
    assert lib.fl_abi_version() == 1


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1708_03912_b200", "lib", "libfraclap_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_no_oracle_in_product():
    """The product package never imports the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_1708_03912_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
