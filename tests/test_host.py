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


def test_assembly_stats_layout_matches_header():
    """The ctypes mirror of fl_assembly_stats has the header's fields, types and order."""
    from paper_1708_03912_b200 import _lib
    src = open(os.path.join(ROOT, "include", "fraclap_b200.h")).read()
    body = re.search(r"typedef struct fl_assembly_stats \{(.*?)\} fl_assembly_stats;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        ctype, names = decl.split(None, 1)
        fields += [(n.strip(), ctype) for n in names.split(",")]
    cmap = {"int64_t": ctypes.c_int64, "int32_t": ctypes.c_int32, "double": ctypes.c_double}
    st = [c for c in vars(_lib).values() if isinstance(c, type) and issubclass(c, ctypes.Structure)
          and [f[0] for f in c._fields_][:2] == ["pairs_identical", "pairs_touching"]]
    assert len(st) == 1
    got = [(n, t) for n, t in st[0]._fields_]
    assert [n for n, _ in got] == [n for n, _ in fields]
    assert all(t == cmap[c] for (_, t), (_, c) in zip(got, fields))


def test_bench_rooflines_and_pair_count():
    """bench.py's pure pieces: the element-pair count and the per-kernel rooflines (the order-4
    evaluations serving both directions add their partner accumulation)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    st = dict(pairs_identical=1, pairs_touching=2, pairs_cross=3, pairs_tail=4, pairs_boundary_singular=5,
              pairs_boundary_flux=6, ms_tail=2.0, evals_tail=3e9, ms_tail_block=1.0, evals_tail_block=2e9,
              evals_tail_sym=1e9, ms_cross=1.0, ms_cross_compute=0.5, evals_cross=1e9, evals_near=2e8, ms_near=0.1)
    assert B.pair_count(st) == 21
    r = B.roofline_of(st, 2, 0.5, 30.0, "tail_block")
    assert r["kernel"] == "tail2d_block_kernel" and r["flops_per_eval"] == 16
    assert abs(r["achieved"] - (2e9 * 16 + 2 * 1e9) / 1e-3 / 1e12) < 1e-9
    assert r["reference_equivalent_evals"] == 3e9
    rp = B.roofline_of(st, 2, 0.5, 30.0, "tail_pairs")
    assert rp["evals_per_launch"] == 1e9 and rp["ms_per_launch"] == 1.0
    rc = B.roofline_of(st, 2, 0.5, 30.0, "cross_far")
    assert rc["evals_per_launch"] == 8e8 and rc["flops_per_eval"] == 20
