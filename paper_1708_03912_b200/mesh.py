"""Mesh / DofMap input contract and the BASELINE mesh builders.

Mirrors `fraclap.mesh` (reference mesh.py) for what the dense path reads: vertices,
cells, boundary edges with OUTWARD unit normals, vertex patches, cell diameters, and
the DoF rule of DofMap (mesh.py:200-240: all vertices for s < 1/2, interior ones else).
Any object with the same attributes (e.g. a reference `fraclap.mesh.Mesh`) is accepted
by the assembly entry points (duck typing, like the reference).

Builders for the BASELINE.json meshes (all host-side, O(n)):
  build_interval_mesh        uniform 1D (mesh.py:273-280)
  build_graded_interval_mesh x = sign(t)(1-(1-|t|)^2), t uniform (config 2)
  build_unit_square_mesh     N x N squares split along the SW-NE diagonal, finished by the
                             same CCW / longest-edge-first rule as _finish_polygon_mesh
                             (mesh.py:351-403) (configs 3-5)
"""
from __future__ import annotations

import numpy as np


class MeshError(ValueError):
    """mesh.py:20."""


class Mesh:
    """Conforming simplicial mesh (intervals or triangles), mesh.py:24-197 (subset)."""

    def __init__(self, vertices, cells, boundary_edges, boundary_normals):
        self.vertices = np.ascontiguousarray(vertices, dtype=float)
        self.cells = np.ascontiguousarray(cells, dtype=np.int64)
        self.boundary_edges = np.ascontiguousarray(boundary_edges, dtype=np.int64)
        self.boundary_normals = np.ascontiguousarray(boundary_normals, dtype=float)
        self.d = self.vertices.shape[1]
        self._patches = None
        self._diams = None

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_cells(self):
        return len(self.cells)

    def cell_coords(self, idx=None):
        return self.vertices[self.cells if idx is None else self.cells[idx]]

    def cell_diameters(self):
        if self._diams is None:
            P = self.cell_coords()
            if self.d == 1:
                self._diams = np.abs(P[:, 1, 0] - P[:, 0, 0])
            else:
                e = [np.linalg.norm(P[:, (i + 1) % 3] - P[:, i], axis=1) for i in range(3)]
                self._diams = np.maximum(e[0], np.maximum(e[1], e[2]))
        return self._diams

    def cell_volumes(self):
        P = self.cell_coords()
        if self.d == 1:
            return np.abs(P[:, 1, 0] - P[:, 0, 0])
        a, b = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
        return 0.5 * np.abs(a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0])

    def boundary_vertex_mask(self):
        m = np.zeros(self.num_vertices, dtype=bool)
        m[self.boundary_edges.ravel()] = True
        return m

    def patch_arrays(self):
        """CSR (offsets, cell ids) of vertex -> cells, ascending cell ids (mesh.py:114-130)."""
        if self._patches is None:
            flat = self.cells.ravel()
            order = np.argsort(flat, kind="stable")
            data = np.repeat(np.arange(self.num_cells), self.cells.shape[1])[order]
            offs = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=self.num_vertices))])
            self._patches = (offs, data)
        return self._patches


class DofMap:
    """DoF enumeration (mesh.py:200-240, without the `identify` sector option)."""

    def __init__(self, mesh, s: float):
        if not 0.0 < s < 1.0:
            raise ValueError("fractional order s must lie in (0,1)")
        self.mesh = mesh
        self.s = s
        nv = mesh.num_vertices
        bmask = np.zeros(nv, dtype=bool)
        bmask[np.asarray(mesh.boundary_edges).ravel()] = True
        take = np.ones(nv, dtype=bool) if s < 0.5 else ~bmask
        self.dofs = np.nonzero(take)[0]
        self.vertex_to_dof = np.full(nv, -1, dtype=np.int64)
        self.vertex_to_dof[self.dofs] = np.arange(len(self.dofs))
        self.cell_dofs = self.vertex_to_dof[mesh.cells]

    @property
    def n(self):
        return len(self.dofs)

    def dof_coords(self):
        return self.mesh.vertices[self.dofs]


# ------------------------------------------------------------------ builders
def build_interval_mesh(a: float, b: float, n_cells: int) -> Mesh:
    """Uniform mesh of (a, b) (mesh.py:273-280)."""
    if not (a < b) or n_cells < 1:
        raise MeshError("need a < b and n_cells >= 1")
    x = np.linspace(a, b, n_cells + 1)
    cells = np.stack([np.arange(n_cells), np.arange(1, n_cells + 1)], axis=1)
    return Mesh(x[:, None], cells, np.array([[0], [n_cells]]), np.array([[-1.0], [1.0]]))


def build_graded_interval_mesh(n_cells: int) -> Mesh:
    """(-1, 1) graded toward +-1: x_i = sign(t_i)(1 - (1 - |t_i|)^2), t uniform (BASELINE c2)."""
    if n_cells < 1:
        raise MeshError("need n_cells >= 1")
    t = np.linspace(-1.0, 1.0, n_cells + 1)
    x = np.sign(t) * (1.0 - (1.0 - np.abs(t)) ** 2)
    cells = np.stack([np.arange(n_cells), np.arange(1, n_cells + 1)], axis=1)
    return Mesh(x[:, None], cells, np.array([[0], [n_cells]]), np.array([[-1.0], [1.0]]))


def finish_polygon_mesh(vertices, cells) -> Mesh:
    """CCW orientation, refinement (longest) edge first with a vertex-pair tie break, and the
    boundary edges with outward normals — the rule of _finish_polygon_mesh (mesh.py:351-403)."""
    V = np.asarray(vertices, float)
    C = np.array(cells, np.int64)
    a = V[C[:, 1]] - V[C[:, 0]]
    b = V[C[:, 2]] - V[C[:, 0]]
    cw = (a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]) < 0
    C[cw] = C[cw][:, [0, 2, 1]]
    P = V[C]
    lens = np.stack([np.linalg.norm(P[:, (i + 1) % 3] - P[:, i], axis=1) for i in range(3)], axis=1)
    nxt = np.roll(C, -1, axis=1)
    lo, hi = np.minimum(C, nxt), np.maximum(C, nxt)
    nv = len(V)
    key = np.round(lens / lens.max(), 12) * (nv * nv * 4.0) + lo * (2.0 * nv) + hi
    first = np.argmax(key, axis=1)
    C = np.take_along_axis(C, (first[:, None] + np.arange(3)[None, :]) % 3, axis=1)
    # boundary edges: undirected edges used by exactly one cell, sorted lexicographically
    raw = np.concatenate([C[:, [0, 1]], C[:, [1, 2]], C[:, [2, 0]]])
    key2 = np.sort(raw, axis=1)
    uniq, inv, cnt = np.unique(key2, axis=0, return_inverse=True, return_counts=True)
    inv = inv.reshape(3, -1).T
    owner = np.full(len(uniq), -1, np.int64)
    for loc in range(3):
        owner[inv[:, loc]] = np.arange(len(C))
    bidx = np.nonzero(cnt == 1)[0]
    be = uniq[bidx]
    p, q = V[be[:, 0]], V[be[:, 1]]
    t = q - p
    nrm = np.stack([t[:, 1], -t[:, 0]], axis=1)
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    cen = V[C[owner[bidx]]].mean(axis=1)
    flip = np.einsum("ij,ij->i", 0.5 * (p + q) - cen, nrm) < 0
    nrm[flip] = -nrm[flip]
    return Mesh(V, C, be, nrm)


def finish_polygon_mesh_device(vertices, cells, device=0) -> Mesh:
    """finish_polygon_mesh on the GPU (fl_finish_polygon_mesh; same rule, mesh.py:351-403)."""
    import ctypes as C
    from . import _lib
    V = np.ascontiguousarray(vertices, dtype=np.float64)
    Cin = np.ascontiguousarray(cells, dtype=np.int64)
    nc = len(Cin)
    Cout = np.empty((nc, 3), np.int64)
    be = np.empty((3 * nc, 2), np.int64)
    bn = np.empty((3 * nc, 2))
    nb = C.c_int64()
    _lib.check(_lib.load().fl_finish_polygon_mesh(V.ctypes.data, len(V), Cin.ctypes.data, nc, int(device),
                                                  Cout.ctypes.data, be.ctypes.data, bn.ctypes.data, 3 * nc,
                                                  C.byref(nb)))
    return Mesh(V, Cout, be[:nb.value].copy(), bn[:nb.value].copy())


def dofmap_device(mesh, s: float, device=0) -> DofMap:
    """DofMap built on the GPU (fl_build_dofmap; mesh.py:200-240)."""
    import ctypes as C
    from . import _lib
    if not 0.0 < s < 1.0:
        raise ValueError("fractional order s must lie in (0,1)")
    m = _lib.Marshal(mesh, _NoDofs(mesh.num_vertices), _Kernel(mesh.vertices.shape[1], s), None)
    v2d = np.empty(mesh.num_vertices, np.int64)
    n = C.c_int64()
    _lib.check(_lib.load().fl_build_dofmap(C.byref(m.mesh), float(s), int(device), v2d.ctypes.data, C.byref(n)))
    dm = DofMap.__new__(DofMap)
    dm.mesh, dm.s = mesh, s
    dm.vertex_to_dof = v2d
    dm.dofs = np.nonzero(v2d >= 0)[0]
    dm.cell_dofs = v2d[mesh.cells]
    assert len(dm.dofs) == n.value
    return dm


class _NoDofs:
    def __init__(self, nv):
        self.n = 0
        self.vertex_to_dof = np.full(nv, -1, np.int64)


class _Kernel:
    def __init__(self, d, s):
        self.d, self.s, self.C_ds, self.variant = d, s, 1.0, "integral"


def build_unit_square_mesh(N: int) -> Mesh:
    """[0,1]^2 with N x N squares, each split by its SW-NE diagonal (BASELINE c3-c5).
    Vertex (i, j) at (i/N, j/N) has index j*(N+1)+i; square (i, j) gives (SW, SE, NE) and
    (SW, NE, NW), squares row by row."""
    if N < 1:
        raise MeshError("need N >= 1")
    g = np.linspace(0.0, 1.0, N + 1)
    X, Y = np.meshgrid(g, g, indexing="xy")
    V = np.stack([X.ravel(), Y.ravel()], axis=1)
    j, i = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    sw = (j * (N + 1) + i).ravel()
    se, nw = sw + 1, sw + N + 1
    ne = nw + 1
    tris = np.empty((2 * N * N, 3), np.int64)
    tris[0::2] = np.stack([sw, se, ne], axis=1)
    tris[1::2] = np.stack([sw, ne, nw], axis=1)
    return finish_polygon_mesh(V, tris)


def baseline_mesh(name: str):
    """(mesh, s) of a BASELINE.json config: c1..c5 (c4a/c4b: s = 0.25 / 0.75)."""
    table = {
        "c1": (lambda: build_interval_mesh(-1.0, 1.0, 512), 0.25),
        "c2": (lambda: build_graded_interval_mesh(8192), 0.75),
        "c3": (lambda: build_unit_square_mesh(64), 0.5),
        "c4a": (lambda: build_unit_square_mesh(128), 0.25),
        "c4b": (lambda: build_unit_square_mesh(128), 0.75),
        "c5": (lambda: build_unit_square_mesh(256), 0.5),
    }
    f, s = table[name]
    return f(), s
