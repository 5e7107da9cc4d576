"""Residual error estimation of the adaptive loop on the GPU:
strong_form_at (adapt.py:81-214) — (-Delta)^s u_h at per-cell nodes through the cluster far field
plus near surface terms — and residual_norms / indicators / mark_maximum (:237-291) around it.

The heavy part (far-field evaluation at every node, surface integrals over the near cells of
the owning leaf and over the point's own cell) runs in fl_cluster_strong_form on the operator a
ClusterOperatorDevice holds; the bookkeeping here (cell -> leaf assignment, near-cell lists per
leaf) restates the reference's host logic."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .quadrature import gauss_legendre, simplex_rule

LOG_CASE_TOL = 1e-12      # adapt.py:25


def cell_leaf_assignment(mesh, dofmap, leaf_of_dof):
    """Leaf node of every cell: the leaf of its first DoF, else of the DoF nearest to its
    centroid (_cell_leaf_assignment, cluster.py:496-508)."""
    cd = np.asarray(dofmap.vertex_to_dof)[np.asarray(mesh.cells)]
    first = np.full(mesh.num_cells, -1, np.int64)
    for loc in range(cd.shape[1]):
        first = np.where((first < 0) & (cd[:, loc] >= 0), cd[:, loc], first)
    missing = np.nonzero(first < 0)[0]
    if len(missing):
        from scipy.spatial import cKDTree
        kd = cKDTree(mesh.vertices[np.asarray(dofmap.dofs)])
        _, nearest = kd.query(mesh.vertices[np.asarray(mesh.cells)[missing]].mean(axis=1))
        first[missing] = nearest
    return np.asarray(leaf_of_dof)[first]


def _near_csr(mesh, dofmap, num_nodes, node_dofs, near_leaf_map):
    """Per node (CSR): its near leaf nodes (default: itself, adapt.py:126) and the cells
    supporting their DoFs (adapt.py:127-133)."""
    offs, pdata = mesh.patch_arrays()
    dofs = np.asarray(dofmap.dofs)
    noff, nval, coff, cval = [0], [], [0], []
    for nd in range(num_nodes):
        leaves = np.asarray(near_leaf_map.get(nd, [nd]), np.int64)
        nval.extend(sorted(leaves.tolist()))
        noff.append(len(nval))
        verts = dofs[np.concatenate([node_dofs(l) for l in leaves])] if len(leaves) else np.zeros(0, np.int64)
        cells = np.unique(np.concatenate([pdata[offs[v]:offs[v + 1]] for v in verts])) if len(verts) else []
        cval.extend(np.asarray(cells, np.int64).tolist())
        coff.append(len(cval))
    a = lambda x: np.ascontiguousarray(x, dtype=np.int64)   # noqa: E731
    return a(noff), a(nval if nval else [0]), a(coff), a(cval if cval else [0])


def cell_nodes(mesh, order):
    """(X (nc, q, d), W (nc, q)) of the per-cell rule of `order` (cell_quadrature, assembly.py:290-298):
    nodes mapped on the device (fl_cell_rule_nodes), weights |det| w."""
    d = mesh.vertices.shape[1]
    pts, w = simplex_rule(d, order)
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    from .assembly import FractionalKernel, _device_index
    from .mesh import _NoDofs
    m = _lib.Marshal(mesh, _NoDofs(mesh.num_vertices), FractionalKernel(d, 0.5), None)
    X = np.empty((mesh.num_cells, len(w), d))
    _lib.check(_lib.load().fl_cell_rule_nodes(C.byref(m.mesh), pts.ctypes.data, len(w), _device_index(None),
                                              X.ctypes.data))
    P = mesh.vertices[mesh.cells]
    if d == 1:
        J = np.abs(P[:, 1, 0] - P[:, 0, 0])
    else:
        a, b = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
        J = np.abs(a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0])
    return X, np.outer(J, w)


def strong_form_at(u, mesh, dofmap, op, X=None, edge_order=6, return_far=False):
    """(-Delta)^s u_h at per-cell nodes X (nc, q, d) (adapt.strong_form_at, adapt.py:81-214) on the GPU.
    `op`: a cluster.ClusterOperatorDevice built with the tree / near-leaf information."""
    if op.tree_info is None:
        raise ValueError("strong_form_at needs a ClusterOperatorDevice built with its tree information")
    s = float(op.s)
    d = mesh.vertices.shape[1]
    if X is None:
        X, _ = cell_nodes(mesh, 4)
    X = np.ascontiguousarray(X, dtype=np.float64)
    nc, q, _ = X.shape
    ti = op.tree_info
    if "csr" not in ti:
        ti["csr"] = _near_csr(mesh, dofmap, ti["num_nodes"], ti["node_dofs"], ti["near_leaf_map"])
    if "cell_leaf" not in ti:
        ti["cell_leaf"] = np.ascontiguousarray(cell_leaf_assignment(mesh, dofmap, ti["leaf_of_dof"]), np.int64)
    noff, nval, coff, cval = ti["csr"]
    gx, gw = gauss_legendre(edge_order)
    gx, gw = np.ascontiguousarray(gx, np.float64), np.ascontiguousarray(gw, np.float64)
    from .assembly import FractionalKernel
    m = _lib.Marshal(mesh, dofmap, FractionalKernel(d, s), None)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty((nc, q))
    far = np.empty((nc, q))
    _lib.check(_lib.load().fl_cluster_strong_form(op.handle, C.byref(m.mesh), C.byref(m.dofmap), s, u.ctypes.data, q,
                                                  X.ctypes.data, ti["cell_leaf"].ctypes.data, noff.ctypes.data,
                                                  nval.ctypes.data, coff.ctypes.data, cval.ctypes.data,
                                                  gx.ctypes.data, gw.ctypes.data, len(gx), out.ctypes.data,
                                                  far.ctypes.data))
    return (out, far) if return_far else out


def residual_norms(u, f, mesh, dofmap, op, order=4, edge_order=6):
    """Per-cell L2 norms of r = f - (-Delta)^s u_h (adapt.py:237-243)."""
    X, W = cell_nodes(mesh, order)
    sf = strong_form_at(u, mesh, dofmap, op, X=X, edge_order=edge_order)
    d = mesh.vertices.shape[1]
    fv = np.asarray(f(X.reshape(-1, d))).reshape(X.shape[:2])
    return np.sqrt(np.sum(W * (fv - sf) ** 2, axis=1))


class Indicators:
    """adapt.py:28-35."""

    def __init__(self, per_node, dof_vertices):
        self.per_node = np.asarray(per_node, float)
        self.dof_vertices = np.asarray(dof_vertices)
        self.total = float(np.sqrt(np.sum(self.per_node ** 2)))

    def __len__(self):
        return len(self.per_node)


def indicators(res_norms, mesh, dofmap):
    """eta_i = sqrt(sum_{K in patch(i)} h_K^{2s} ||r||_K^2) (adapt.py:246-255)."""
    h2s = mesh.cell_diameters() ** (2 * dofmap.s)
    wsq = h2s * np.asarray(res_norms) ** 2
    offs, pdata = mesh.patch_arrays()
    vals = np.array([np.sqrt(np.sum(wsq[pdata[offs[v]:offs[v + 1]]])) for v in np.asarray(dofmap.dofs)])
    return Indicators(vals, dofmap.dofs)


def mark_maximum(ind, theta, mesh, dofmap):
    """Cells in the patch of every node whose indicator reaches theta * max (adapt.py:258-269)."""
    if not 0 < theta <= 1:
        raise ValueError("theta must lie in (0, 1]")
    if ind.total == 0:
        return np.zeros(0, np.int64)
    chosen = ind.dof_vertices[ind.per_node >= theta * ind.per_node.max()]
    offs, pdata = mesh.patch_arrays()
    return np.unique(np.concatenate([pdata[offs[v]:offs[v + 1]] for v in chosen]))
