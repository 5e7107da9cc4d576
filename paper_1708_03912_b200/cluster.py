"""Cluster tree, admissible partition and the near-field leaf-pair structure — the host-side
control of the reference's cluster path (cluster.py:25-255, :743-777) that decides which DoF
pairs `assemble_near_field` assembles.  Pure bookkeeping over O(n log n) boxes; the assembly
itself runs on the GPU (assembly.assemble_near_field -> fl_assemble_near_field).

Node numbering, DoF permutation, leaf order and pair order follow the reference exactly (a
depth-first bisection that creates both children when a node is split and then descends into
the second child first), so a NearStructure built here and one built by the reference describe
the same leaves and pairs.  Any object with the same attributes (e.g. the reference's own
NearStructure) is accepted by assemble_near_field (duck typing, like the reference).
"""
from __future__ import annotations

import numpy as np


class ClusterTree:
    """Binary tree over DoFs; node k owns dof_perm[ranges[k][0]:ranges[k][1]] (cluster.py:25-117)."""

    def __init__(self, mesh, dofmap, leaf_cap):
        self.mesh = mesh
        self.dofmap = dofmap
        self.leaf_cap = int(leaf_cap)
        d = mesh.vertices.shape[1]
        n = int(dofmap.n)
        dofs = np.asarray(dofmap.dofs)
        pos = mesh.vertices[dofs]
        # support box of every DoF: bounding box of the cells around its vertex
        cells = np.asarray(mesh.cells)
        P = mesh.vertices[cells]                                   # (nc, d+1, d)
        clo, chi = P.min(axis=1), P.max(axis=1)
        flat = cells.ravel()
        owner = np.repeat(np.arange(len(cells)), cells.shape[1])
        vlo = np.full((mesh.vertices.shape[0], d), np.inf)
        vhi = np.full((mesh.vertices.shape[0], d), -np.inf)
        np.minimum.at(vlo, flat, clo[owner])
        np.maximum.at(vhi, flat, chi[owner])
        lo, hi = vlo[dofs], vhi[dofs]
        self.dof_perm = np.arange(n)
        self.ranges, self.children, self.parent, center, half = [], [], [], [], []

        def new_node(a, b, par):
            sel = self.dof_perm[a:b]
            l, h = lo[sel].min(axis=0), hi[sel].max(axis=0)
            self.ranges.append((a, b))
            self.children.append([])
            self.parent.append(par)
            center.append(0.5 * (l + h))
            half.append(0.5 * float((h - l).max()))
            return len(self.ranges) - 1

        todo = [new_node(0, n, -1)]
        while todo:
            node = todo.pop()
            a, b = self.ranges[node]
            if b - a <= self.leaf_cap:
                continue
            sel = self.dof_perm[a:b]
            pts = pos[sel]
            axis = int(np.argmax(pts.max(axis=0) - pts.min(axis=0)))
            coord = pts[:, axis]
            left = coord <= 0.5 * (coord.max() + coord.min())
            if left.all() or not left.any():           # degenerate cut: median split
                left = np.zeros(b - a, bool)
                left[np.argsort(coord, kind="stable")[:(b - a) // 2]] = True
            self.dof_perm[a:b] = np.concatenate([sel[left], sel[~left]])
            mid = a + int(left.sum())
            kids = [new_node(a, mid, node), new_node(mid, b, node)]
            self.children[node] = kids
            todo.extend(kids)
        self.center = np.asarray(center)
        self.half = np.asarray(half)
        self.num_nodes = len(self.ranges)
        self.leaves = [k for k in range(self.num_nodes) if not self.children[k]]
        self.leaf_id = {nd: k for k, nd in enumerate(self.leaves)}
        self.leaf_of_dof = np.empty(n, np.int64)
        for nd in self.leaves:
            a, b = self.ranges[nd]
            self.leaf_of_dof[self.dof_perm[a:b]] = nd
        self.depth = np.zeros(self.num_nodes, np.int64)
        order = [0]
        for nd in order:
            for c in self.children[nd]:
                self.depth[c] = self.depth[nd] + 1
                order.append(c)
        self.topo_order = order

    def node_dofs(self, nd):
        a, b = self.ranges[nd]
        return self.dof_perm[a:b]

    def diam(self, nd):
        return 2.0 * self.half[nd] * np.sqrt(self.mesh.vertices.shape[1])

    def dist(self, a, b):
        gap = np.abs(self.center[a] - self.center[b]) - (self.half[a] + self.half[b])
        return float(np.linalg.norm(np.maximum(gap, 0.0)))


def build_tree(mesh, dofmap, leaf_cap: int) -> ClusterTree:
    """cluster.py:195-198."""
    if leaf_cap < 1:
        raise ValueError("leaf_cap must be >= 1")
    return ClusterTree(mesh, dofmap, leaf_cap)


def admissible_partition(tree: ClusterTree, eta: float):
    """Far / near node pairs by recursive descent from (root, root) (cluster.py:201-227):
    (a, b) is far when a != b and eta * dist >= max(diam); two leaves that are not far are near;
    otherwise the larger box is split (equal boxes: the lower node id)."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    far, near = [], []
    todo = [(0, 0)]
    while todo:
        a, b = todo.pop()
        if a != b and eta * tree.dist(a, b) >= max(tree.diam(a), tree.diam(b)):
            far.append((a, b))
            continue
        ka, kb = tree.children[a], tree.children[b]
        if not ka and not kb:
            near.append((a, b))
            continue
        ha, hb = tree.half[a], tree.half[b]
        split_a = bool(ka) and (not kb or ha > hb * (1 + 1e-12) or (abs(ha - hb) <= 1e-12 * ha and a <= b))
        todo.extend([(c, b) for c in ka] if split_a else [(a, c) for c in kb])
    return far, near


class NearStructure:
    """Near leaf pairs handed to assemble_near_field (cluster.py:743-777)."""

    def __init__(self, mesh, dofmap, tree, near_pairs):
        self.tree = tree
        self.leaf_of_dof = tree.leaf_of_dof
        keys = sorted({(min(a, b), max(a, b)) for a, b in near_pairs})
        self.nl_pairs = np.asarray(keys, np.int64).reshape(-1, 2)
        offs, pdata = mesh.patch_arrays()
        dofs = np.asarray(dofmap.dofs)
        self.leaf_cells = {}
        for nd in tree.leaves:
            vs = dofs[tree.node_dofs(nd)]
            parts = [pdata[offs[v]:offs[v + 1]] for v in vs]
            self.leaf_cells[nd] = np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
        nbr = {}
        for a, b in self.nl_pairs:
            nbr.setdefault(int(a), set()).add(int(b))
            nbr.setdefault(int(b), set()).add(int(a))
        self.near_leaf_map = {k: np.asarray(sorted(v), np.int64) for k, v in nbr.items()}
        self.leaf_index = {nd: k for k, nd in enumerate(tree.leaves)}
        nl = len(tree.leaves)
        self.mask = np.zeros((nl, nl), dtype=bool)
        if len(self.nl_pairs):
            ia = np.array([self.leaf_index[int(a)] for a in self.nl_pairs[:, 0]])
            ib = np.array([self.leaf_index[int(b)] for b in self.nl_pairs[:, 1]])
            self.mask[ia, ib] = True
            self.mask[ib, ia] = True
        self.leaf_idx_of_dof = np.empty(int(dofmap.n), np.int64)
        for nd in tree.leaves:
            self.leaf_idx_of_dof[tree.node_dofs(nd)] = self.leaf_index[nd]

    def near_mask(self, I, J):
        return self.mask[self.leaf_idx_of_dof[I], self.leaf_idx_of_dof[J]]
