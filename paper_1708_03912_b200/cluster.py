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

import math

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
    # scalar fast path: the gap is the reference's elementwise float64 arithmetic; only the norm
    # may differ from np.linalg.norm in the last ulp, so near-ties re-check with tree.dist
    cen = [tuple(float(v) for v in row) for row in np.asarray(tree.center).reshape(tree.num_nodes, -1)]
    half = [float(v) for v in tree.half]
    diam = [float(tree.diam(nd)) for nd in range(tree.num_nodes)]
    todo = [(0, 0)]
    while todo:
        a, b = todo.pop()
        if a != b:
            hab = half[a] + half[b]
            d2 = 0.0
            for ca, cb in zip(cen[a], cen[b]):
                g = abs(ca - cb) - hab
                if g > 0.0:
                    d2 += g * g
            lhs, rhs = eta * math.sqrt(d2), max(diam[a], diam[b])
            if abs(lhs - rhs) <= 1e-12 * rhs:
                lhs = eta * tree.dist(a, b)
            if lhs >= rhs:
                far.append((a, b))
                continue
        ka, kb = tree.children[a], tree.children[b]
        if not ka and not kb:
            near.append((a, b))
            continue
        ha, hb = half[a], half[b]
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


class ClusterOperatorDevice:
    """The cluster (H-matrix) stiffness operator with its matvec on the GPU (fl_cluster_*):
    ClusterOperator.matvec (cluster.py:417-456) = near CSR product + Chebyshev far field (leaf
    moments, upward shifts, far-pair blocks, downward shifts, leaf evaluation), in the
    reference's accumulation order.  Duck-types the reference's solver contract (`.matvec`,
    `.diag()`, `@`), so the reference's own pcg / multigrid can run on it.

    `from_operator(op)` wraps an operator built by the reference's `cluster.compress` (or any
    object with its attributes: tree, cheb, near, far_pairs, far_blocks, basis_coef, kernel)."""

    def __init__(self, handle, n, diag, d, M, s=None, tree_info=None, device=0):
        self._h = handle
        self.device = int(device)
        self.n = int(n)
        self._diag = diag
        self.d, self.M = d, M
        self.s = s
        self.tree_info = tree_info      # host tree data for adapt.strong_form_at (or None)
        self.shape = (self.n, self.n)
        self.dtype = np.float64

    @classmethod
    def from_arrays(cls, d, m, parent, topo_order, ranges, dof_perm, shift, basis_coef, far_pairs, far_blocks,
                    points, s, C_ds, near, diag=None, device=None, center=None, half=None, near_leaf_map=None):
        """`center`, `half` (tree boxes) and `near_leaf_map` (node -> near leaf nodes,
        ClusterOperator.near_dof_leaves) enable adapt.strong_form_at on this operator."""
        import ctypes as C
        from scipy.sparse import csr_matrix
        from . import _lib  # noqa: F811
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)           # noqa: E731
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)         # noqa: E731
        near = csr_matrix(near)
        near.sum_duplicates()
        n = near.shape[0]
        M = m ** d
        keep = dict(parent=i64(parent), topo=i64(topo_order), ranges=i64(ranges).reshape(-1, 2),
                    perm=i64(dof_perm), shift=f64(shift).reshape(-1, d, m, m), bc=f64(basis_coef).reshape(n, M),
                    pairs=i64(far_pairs).reshape(-1, 2), indptr=i64(near.indptr), indices=i64(near.indices),
                    data=f64(near.data))
        keep["blocks"] = None if far_blocks is None else f64(far_blocks).reshape(-1, M, M)
        keep["points"] = None if points is None else f64(points)
        have_boxes = center is not None and half is not None
        keep["center"] = f64(center).reshape(-1, d) if have_boxes else None
        keep["half"] = f64(half).reshape(-1) if have_boxes else None
        j = np.arange(m)
        keep["ref"] = f64(np.cos((2 * j + 1) * np.pi / (2 * m))) if have_boxes else None   # cheb_points_1d
        ptr = lambda a: None if a is None or a.size == 0 else a.ctypes.data   # noqa: E731
        desc = _lib.fl_cluster_desc(d, m, n, len(keep["parent"]), ptr(keep["parent"]), ptr(keep["topo"]),
                                    ptr(keep["ranges"]), ptr(keep["perm"]), ptr(keep["shift"]), ptr(keep["bc"]),
                                    len(keep["pairs"]), ptr(keep["pairs"]), ptr(keep["blocks"]), ptr(keep["points"]),
                                    float(s), float(C_ds), int(near.nnz), ptr(keep["indptr"]), ptr(keep["indices"]),
                                    ptr(keep["data"]), ptr(keep["center"]), ptr(keep["half"]), ptr(keep["ref"]))
        from .assembly import _device_index
        h = C.c_void_p()
        _lib.check(_lib.load().fl_cluster_create(C.byref(desc), _device_index(device), C.byref(h)))
        info = None
        if have_boxes and near_leaf_map is not None:
            rng, perm, par = keep["ranges"], keep["perm"], keep["parent"]
            nn = len(par)
            internal = np.zeros(nn, bool)
            internal[par[par >= 0]] = True
            leaf_of_dof = np.empty(n, np.int64)
            for nd in np.nonzero(~internal)[0]:
                leaf_of_dof[perm[rng[nd, 0]:rng[nd, 1]]] = nd
            info = {"num_nodes": nn, "node_dofs": lambda nd: perm[rng[nd, 0]:rng[nd, 1]],
                    "near_leaf_map": {int(k): np.asarray(v) for k, v in near_leaf_map.items()},
                    "leaf_of_dof": leaf_of_dof}
        return cls(h, n, near.diagonal().copy() if diag is None else np.asarray(diag, float), d, M, float(s), info,
                   device=_device_index(device))

    @classmethod
    def from_operator(cls, op, device=None, build_blocks_on_device=False):
        tree, cheb = op.tree, op.cheb
        d, m = int(cheb.d), int(cheb.m)
        nn = int(tree.num_nodes)
        shift = np.zeros((nn, d, m, m))
        for nd in range(nn):
            if cheb.shift[nd] is not None:
                for j in range(d):
                    shift[nd, j] = cheb.shift[nd][j]
        return cls.from_arrays(d, m, tree.parent, tree.topo_order, tree.ranges, tree.dof_perm, shift, op.basis_coef,
                               op.far_pairs, None if build_blocks_on_device else op.far_blocks, cheb.points,
                               op.kernel.s, op.kernel.C_ds, op.near, op.diag(), device, tree.center, tree.half,
                               op.near_dof_leaves())

    # ------------------------------------------------------------ contract
    def _apply(self, x, want_far=False):
        from . import _lib  # noqa: F811
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("dimension mismatch")
        y = np.empty(self.n)
        yf = np.empty(self.n) if want_far else None
        _lib.check(_lib.load().fl_cluster_matvec(self.handle, x.ctypes.data, y.ctypes.data,
                                                 None if yf is None else yf.ctypes.data, 0))
        return y, yf

    def matvec(self, x):
        return self._apply(x)[0]

    def far_apply(self, x):
        return self._apply(x, True)[1]

    def __matmul__(self, x):
        return self.matvec(x)

    def diag(self):
        return self._diag

    def evaluate_far_field_at_points(self, u, points, owner_leaves):
        """-C * int k(x, y) u_far(y) dy at points (cluster.py:469-485); owner_leaves = the leaf node
        owning each point."""
        from . import _lib  # noqa: F811
        pts = np.ascontiguousarray(np.asarray(points, float).reshape(-1, self.d))
        own = np.ascontiguousarray(owner_leaves, dtype=np.int64).reshape(-1)
        if len(own) != len(pts):
            raise ValueError("one owner leaf per point")
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(len(pts))
        _lib.check(_lib.load().fl_cluster_far_at_points(self.handle, u.ctypes.data, len(pts), pts.ctypes.data,
                                                        own.ctypes.data, out.ctypes.data))
        return out

    def memory_entries(self):
        """Stored entries: near nnz + far block entries (cluster.py:402-403)."""
        near = getattr(self, "near", None)
        npairs = len(getattr(self, "far_pairs", ()))
        return (near.nnz if near is not None else 0) + npairs * self.M * self.M

    def block_stats(self):
        """cluster.py:405-413."""
        near = getattr(self, "near", None)
        cheb = getattr(self, "cheb", None)
        return {"n": self.n, "near_nnz": int(near.nnz) if near is not None else 0,
                "far_blocks": int(len(getattr(self, "far_pairs", ()))), "block_size": int(self.M ** 2),
                "memory_entries": int(self.memory_entries()), "cheb_order": int(cheb.m) if cheb is not None else 0}

    def near_dof_leaves(self):
        """Leaf node -> its near leaf nodes (ClusterOperator.near_dof_leaves, cluster.py:487-489)."""
        if self.tree_info is None:
            raise ValueError("built without tree information")
        return self.tree_info["near_leaf_map"]

    def to_dense(self):
        """The operator as a dense (n, n) array (ClusterOperator.to_dense, cluster.py:460-467): the
        device matvec of every unit vector."""
        A = np.empty((self.n, self.n))
        e = np.zeros(self.n)
        for j in range(self.n):
            e[j] = 1.0
            A[:, j] = self.matvec(e)
            e[j] = 0.0
        return A

    def far_blocks(self, npairs):
        from . import _lib  # noqa: F811
        out = np.empty((int(npairs), self.M, self.M))
        _lib.check(_lib.load().fl_cluster_far_blocks(self.handle, out.ctypes.data))
        return out

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("operator already freed")
        return self._h

    def free(self):
        if self._h is not None and self._h.value:
            from . import _lib
            _lib.load().fl_cluster_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ------------------------------------------------------------------ Chebyshev data (host setup)
def cheb_points_1d(m):
    """cluster.py:271-273."""
    j = np.arange(m)
    return np.cos((2 * j + 1) * np.pi / (2 * m))


def lagrange_eval(ref_nodes, t):
    """Lagrange basis at the Chebyshev nodes evaluated at t (..., ) -> (..., m) (cluster.py:276-287):
    prod_{b != a} (t - x_b) / (x_a - x_b), the numerator as prefix x suffix products."""
    ref_nodes = np.asarray(ref_nodes, float)
    m = len(ref_nodes)
    t = np.asarray(t, float)
    diff = t[..., None] - ref_nodes
    pre = np.ones(t.shape + (m,))
    suf = np.ones(t.shape + (m,))
    if m > 1:
        pre[..., 1:] = np.cumprod(diff[..., :-1], axis=-1)
        suf[..., :-1] = np.cumprod(diff[..., :0:-1], axis=-1)[..., ::-1]
    return pre * suf / _lagrange_denominators(ref_nodes)


def _lagrange_denominators(ref_nodes):
    m = len(ref_nodes)
    return np.array([np.prod(ref_nodes[a] - ref_nodes[np.arange(m) != a]) for a in range(m)])


def choose_order(mesh_stats, tol=1e-6):
    """m = ceil(c0 + c1 |log h_min| + log3(1e-6 / tol)) clipped to [3, 12] (cluster.py:256-268)."""
    h_min = max(mesh_stats.h_min, 1e-300)
    c0, c1 = (2.4, 0.85) if getattr(mesh_stats, "dim", None) == 1 else (2.0, 0.55)
    m = c0 + c1 * abs(np.log(h_min)) + np.log(max(1e-6 / tol, 1.0)) / np.log(3.0)
    return int(np.clip(np.ceil(m), 3, 12))


class _Boxes:
    """Tensor Chebyshev points, parent shift matrices and basis evaluation over a tree of boxes
    (ChebData / ChebDataEdges, cluster.py:290-374, :596-664)."""

    def __init__(self, center, half, parent, order, d, m, half_floor=None):
        self.m, self.d, self.M = m, d, m ** d
        self.ref = cheb_points_1d(m)
        self.multi = np.arange(m)[:, None] if d == 1 else \
            np.stack([a.ravel() for a in np.meshgrid(np.arange(m), np.arange(m), indexing="ij")], axis=1)
        cen = np.asarray(center)
        half = np.asarray(half) if half_floor is None else np.maximum(np.asarray(half), half_floor)
        self.cen, self.half = cen, half
        pts1 = cen[:, None, :] + half[:, None, None] * self.ref[None, :, None]
        P = np.empty((len(cen), self.M, d))
        for j in range(d):
            P[:, :, j] = pts1[:, self.multi[:, j], j]
        self.points = P
        self.parent = np.asarray(parent)
        self.order = list(order)
        self.shift = [None] * len(cen)
        kids = np.asarray([nd for nd in self.order if self.parent[nd] >= 0], np.int64)
        if len(kids):
            par = self.parent[kids]
            T = (cen[kids, :, None] + half[kids, None, None] * self.ref - cen[par, :, None]) / half[par, None, None]
            L = np.swapaxes(lagrange_eval(self.ref, T), -1, -2)           # (kids, d, m, m)
            for i, nd in enumerate(kids):
                self.shift[nd] = [L[i, j] for j in range(d)]

    def eval_basis(self, nd, X):
        per = [lagrange_eval(self.ref, (X[..., j] - self.cen[nd][j]) / self.half[nd]) for j in range(self.d)]
        return per[0] if self.d == 1 else per[0][..., self.multi[:, 0]] * per[1][..., self.multi[:, 1]]

    def push_up(self, vals):
        for nd in reversed(self.order):
            par = self.parent[nd]
            if par < 0 or not np.any(vals[nd]):
                continue
            if self.d == 1:
                vals[par] += self.shift[nd][0] @ vals[nd]
            else:
                V = vals[nd].reshape(self.m, self.m)
                vals[par] += (self.shift[nd][0] @ V @ self.shift[nd][1].T).ravel()
        return vals

    def push_down(self, vals):
        for nd in self.order:
            par = self.parent[nd]
            if par < 0 or not np.any(vals[par]):
                continue
            if self.d == 1:
                vals[nd] += self.shift[nd][0].T @ vals[par]
            else:
                V = vals[par].reshape(self.m, self.m)
                vals[nd] += (self.shift[nd][0].T @ V @ self.shift[nd][1]).ravel()
        return vals


class EdgeTree:
    """Cluster tree over the boundary edges (boxes cover whole edges; cluster.py:120-192)."""

    def __init__(self, mesh, leaf_cap=8):
        d = mesh.vertices.shape[1]
        E = np.asarray(mesh.boundary_edges)
        if d == 1:
            lo = hi = pts = mesh.vertices[E[:, 0]]
        else:
            p0, p1 = mesh.vertices[E[:, 0]], mesh.vertices[E[:, 1]]
            lo, hi, pts = np.minimum(p0, p1), np.maximum(p0, p1), 0.5 * (p0 + p1)
        self.perm = np.arange(len(E))
        self.ranges, self.children, center, half = [], [], [], []

        def add(a, b):
            sel = self.perm[a:b]
            l, h = lo[sel].min(axis=0), hi[sel].max(axis=0)
            self.ranges.append((a, b))
            self.children.append([])
            center.append(0.5 * (l + h))
            half.append(0.5 * float((h - l).max()) if b > a else 0.0)
            return len(self.ranges) - 1

        todo = [add(0, len(E))]
        while todo:
            nd = todo.pop()
            a, b = self.ranges[nd]
            if b - a <= leaf_cap:
                continue
            sel = self.perm[a:b]
            P = pts[sel]
            axis = int(np.argmax(P.max(axis=0) - P.min(axis=0)))
            left = P[:, axis] <= 0.5 * (P[:, axis].max() + P[:, axis].min())
            if left.all() or not left.any():
                left = np.zeros(b - a, bool)
                left[np.argsort(P[:, axis], kind="stable")[:(b - a) // 2]] = True
            self.perm[a:b] = np.concatenate([sel[left], sel[~left]])
            mid = a + int(left.sum())
            kids = [add(a, mid), add(mid, b)]
            self.children[nd] = kids
            todo.extend(kids)
        self.center, self.half = np.asarray(center), np.asarray(half)
        self.num_nodes = len(self.ranges)
        self.d = d

    def node_edges(self, nd):
        a, b = self.ranges[nd]
        return self.perm[a:b]

    def diam(self, nd):
        return 2.0 * self.half[nd] * np.sqrt(self.d)


def dual_partition(tree, etree, eta):
    """Far / near pairs between DoF clusters and boundary-edge clusters (cluster.py:230-253)."""
    far, near = [], []
    if etree.num_nodes == 0 or len(etree.node_edges(0)) == 0:
        return far, near
    todo = [(0, 0)]
    while todo:
        a, b = todo.pop()
        gap = np.abs(tree.center[a] - etree.center[b]) - (tree.half[a] + etree.half[b])
        dist = float(np.linalg.norm(np.maximum(gap, 0.0)))
        if eta * dist >= max(tree.diam(a), etree.diam(b)) and dist > 0:
            far.append((a, b))
            continue
        ka, kb = tree.children[a], etree.children[b]
        if not ka and not kb:
            near.append((a, b))
            continue
        todo.extend([(c, b) for c in ka] if ka and (not kb or tree.half[a] >= etree.half[b]) else
                    [(a, c) for c in kb])
    return far, near


def boundary_flux_at_nodes(mesh, s, tree, cheb, eta, X, cell_leaf, device=None):
    """V(x) = int_dOmega n_out.(x-y)|x-y|^(-d-2s) dy at the cell nodes through the dual (DoF tree x
    edge tree) partition (cluster.py:525-593).  1D / <= 16 edges: None (the device computes V
    directly with the same rule).  The edge-tree moments and far pairs are host numpy; the direct
    near-edge sums (:586-592) run on the device (fl_boundary_flux_near)."""
    from .quadrature import gauss_legendre
    d = mesh.vertices.shape[1]
    E = np.asarray(mesh.boundary_edges)
    if d == 1 or len(E) <= 16:
        return None
    nc, q, _ = X.shape
    etree = EdgeTree(mesh)
    far, near = dual_partition(tree, etree, eta)
    gl = gauss_legendre(8)
    p0, p1 = mesh.vertices[E[:, 0]], mesh.vertices[E[:, 1]]
    nrm = np.asarray(mesh.boundary_normals)
    L = np.linalg.norm(p1 - p0, axis=1)
    Y = p0[:, None, :] + gl[0][None, :, None] * (p1 - p0)[:, None, :]
    eparent = np.full(etree.num_nodes, -1, np.int64)
    for nd in range(etree.num_nodes):
        for c in etree.children[nd]:
            eparent[c] = nd
    eorder = [0]
    for nd in eorder:
        eorder.extend(etree.children[nd])
    echeb = _Boxes(etree.center, etree.half, eparent, eorder, d, cheb.m, half_floor=1e-300)
    emom = np.zeros((etree.num_nodes, cheb.M, d))
    for nd in range(etree.num_nodes):
        if etree.children[nd]:
            continue
        eids = etree.node_edges(nd)
        if not len(eids):
            continue
        Lb = echeb.eval_basis(nd, Y[eids].reshape(-1, d)).reshape(len(eids), len(gl[0]), -1)
        base = np.einsum("eqm,q,e->em", Lb, gl[1], L[eids], optimize=True)
        for j in range(d):
            emom[nd, :, j] = nrm[eids][:, j] @ base
    for j in range(d):
        echeb.push_up(emom[:, :, j])
    F = np.zeros((tree.num_nodes, cheb.M))
    ex = -(d / 2.0 + s)
    for a, b in far:
        diff = cheb.points[a][:, None, :] - echeb.points[b][None, :, :]
        kern = np.sum(diff ** 2, axis=-1) ** ex
        for j in range(d):
            F[a] += (diff[:, :, j] * kern) @ emom[b, :, j]
    cheb.push_down(F)
    V = np.zeros((nc, q))
    near_map = {}
    for a, b in near:
        near_map.setdefault(a, []).append(b)
    by_leaf = {}
    for c in range(nc):
        by_leaf.setdefault(cell_leaf[c], []).append(c)
    groups, poff, eoff, eid = [], [0], [0], []
    cl = np.asarray(cell_leaf, np.int64)
    for a in range(0, nc, 16384):                                          # far part, bounded temporaries
        l = cl[a:a + 16384]
        T = (X[a:a + 16384] - cheb.cen[l][:, None, :]) / cheb.half[l][:, None, None]
        per = [lagrange_eval(cheb.ref, T[..., j]) for j in range(d)]
        Lb = per[0] if d == 1 else per[0][..., cheb.multi[:, 0]] * per[1][..., cheb.multi[:, 1]]
        V[a:a + 16384] = np.einsum("cqm,cm->cq", Lb, F[l])
    for nd, cs in by_leaf.items():
        cs = np.asarray(cs)
        if near_map.get(nd):
            eids = np.concatenate([etree.node_edges(b) for b in near_map[nd]])
            if len(eids):
                groups.append(cs)
                poff.append(poff[-1] + len(cs) * q)
                eid.append(eids)
                eoff.append(eoff[-1] + len(eids))
    if groups:
        # the near edges of every leaf in one device launch (fl_boundary_flux_near)
        from . import _lib
        from .assembly import _device_index
        cells = np.concatenate(groups)
        P = np.ascontiguousarray(X[cells].reshape(-1, d), dtype=np.float64)
        poff, eoff = np.asarray(poff, np.int64), np.asarray(eoff, np.int64)
        eid = np.ascontiguousarray(np.concatenate(eid), dtype=np.int64)
        p0c, p1c, nrmc = (np.ascontiguousarray(a, dtype=np.float64) for a in (p0, p1, nrm))
        gx, gw = (np.ascontiguousarray(a, dtype=np.float64) for a in gl)
        out = np.empty(len(P))
        _lib.check(_lib.load().fl_boundary_flux_near(
            _device_index(device), float(s), len(P), P.ctypes.data, len(poff) - 1, poff.ctypes.data,
            eoff.ctypes.data, eid.ctypes.data, len(E), p0c.ctypes.data, p1c.ctypes.data, nrmc.ctypes.data,
            gx.ctypes.data, gw.ctypes.data, len(gx), out.ctypes.data))
        V[cells] += out.reshape(len(cells), q)
    return V


def _basis_coefficients(mesh, dofmap, tree, cheb):
    """int phi_i L_alpha^leaf(i) over supp phi_i by the order m+1 cell rule (cluster.py:719-740)."""
    from .adapt import cell_nodes
    from .quadrature import simplex_rule
    d = mesh.vertices.shape[1]
    n = int(dofmap.n)
    out = np.zeros((n, cheb.M))
    X, W = cell_nodes(mesh, cheb.m + 1)
    pts, _ = simplex_rule(d, cheb.m + 1)
    lam = np.stack([1 - pts[:, 0], pts[:, 0]], 1) if d == 1 else \
        np.stack([1 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1)
    offs, pdata = mesh.patch_arrays()
    offs, pdata = np.asarray(offs, np.int64), np.asarray(pdata, np.int64)
    cd = np.asarray(dofmap.vertex_to_dof)[np.asarray(mesh.cells)]
    dofs = np.asarray(dofmap.dofs)
    lod = np.asarray(tree.leaf_of_dof, np.int64)
    # (leaf, cell) pairs: every cell of the patch of every DoF of the leaf, unique and sorted
    v = dofs[np.arange(n)]
    cnt = offs[v + 1] - offs[v]
    first = np.repeat(offs[v] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    pc = pdata[first + np.arange(cnt.sum())]
    key = np.unique(np.repeat(lod, cnt) * np.int64(mesh.cells.shape[0]) + pc)
    pl, pcell = key // mesh.cells.shape[0], key % mesh.cells.shape[0]
    for a in range(0, len(key), 16384):                                    # bounded temporaries
        l, c = pl[a:a + 16384], pcell[a:a + 16384]
        T = (X[c] - cheb.cen[l][:, None, :]) / cheb.half[l][:, None, None]   # (pairs, q, d)
        per = [lagrange_eval(cheb.ref, T[..., j]) for j in range(d)]
        Lb = per[0] if d == 1 else per[0][..., cheb.multi[:, 0]] * per[1][..., cheb.multi[:, 1]]
        mom = np.tensordot(W[c][:, :, None] * Lb, lam, axes=([1], [0]))     # (pairs, M, d+1)
        gd = cd[c]
        ok = (gd >= 0) & (lod[np.clip(gd, 0, None)] == l[:, None])
        g, vals = gd[ok], mom.transpose(0, 2, 1)[ok]                         # (entries, M)
        for k in range(cheb.M):
            out[:, k] += np.bincount(g, weights=vals[:, k], minlength=n)
    return out


def compress(mesh, dofmap, kernel, tree, eta, m, params=None, device=None):
    """The cluster-compressed stiffness operator (cluster.compress, cluster.py:667-712) with the
    heavy parts on the GPU: far blocks built on the device from the Chebyshev points, the near
    field by assemble_near_field (fl_assemble_near_field) with the dual-tree boundary flux V, the
    matvec / strong form through ClusterOperatorDevice.  Host: Chebyshev data, basis coefficients,
    the edge-tree boundary flux (as the reference)."""
    from .assembly import Variant, assemble_near_field
    from .adapt import cell_leaf_assignment, cell_nodes
    variant = getattr(getattr(kernel, "variant", Variant.INTEGRAL), "value", "integral")
    if variant == "symmetrized":
        raise NotImplementedError("symmetrized kernels are assembled densely")
    d = mesh.vertices.shape[1]
    far, near = admissible_partition(tree, eta)
    cheb = _Boxes(tree.center, tree.half, tree.parent, tree.topo_order, d, m)
    seen, fp = set(), []
    for a, b in far:
        key = (min(a, b), max(a, b))
        if key not in seen:
            seen.add(key)
            fp.append(key)
    far_pairs = np.asarray(fp, np.int64).reshape(-1, 2)
    basis_coef = _basis_coefficients(mesh, dofmap, tree, cheb)
    ns = NearStructure(mesh, dofmap, tree, near)
    cell_leaf = cell_leaf_assignment(mesh, dofmap, tree.leaf_of_dof)
    X, _ = cell_nodes(mesh, 6 if d == 1 else 4)
    V = boundary_flux_at_nodes(mesh, float(kernel.s), tree, cheb, eta, X, cell_leaf, device)
    A_near = assemble_near_field(mesh, dofmap, kernel, ns, params, V_nodes=V, device=device)
    shift = np.zeros((tree.num_nodes, d, m, m))
    for nd in range(tree.num_nodes):
        if cheb.shift[nd] is not None:
            for j in range(d):
                shift[nd, j] = cheb.shift[nd][j]
    op = ClusterOperatorDevice.from_arrays(d, m, tree.parent, tree.topo_order, tree.ranges, tree.dof_perm, shift,
                                           basis_coef, far_pairs, None, cheb.points, kernel.s, kernel.C_ds, A_near,
                                           A_near.diagonal().copy(), device, tree.center, tree.half,
                                           ns.near_leaf_map)
    op.far_pairs, op.basis_coef, op.near, op.cheb, op.tree = far_pairs, basis_coef, A_near, cheb, tree
    op.meta = {"near_leaf_map": ns.near_leaf_map, "eta": eta}
    return op


def matvec(op, x):
    """cluster.py:814-815."""
    return op.matvec(x)


def evaluate_far_field_at_points(op, u, points, owner_leaves):
    """cluster.py:818-819."""
    return op.evaluate_far_field_at_points(u, points, owner_leaves)
