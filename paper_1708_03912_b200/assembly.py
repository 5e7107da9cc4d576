"""Dense P1 stiffness assembly of the integral fractional Laplacian on a B200.

Drop-in for `fraclap.assembly.assemble_dense` (reference assembly.py:1059-1104): same
signature, same refusal beyond `n_limit`, same (n, n) float64 result.  The work runs in
libfraclap_b200.so (csrc/): classification, singular pairs, tail, boundary flux, cross
tiles and the deterministic accumulation; Python only marshals arrays.

`assemble_dense_device` returns the matrix left in HBM as a `DenseDeviceOperator`, which
`solve.pcg` — and the reference's own pcg through LinearOperatorHandle.from_matrix
(solve.py:29-30) — accept directly.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
from scipy.special import gammaln

from . import _lib
from .quadrature import OrderParams, XQ_ORDER, EDGE_GL_ORDER, pack_tables, simplex_rule

DENSE_LIMIT = 4000            # assembly.py:44


class Variant(Enum):
    """assembly.py:47-50."""
    INTEGRAL = "integral"
    REGIONAL = "regional"
    SYMMETRIZED = "symmetrized"


class AssemblyError(RuntimeError):
    """assembly.py:53."""


def normalisation(d: int, s: float) -> float:
    """C(d,s) = 2^{2s} s Gamma(s+d/2) / (pi^{d/2} Gamma(1-s))  (assembly.py:57-63)."""
    if not 0.0 < s < 1.0:
        raise ValueError("s must lie in (0,1)")
    return float(2.0 ** (2 * s) * s * math.exp(gammaln(s + d / 2) - gammaln(1.0 - s)) / math.pi ** (d / 2))


@dataclass
class FractionalKernel:
    """assembly.py:66-94 (the symmetrized variant is outside the dense device path)."""
    d: int
    s: float
    variant: Variant = Variant.INTEGRAL

    def __post_init__(self):
        self.C_ds = normalisation(self.d, self.s)

    @property
    def exponent(self):
        return -(self.d / 2.0 + self.s)


def _device_index(device):
    if device is None:
        try:
            import torch
            return torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:
            return 0
    return int(getattr(device, "index", device) or 0)


def _tables(mesh, dofmap, s, params):
    from .quadrature import needed_orders
    # the needed-order sets depend on the cell diameters, n, s and params only; cached on the
    # mesh like its patches / diameters (meshes are not mutated after construction)
    cache = mesh.__dict__.setdefault("_fl_orders", {})
    key = (int(dofmap.n), float(s), None if params is None else tuple(vars(params).items()))
    if key not in cache:
        cache[key] = needed_orders(mesh, dofmap, float(s), params)
    kt, kb = cache[key]
    dir_, data = pack_tables(mesh.vertices.shape[1], float(s), kt, kb)
    return dir_, data, _lib.fl_tables(dir_.ctypes.data, data.ctypes.data, len(data))


def assemble_dense_device(mesh, dofmap, kernel, params: OrderParams | None = None, n_limit=None,
                          rows=None, device=None, stream=None):
    """Assemble rows [r0, r1) (default: all) of A on the GPU; returns a DenseDeviceOperator."""
    from .operator import DenseDeviceOperator
    lib = _lib.load()
    variant = getattr(getattr(kernel, "variant", Variant.INTEGRAL), "value", "integral")
    if variant == "symmetrized":
        raise AssemblyError("symmetrized kernels are not supported by the dense device path")
    m = _lib.Marshal(mesh, dofmap, kernel, params)
    dir_, data, tb = _tables(mesh, dofmap, float(kernel.s), params)
    n = int(dofmap.n)
    r0, r1 = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
    handle = C.c_void_p()
    code = lib.fl_assemble_dense(C.byref(m.mesh), C.byref(m.dofmap), C.byref(m.kernel), C.byref(m.params),
                                 C.byref(tb), -1 if n_limit is None else int(n_limit), r0, r1,
                                 _device_index(device), _lib.stream_arg(stream),
                                 C.byref(handle))
    _lib.check(code)
    return DenseDeviceOperator(handle, n, r0, r1)


def assemble_dense(mesh, dofmap, kernel, params: OrderParams | None = None, n_limit=DENSE_LIMIT, *,
                   out=None):
    """Dense stiffness matrix, all cell pairs (assembly.py:1059-1104) -> np.ndarray (n, n).
    `out` (keyword only): a preallocated C-contiguous (n, n) float64 array, e.g. pinned."""
    if dofmap.n > n_limit:
        raise AssemblyError("dense assembly refused beyond %d dofs" % n_limit)
    lib = _lib.load()
    variant = getattr(getattr(kernel, "variant", Variant.INTEGRAL), "value", "integral")
    if variant == "symmetrized":
        raise AssemblyError("symmetrized kernels are not supported by the dense device path")
    n = int(dofmap.n)
    if out is None:
        out = np.empty((n, n))
    elif out.shape != (n, n) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array of shape %r" % ((n, n),))
    m = _lib.Marshal(mesh, dofmap, kernel, params)
    dir_, data, tb = _tables(mesh, dofmap, float(kernel.s), params)
    _lib.check(lib.fl_assemble_dense_host(C.byref(m.mesh), C.byref(m.dofmap), C.byref(m.kernel), C.byref(m.params),
                                          C.byref(tb), int(n_limit), _device_index(None), out.ctypes.data))
    return out


def load_vector(mesh, dofmap, f, order=4, discontinuity=None, device=None):
    """b_i = int f phi_i by the per-cell rule of `order` (assembly.py:550-570) on the GPU
    (fl_load_vector).  `f` is a callable on (m, d) points, as in the reference — evaluated on the
    host at the rule nodes the device maps (fl_cell_rule_nodes) — or a number (f constant: no
    host evaluation at all).  Per DoF the cell contributions are summed in ascending cell order,
    like np.add.at.  Cells cut by a `discontinuity` (split at assembly.py:574-596) are not
    supported on the device path."""
    if discontinuity is not None:
        raise ValueError("load_vector: discontinuity splitting is not supported by the device path")
    lib = _lib.load()
    d = int(mesh.vertices.shape[1])
    pts, w = simplex_rule(d, order)
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    q = len(w)
    m = _lib.Marshal(mesh, dofmap, FractionalKernel(d, 0.5), None)
    dev = _device_index(device)
    fvals, fconst = None, 0.0
    if callable(f):
        X = np.empty((mesh.num_cells, q, d))
        _lib.check(lib.fl_cell_rule_nodes(C.byref(m.mesh), pts.ctypes.data, q, dev, X.ctypes.data))
        fvals = np.ascontiguousarray(np.asarray(f(X.reshape(-1, d)), dtype=np.float64).reshape(mesh.num_cells, q))
    else:
        fconst = float(f)
    b = np.empty(int(dofmap.n))
    _lib.check(lib.fl_load_vector(C.byref(m.mesh), C.byref(m.dofmap), pts.ctypes.data, w.ctypes.data, q,
                                  None if fvals is None else fvals.ctypes.data, fconst, dev, b.ctypes.data))
    return b


def assemble_near_field(mesh, dofmap, kernel, near_pairs, params: OrderParams | None = None, V_nodes=None,
                        xquad=None, device=None):
    """Near-field sparse matrix over the non-admissible DoF pairs (assembly.py:860-970) on the GPU
    (fl_assemble_near_field) -> scipy.sparse.csr_matrix (n, n), canonical (sorted indices).

    `near_pairs`: a NearStructure (this package's cluster.NearStructure or the reference's):
    its `nl_pairs` (leaf node pairs), `leaf_index` and `leaf_idx_of_dof` are read.  `V_nodes`:
    the boundary flux potential at the (nc, q) cell-rule nodes (e.g. the cluster far field's),
    default: direct GL8 over every boundary edge.  `xquad` may only restate the standard cell
    rule (cell_quadrature(mesh, XQ_ORDER[d]), which is what the device uses)."""
    from scipy.sparse import csr_matrix
    lib = _lib.load()
    variant = getattr(getattr(kernel, "variant", Variant.INTEGRAL), "value", "integral")
    if variant == "symmetrized":
        raise AssemblyError("symmetrized kernels are assembled densely")
    d = int(mesh.vertices.shape[1])
    nc = int(mesh.num_cells)
    q = 6 if d == 1 else 16
    if xquad is not None and np.shape(xquad[1]) != (nc, q):
        raise ValueError("xquad must be the cell rule of order XQ_ORDER[d] (%d nodes per cell)" % q)
    n = int(dofmap.n)
    leaf_idx = np.ascontiguousarray(near_pairs.leaf_idx_of_dof, dtype=np.int64)
    li = near_pairs.leaf_index
    nl = max(li.values()) + 1 if len(li) else 1
    pairs = np.ascontiguousarray([[li[int(a)], li[int(b)]] for a, b in np.asarray(near_pairs.nl_pairs).reshape(-1, 2)],
                                 dtype=np.int64).reshape(-1, 2)
    if V_nodes is not None:
        V_nodes = np.ascontiguousarray(V_nodes, dtype=np.float64)
        if V_nodes.shape != (nc, q):
            raise ValueError("V_nodes must have shape %r" % ((nc, q),))
    m = _lib.Marshal(mesh, dofmap, kernel, params)
    dir_, data, tb = _tables(mesh, dofmap, float(kernel.s), params)
    ns = _lib.fl_near_structure(nl, leaf_idx.ctypes.data if n else None, len(pairs),
                                pairs.ctypes.data if len(pairs) else None)
    h = C.c_void_p()
    _lib.check(lib.fl_assemble_near_field(C.byref(m.mesh), C.byref(m.dofmap), C.byref(m.kernel), C.byref(m.params),
                                          C.byref(tb), C.byref(ns),
                                          None if V_nodes is None else V_nodes.ctypes.data,
                                          _device_index(device), C.byref(h)))
    try:
        nn, nnz, npair = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(lib.fl_sparse_info(h, C.byref(nn), C.byref(nnz), C.byref(npair)))
        indptr = np.empty(n + 1, np.int64)
        indices = np.empty(max(nnz.value, 1), np.int32)
        vals = np.empty(max(nnz.value, 1))
        _lib.check(lib.fl_sparse_to_host(h, indptr.ctypes.data, indices.ctypes.data, vals.ctypes.data))
    finally:
        lib.fl_sparse_free(h)
    A = csr_matrix((vals[:nnz.value], indices[:nnz.value], indptr), shape=(n, n))
    A.has_sorted_indices = True
    return A
