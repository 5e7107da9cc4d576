"""Quadrature rules, pair classification and Gauss-order selection — host side.

Mirrors `fraclap.quadrature` (reference quadrature.py): the same public names and
argument meaning.  The 1-D node sets come from the same third-party generators the reference
calls (numpy `leggauss`, scipy `roots_jacobi`).  The Sauter–Schwab/Duffy singular rules are
re-derived as unions of radial pieces (`_rule`: a Gauss–Jacobi radial variable, Gauss–Legendre
regular variables and one map per piece) and agree with the reference's payloads
(quadrature.py:188-398) node by node to <= 1e-14 (tests/test_tables.py).

`pack_tables(d, s)` flattens every rule the device kernels can ask for into the
`fl_tables` blob of include/fraclap_b200.h.
"""
from __future__ import annotations

import logging
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.special import roots_jacobi

log = logging.getLogger(__name__)

K_MAX = 32                    # quadrature.py:35
XQ_ORDER = {1: 6, 2: 4}       # assembly.py:635
EDGE_GL_ORDER = 8             # assembly.py:43


class PairTopology(Enum):
    """quadrature.py:38-46."""
    IDENTICAL = "identical"
    COMMON_EDGE = "common_edge"
    COMMON_VERTEX = "common_vertex"
    DISJOINT = "disjoint"
    EDGE_OF_CELL = "edge_of_cell"
    TOUCHING_EDGE = "touching_edge"
    DISJOINT_EDGE = "disjoint_edge"


class QuadratureError(RuntimeError):
    """quadrature.py:49."""


# ids of the device table directory (include/fraclap_b200.h FL_TOPO_*)
TOPO_ID = {PairTopology.IDENTICAL: 0, PairTopology.COMMON_EDGE: 1, PairTopology.COMMON_VERTEX: 2,
           PairTopology.DISJOINT: 3, PairTopology.EDGE_OF_CELL: 4, PairTopology.TOUCHING_EDGE: 5}
TOPO_CELL, TOPO_EDGE_GL, NTOPO, KDIR, NODE = 6, 7, 8, 33, 8


# ------------------------------------------------------------------ 1-D rules
@lru_cache(maxsize=None)
def gauss_legendre(k: int):
    """k-point Gauss–Legendre on [0,1] (quadrature.py:53-59)."""
    if k < 1:
        raise ValueError("order must be >= 1")
    t, w = leggauss(k)
    return 0.5 * (t + 1.0), 0.5 * w


@lru_cache(maxsize=None)
def gauss_jacobi(k: int, alpha: float):
    """k-point Gauss rule on [0,1] for the weight t^alpha (quadrature.py:62-68)."""
    if alpha <= -1:
        raise ValueError("weight exponent must be > -1")
    t, w = roots_jacobi(k, alpha, 0.0)
    return 0.5 * (1.0 - t), w * 2.0 ** (-alpha - 1.0)


@lru_cache(maxsize=None)
def triangle_rule(k: int):
    """Collapsed (Duffy) tensor rule on the unit triangle (quadrature.py:71-78)."""
    t, wt = gauss_legendre(k)
    a, b = np.meshgrid(t, t, indexing="ij")
    w = np.outer(wt, wt) * (1 - a)
    return np.stack([a, b * (1 - a)], axis=-1).reshape(-1, 2), w.ravel()


def simplex_rule(d: int, k: int):
    """quadrature.py:81-85."""
    if d == 1:
        t, w = gauss_legendre(k)
        return t[:, None], w
    return triangle_rule(k)


# ------------------------------------------------------------------ classification
def classify_pair(cell_a, cell_b=None, edge=None) -> PairTopology:
    """By shared-vertex count (quadrature.py:90-110)."""
    a = set(cell_a)
    if edge is not None:
        e = list(edge)
        shared = len(a & set(e))
        if shared == len(e):
            return PairTopology.EDGE_OF_CELL
        return PairTopology.TOUCHING_EDGE if shared else PairTopology.DISJOINT_EDGE
    b = set(cell_b)
    d = len(list(cell_a)) - 1
    shared = len(a & b)
    if shared == d + 1:
        return PairTopology.IDENTICAL
    if d == 2 and shared == 2:
        return PairTopology.COMMON_EDGE
    return PairTopology.COMMON_VERTEX if shared else PairTopology.DISJOINT


# ------------------------------------------------------------------ order selection
@dataclass
class OrderParams:
    """quadrature.py:115-131."""
    rho1: float = 2.0
    rho2: float = 2.0
    rho3: float = 2.0
    rho4: float = 2.0
    C_offset: float = 1.0
    alpha: float | None = None

    def __post_init__(self):
        if min(self.rho1, self.rho2, self.rho3, self.rho4) <= 1:
            raise ValueError("all rho parameters must exceed 1")

    def target_alpha(self, d, s):
        if self.alpha is not None:
            return self.alpha
        return 2.0 - s if d == 1 else 1.0


_TOUCHING = (PairTopology.IDENTICAL, PairTopology.COMMON_EDGE, PairTopology.COMMON_VERTEX,
             PairTopology.EDGE_OF_CELL, PairTopology.TOUCHING_EDGE)


def select_order(pair, h_K, h_K2, dist, n, s, params: OrderParams, boundary=False, d=2):
    """Gauss points per direction (quadrature.py:138-179).  Host restatement; the device
    evaluates the same expression per pair (csrc/fl_device.cuh order_*)."""
    h_K = np.asarray(h_K, float)
    h_K2 = np.asarray(h_K2, float)
    dist = np.asarray(dist, float)
    lead = params.target_alpha(d, s) / 2 + (0.25 if boundary else 0.5)
    lnn = np.log(max(float(n), 2.0))
    if pair in _TOUCHING:
        rho = params.rho3 if boundary else params.rho1
        k = (lead * lnn + s * np.abs(np.log(np.minimum(h_K, h_K2)))) / np.log(rho) - params.C_offset
    else:
        if np.any(dist <= 0):
            raise QuadratureError("disjoint pair classified with zero distance")
        rho = params.rho4 if boundary else params.rho2
        lK, lK2 = np.abs(np.log(h_K)), np.abs(np.log(h_K2))
        mx = np.maximum(lK, lK2)

        def one(ha, hb, lhb):
            num = lead * lnn + (s - 1) * lhb + mx - s * np.log(dist / hb) - params.C_offset
            return num / (np.maximum(np.log(np.maximum(dist / ha, 1e-300)), 0.0) + np.log(rho))

        k = np.maximum(one(h_K, h_K2, lK2), one(h_K2, h_K, lK))
    k = np.ceil(k)
    cap = 9 if (pair not in _TOUCHING and d == 2) else K_MAX
    if np.any(k > cap):
        log.info("quadrature order clamped to %d for %d pair(s)", cap, int(np.sum(k > cap)))
    return np.clip(k, 2, cap).astype(np.int64)


# ------------------------------------------------------------------ singular payloads
# Each singular pair integral (Sauter–Schwab / Duffy, §3, SPEC.md "singular rules") is
# regularised by splitting the pair's parameter domain into PIECES on which one RADIAL variable
# r in (0, 1) measures the distance to the singular set; in r the integrand behaves like r^alpha
# and a Gauss–Jacobi rule for that weight is used, the remaining (regular) variables get
# Gauss–Legendre rules.  A rule is therefore fully described by
#   * the radial rule (points, Jacobi exponent) and the extra power of r left after the weight,
#   * the list of regular 1-D rules,
#   * per piece, the map (r, v1, v2, ...) -> (point in K, point in K~ [or the edge parameter a])
#     and the Jacobian of that map.
# `_rule` builds the tensor grid (radial outermost, then the regular variables in order) and
# concatenates the pieces — the reference's node order (quadrature.py:188-398), so the tables
# can be compared node by node (tests/test_tables.py, ≤ 1e-14 against the reference's arrays).


def _rule(radial, axes, pieces, rfac, second="y"):
    """radial = (nodes, weights) of the radial rule; axes = list of (nodes, weights); pieces =
    maps f(r, *V) -> (X, Y, jac) on the open grid V of the regular variables (X, Y: point
    fields (..., dim); for second == "a", Y is the edge parameter (...)); rfac(r) = the radial
    factor beyond the Jacobi weight.  Weight of a node = prod w_v * jac * w_r * rfac(r)."""
    rq, rw = radial
    shape = tuple(len(a[0]) for a in axes)
    npts = int(np.prod(shape, dtype=np.int64))
    V = np.ix_(*[a[0] for a in axes]) if axes else ()
    Wv = np.ones(shape)
    for ax, (_, w) in enumerate(axes):
        Wv = Wv * np.asarray(w).reshape([len(w) if i == ax else 1 for i in range(len(axes))])
    X, Y, W = [], [], []
    for f in pieces:
        for r, wr in zip(rq, rw):
            x, y, jac = f(r, *V)
            x = np.asarray(x, float)
            X.append(np.broadcast_to(x, shape + x.shape[-1:]).reshape(npts, -1))
            y = np.asarray(y, float)
            Y.append(np.broadcast_to(y, shape + (y.shape[-1:] if second == "y" else ())).reshape(npts, -1))
            W.append(np.broadcast_to(Wv * jac, shape).reshape(npts) * (wr * rfac(r)))
    X, Y, W = np.concatenate(X), np.concatenate(Y), np.concatenate(W)
    return {"x": X if X.shape[1] > 1 else X[:, 0], second: Y if Y.shape[1] > 1 else Y[:, 0], "w": W}


def _pt(a, b):
    """Point field from two coordinate arrays broadcast together: (..., 2)."""
    a, b = np.broadcast_arrays(a, b)
    return np.stack([a, b], axis=-1)


def _pt1(a):
    return np.asarray(a, float)[..., None]


# identical 2D pair: for a difference w = x - y of two points of the reference triangle T, the
# points x with x, x - w in T form T ∩ (T + w) = {x >= max(w, 0), x1 + x2 <= min(1, 1 + w1 + w2)},
# a right triangle of leg L = min(1, 1 + w1 + w2) - max(w1, 0) - max(w2, 0): area L^2/2; the
# integrand (P1 hat differences: constant in x for fixed w) is sampled at its centroid.
def _overlap(wv):
    lo = np.maximum(wv, 0.0)
    L = np.minimum(1.0, 1.0 + wv[..., 0] + wv[..., 1]) - lo[..., 0] - lo[..., 1]
    return 0.5 * L * L, lo + (L / 3.0)[..., None]


_HEX = np.array([(1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1)], float)   # corners of {x - y}


@lru_cache(maxsize=None)
def rule_identical_1d(s):
    """K = K~ = [0, 1]: radial z = |x - y| (weight (1 - z) z^(2s-1) after the Jacobi factor), the
    integrand is constant along x - y = z, one node at the midpoint of each orientation
    (quadrature.py:221-230)."""
    return _rule(gauss_jacobi(3, 1 - 2 * s), [],
                 [lambda z: (_pt1((1 + z) / 2), _pt1((1 - z) / 2), 1.0),
                  lambda z: (_pt1((1 - z) / 2), _pt1((1 + z) / 2), 1.0)],
                 lambda z: (1 - z) * z ** (2 * s - 1))


@lru_cache(maxsize=None)
def rule_vertex_1d(k, s):
    """Cells meeting at the local origin: radial t = the farther point, v = ratio of the nearer
    (quadrature.py:233-243)."""
    return _rule(gauss_jacobi(3, 2 - 2 * s), [gauss_legendre(k)],
                 [lambda t, v: (_pt1(t), _pt1(t * v), 1.0),
                  lambda t, v: (_pt1(t * v), _pt1(t), 1.0)],
                 lambda t: t ** (2 * s - 1))


@lru_cache(maxsize=None)
def rule_identical_2d(k, s):
    """The differences x - y fill the hexagon conv(_HEX): six radial sectors, r along the ray,
    t along the sector's outer edge (quadrature.py:246-260)."""
    def sector(c):
        def f(r, t):
            wv = r * ((1 - t)[:, None] * _HEX[c] + t[:, None] * _HEX[(c + 1) % 6])
            area, x = _overlap(wv)
            return x, x - wv, area
        return f
    return _rule(gauss_jacobi(3, 1 - 2 * s), [gauss_legendre(k)], [sector(c) for c in range(6)],
                 lambda r: r ** (2 * s))


@lru_cache(maxsize=None)
def rule_common_edge_2d(k, s):
    """Shared edge = local (0, 1) of both cells; four Duffy pieces (which cell carries the
    longer transversal leg x which side of the edge point), radial r = the transversal size
    (quadrature.py:263-294)."""
    k = min(k, 16)
    g = gauss_legendre(k)

    def piece(swap, inner):
        def f(r, z, v):
            if inner:          # the transversal legs scaled by v
                zz, bb, bp, jac = r * v * z, r * v * (1 - z), r, v
            else:
                zz, bb, bp, jac = r * z, r * (1 - z), r * v, 1.0
            al = zz + 0.5 * (1 - r)
            u, uu = _pt(al, bb), _pt(al - zz, bp)
            return (uu, u, jac) if swap else (u, uu, jac)
        return f
    return _rule(gauss_jacobi(3, 2 - 2 * s), [g, g],
                 [piece(sw, inn) for sw in (False, True) for inn in (False, True)],
                 lambda r: (1 - r) * r ** (2 * s))


def _cv_order(k):
    return max(2, min(8, (k + 1) // 2 + 1))


@lru_cache(maxsize=None)
def _rule_common_vertex_2d(kk, s):
    g = gauss_legendre(kk)

    def piece(y_far):
        def f(r, a, b, w):
            rx, ry = (r * w, r) if y_far else (r, r * w)
            return _pt(rx * (1 - a), rx * a), _pt(ry * (1 - b), ry * b), w
        return f
    return _rule(gauss_jacobi(3, 3 - 2 * s), [g, g, g], [piece(False), piece(True)], lambda r: r ** (2 * s))


def rule_common_vertex_2d(k, s):
    """Shared vertex = local 0 of both cells: each cell in polar-like coordinates (distance to the
    vertex, position along the opposite edge); radial r = the larger distance, w = the ratio of
    the smaller (quadrature.py:297-315)."""
    return _rule_common_vertex_2d(_cv_order(k), s)


@lru_cache(maxsize=None)
def rule_edge_of_cell_1d(s, vanishing):
    """Boundary point at the cell's local origin: radial r = distance (quadrature.py:332-335)."""
    return _rule(gauss_jacobi(3, vanishing - 2 * s), [], [lambda r: (_pt1(r), 0.0, 1.0)],
                 lambda r: r ** (2 * s - vanishing), second="a")


@lru_cache(maxsize=None)
def rule_edge_of_cell_2d(k, s, vanishing):
    """Cell (e0, e1, p) against its own boundary edge (e0, e1): three pieces by where the edge
    point a lies relative to the cell point's projection, radial r = distance to the edge line
    scale (quadrature.py:338-360)."""
    def piece(c):
        def f(r, z, t):
            if c == 1:
                zrel, beta = r * z, r * (1 - z)
                al = zrel + t * (1 - r)
            elif c == 2:
                beta, zrel, al = r * z, -r, t * (1 - r)
            else:
                beta, zrel, al = r, -r * z, t * (1 - r)
            return _pt(al, beta), al - zrel, 1.0
        return f
    return _rule(gauss_jacobi(4, vanishing - 2 * s), [gauss_legendre(k), gauss_legendre(max(3, k // 2))],
                 [piece(c) for c in (1, 2, 3)], lambda r: (1 - r) * r ** (1 + 2 * s - vanishing), second="a")


@lru_cache(maxsize=None)
def rule_touching_edge_2d(k, s):
    """Cell (c, A, B) against a boundary edge leaving the shared vertex c: radial xi = the larger
    of the two distances to c, w = the ratio of the smaller (quadrature.py:363-384)."""
    kk = max(2, (k + 1) // 2 + 1)
    g = gauss_legendre(kk)

    def piece(edge_far):
        def f(xi, a, w):
            ru, ap, jac = (xi * w, xi, w) if edge_far else (xi, xi * w, 1.0)
            return _pt(ru * (1 - a), ru * a), np.broadcast_to(ap, np.broadcast_shapes(np.shape(a), np.shape(w))), jac
        return f
    return _rule(gauss_jacobi(4, 1 - 2 * s), [g, g], [piece(False), piece(True)], lambda x: x ** (1 + 2 * s),
                 second="a")


def payload(topology: PairTopology, k: int, s: float, d: int, vanishing=0):
    """Same contract as reference_payload (quadrature.py:401-420)."""
    T = PairTopology
    if topology is T.IDENTICAL:
        return rule_identical_1d(s) if d == 1 else rule_identical_2d(min(k, 24), s)
    if topology is T.COMMON_EDGE:
        if d != 2:
            raise QuadratureError("common-edge pairs exist in 2D only")
        return rule_common_edge_2d(k, s)
    if topology is T.COMMON_VERTEX:
        return rule_vertex_1d(k, s) if d == 1 else rule_common_vertex_2d(k, s)
    if topology is T.DISJOINT:
        px, wx = simplex_rule(d, k)
        nx = len(wx)
        x = np.repeat(px, nx, axis=0)
        y = np.tile(px, (nx, 1))
        w = np.outer(wx, wx).ravel()
        return dict(x=x.ravel(), y=y.ravel(), w=w) if d == 1 else dict(x=x, y=y, w=w)
    if topology is T.EDGE_OF_CELL:
        return rule_edge_of_cell_1d(s, vanishing) if d == 1 else rule_edge_of_cell_2d(k, s, vanishing)
    if topology is T.TOUCHING_EDGE:
        if d != 2:
            raise QuadratureError("1D boundary points touching a cell are EDGE_OF_CELL")
        return rule_touching_edge_2d(k, s)
    if topology is T.DISJOINT_EDGE:
        px, wx = simplex_rule(d, k)
        if d == 1:
            return dict(x=px.ravel(), a=np.zeros(len(wx)), w=wx)
        aq, aw = gauss_legendre(k)
        return dict(x=np.repeat(px, k, axis=0), a=np.tile(aq, len(wx)), w=np.outer(wx, aw).ravel())
    raise QuadratureError("unsupported topology %r" % topology)


# ------------------------------------------------------------------ device tables
def _lam(d, pts):
    if d == 1:
        return np.stack([1 - pts[:, 0], pts[:, 0]], axis=1)
    return np.stack([1 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], axis=1)


def needed_orders(mesh, dofmap, s, params: OrderParams | None = None):
    """Sets of touching / boundary orders the device can ask for on this mesh: every touching
    pair's order is the touching formula at one of its cells' diameters (quadrature.py:150-155,
    hmin = min(h_K, h_K2)), so evaluating it per cell bounds them; +-1 guards a last-ulp log
    difference.  Returns two sorted tuples."""
    params = params or OrderParams()
    d = mesh.vertices.shape[1]
    h = np.asarray(mesh.cell_diameters(), float) if hasattr(mesh, "cell_diameters") else None
    if h is None:
        P = mesh.vertices[mesh.cells]
        h = np.abs(P[:, 1, 0] - P[:, 0, 0]) if d == 1 else np.max(
            [np.linalg.norm(P[:, (i + 1) % 3] - P[:, i], axis=1) for i in range(3)], axis=0)
    out = []
    for bnd in (False, True):
        k = np.unique(select_order(PairTopology.IDENTICAL, h, h, 0.0, dofmap.n, s, params, boundary=bnd, d=d))
        ks = set()
        for v in k.tolist():
            ks.update((v - 1, v, v + 1))
        out.append(tuple(sorted(x for x in ks if 2 <= x <= K_MAX)))
    return out[0], out[1]


@lru_cache(maxsize=32)
def pack_tables(d: int, s: float, korders=None, borders=None):
    """Rules of one (d, s) in the fl_tables layout: (dir int64[8*33*2], data float64).
    korders / borders restrict the touching / boundary singular rules to those orders
    (default: every order 2..32)."""
    if not 0.0 < s < 1.0:
        raise ValueError("s must lie in (0,1)")
    recs = []          # (topo_id, k, records[N, 8])
    T = PairTopology
    vanish = 0 if s < 0.5 else 2          # assembly.py:794

    def pair_rec(p):
        N = len(p["w"])
        r = np.zeros((N, NODE))
        x = np.asarray(p["x"], float).reshape(N, -1)
        y = np.asarray(p["y"], float).reshape(N, -1)
        r[:, 0:x.shape[1]] = x
        r[:, 2:2 + y.shape[1]] = y
        r[:, 4] = p["w"]
        return r

    def edge_rec(p):
        N = len(p["w"])
        r = np.zeros((N, NODE))
        x = np.asarray(p["x"], float).reshape(N, -1)
        r[:, 0:x.shape[1]] = x
        r[:, 2] = p["a"]
        r[:, 3] = p["w"]
        return r

    def cell_rec(pts, w, weighted):
        N = len(w)
        r = np.zeros((N, NODE))
        r[:, 0:pts.shape[1]] = pts
        r[:, 2] = w
        lam = _lam(d, pts)
        r[:, 3:3 + lam.shape[1]] = lam * w[:, None] if weighted else lam
        return r

    kt = range(2, K_MAX + 1) if korders is None else korders
    kb = range(2, K_MAX + 1) if borders is None else borders
    if d == 1:
        recs.append((0, 0, pair_rec(rule_identical_1d(s))))
        for k in kt:
            recs.append((2, k, pair_rec(rule_vertex_1d(k, s))))
        recs.append((4, 0, edge_rec(rule_edge_of_cell_1d(s, vanish))))
    else:
        for k in kt:
            recs.append((0, k, pair_rec(rule_identical_2d(min(k, 24), s))))
            recs.append((1, k, pair_rec(rule_common_edge_2d(k, s))))
            recs.append((2, k, pair_rec(rule_common_vertex_2d(k, s))))
        for k in kb:
            recs.append((4, k, edge_rec(rule_edge_of_cell_2d(k, s, vanish))))
            recs.append((5, k, edge_rec(rule_touching_edge_2d(k, s))))
    for k in range(2, (K_MAX if d == 1 else 9) + 1):
        pts, w = simplex_rule(d, k)
        recs.append((3, k, cell_rec(pts, w, True)))
    pts, w = simplex_rule(d, XQ_ORDER[d])
    recs.append((TOPO_CELL, 0, cell_rec(pts, w, False)))
    t, w = gauss_legendre(EDGE_GL_ORDER)
    er = np.zeros((len(w), NODE))
    er[:, 0], er[:, 1] = t, w
    recs.append((TOPO_EDGE_GL, 0, er))
    dir_ = np.zeros((NTOPO * KDIR, 2), np.int64)
    off = 0
    for topo, k, r in recs:
        dir_[topo * KDIR + k] = (off, len(r))
        off += len(r)
    data = np.ascontiguousarray(np.concatenate([r for _, _, r in recs]).ravel())
    dir_ = np.ascontiguousarray(dir_.ravel())
    dir_.setflags(write=False)
    data.setflags(write=False)
    return dir_, data
