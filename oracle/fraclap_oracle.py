"""CPU ORACLE — test infrastructure only.

A plain numpy restatement of the reference path (`fraclap` assemble_dense + pcg, reference
files under /root/reference/pkg/src/fraclap) used as the checker for the CUDA product:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
may import this module.  The product (paper_1708_03912_b200) never does.

Pinned against the reference itself: tests/golden/*.npz were produced by running the
unmodified reference in the build container (tests/golden/make_golden.py) and
tests/test_oracle.py checks this restatement against them (full matrices of the small
meshes and c1, sampled rows of c2/c3, exact per-pair Gauss orders, rule tables).

Organisation (owner-computes by cell, memory O(n^2 + nc), unlike the reference's nc^2
pair arrays):  for every cell K the contributions whose ROW lies in K are computed by
`_cell_rows`; `assemble(rows=None)` sums them into A (all rows), `assemble(rows=R)` only
for the cells touching the rows R (the sampled-row oracle of SURVEY.md §8(c)).

fp32 switch: the reference evaluates large 2D disjoint groups in float32 (assembly.py:
203-227).  `cross_fp32=True` reproduces that shortcut; the default is the fp64 variant
that the parity bar is defined against (SURVEY.md §0 hazard 1).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace
from functools import lru_cache

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.special import gammaln, roots_jacobi

K_MAX = 32
XQ = {1: 6, 2: 4}
EDGE_GL = 8


# =================================================================== rules
@lru_cache(maxsize=None)
def gl(k):
    """quadrature.py:53-59"""
    x, w = leggauss(k)
    return 0.5 * (x + 1.0), 0.5 * w


@lru_cache(maxsize=None)
def gj(k, a):
    """quadrature.py:62-68"""
    x, w = roots_jacobi(k, a, 0.0)
    return 0.5 * (1.0 - x), w * 2.0 ** (-a - 1.0)


@lru_cache(maxsize=None)
def simplex(d, k):
    """quadrature.py:71-85 (Duffy triangle rule)."""
    x, w = gl(k)
    if d == 1:
        return x[:, None], w
    pts = np.array([[x[i], x[j] * (1 - x[i])] for i in range(k) for j in range(k)])
    wts = np.array([w[i] * w[j] * (1 - x[i]) for i in range(k) for j in range(k)])
    return pts, wts


def _area(w1, w2):
    """quadrature.py:191-198, one offset."""
    t = w1 + w2
    if w1 >= 0 and w2 >= 0:
        A = (1 - t) ** 2
    elif w1 <= 0 and w2 <= 0:
        A = (1 + t) ** 2
    elif w1 > 0:
        A = (1 - w1) ** 2 if t >= 0 else (1 + w2) ** 2
    else:
        A = (1 - w2) ** 2 if t >= 0 else (1 + w1) ** 2
    return 0.5 * A


def _rep(w1, w2):
    """quadrature.py:201-218, one offset."""
    t = w1 + w2
    if w1 >= 0 and w2 >= 0:
        return w1 + (1 - t) / 3, w2 + (1 - t) / 3
    if w1 <= 0 and w2 <= 0:
        return (1 + t) / 3, (1 + t) / 3
    if w1 > 0 and w2 < 0:
        return ((1 + 2 * w1) / 3, (1 - w1) / 3) if t >= 0 else (w1 + (1 + w2) / 3, (1 + w2) / 3)
    if w1 < 0 and w2 > 0:
        return ((1 - w2) / 3, (1 + 2 * w2) / 3) if t >= 0 else ((1 + w1) / 3, w2 + (1 + w1) / 3)
    return np.nan, np.nan


@lru_cache(maxsize=None)
def rule(topo, k, s, d, van=0):
    """Reference payloads (quadrature.py:221-398) as arrays: pair rules -> (x, y, w),
    cell/edge rules -> (x, a, w).  Node loops written out explicitly."""
    X, Y, W = [], [], []
    if topo == "ident" and d == 1:
        q, wq = gj(3, 1 - 2 * s)
        for sg in (1.0, -1.0):
            for i in range(3):
                xh = (1 + q[i]) / 2 if sg > 0 else (1 - q[i]) / 2
                X.append(xh); Y.append(xh - sg * q[i]); W.append(wq[i] * (1 - q[i]) * q[i] ** (2 * s - 1))
    elif topo == "cv" and d == 1:
        tq, tw = gj(3, 2 - 2 * s)
        vq, vw = gl(k)
        base = [(tq[i], tq[i] * vq[j], tw[i] * tq[i] ** (2 * s - 1) * vw[j]) for i in range(3) for j in range(k)]
        for T, TV, w in base:
            X.append(T); Y.append(TV); W.append(w)
        for T, TV, w in base:
            X.append(TV); Y.append(T); W.append(w)
    elif topo == "ident":
        k = min(k, 24)
        t, wt = gl(k)
        r, wr = gj(3, 1 - 2 * s)
        hexv = [(1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1)]
        for a in range(6):
            Va, Vb = np.array(hexv[a], float), np.array(hexv[(a + 1) % 6], float)
            for q in range(3):
                for j in range(k):
                    e = (1 - t[j]) * Va + t[j] * Vb
                    w1, w2 = r[q] * e
                    cx, cy = _rep(w1, w2)
                    X.append((cx, cy)); Y.append((cx - w1, cy - w2))
                    W.append(wt[j] * wr[q] * _area(w1, w2) * r[q] ** (2 * s))
    elif topo == "ce":
        k = min(k, 16)
        z, wz = gl(k)
        r, wr = gj(3, 2 - 2 * s)
        for swap in (False, True):
            for piece in ("a", "b"):
                for q in range(3):
                    rq = r[q]
                    for i in range(k):
                        for j in range(k):
                            Z, V = z[i], z[j]
                            if piece == "a":
                                zz, bb, bp, jac = rq * Z, rq * (1 - Z), rq * V, 1.0
                            else:
                                zz, bb, bp, jac = rq * V * Z, rq * V * (1 - Z), rq, V
                            al = zz + 0.5 * (1 - rq)
                            u, v = (al, bb), (al - zz, bp)
                            if swap:
                                u, v = v, u
                            X.append(u); Y.append(v)
                            W.append(wz[i] * wz[j] * jac * wr[q] * (1 - rq) * rq ** (2 * s))
    elif topo == "cv":
        kk = max(2, min(8, (k + 1) // 2 + 1))
        su, ws = gl(kk)
        r, wr = gj(3, 3 - 2 * s)
        for pieceB in (False, True):
            for q in range(3):
                rq = r[q]
                for i in range(kk):
                    for j in range(kk):
                        for l in range(kk):
                            ru = rq * su[l] if pieceB else rq
                            rv = rq if pieceB else rq * su[l]
                            X.append((ru * (1 - su[i]), ru * su[i]))
                            Y.append((rv * (1 - su[j]), rv * su[j]))
                            W.append(ws[i] * ws[j] * ws[l] * su[l] * wr[q] * rq ** (2 * s))
    elif topo == "eoc" and d == 1:
        rq, rw = gj(3, van - 2 * s)
        return rq.copy(), np.zeros(3), rw * rq ** (2 * s - van)
    elif topo == "eoc":
        zq, zw = gl(k)
        tq, tw = gl(max(3, k // 2))
        rq, rw = gj(4, van - 2 * s)
        for piece in (1, 2, 3):
            for q in range(4):
                rho = rq[q]
                for i in range(k):
                    for j in range(len(tq)):
                        Z, T = zq[i], tq[j]
                        if piece == 1:
                            zrel, beta = rho * Z, rho * (1 - Z)
                            al = zrel + T * (1 - rho)
                        elif piece == 2:
                            beta, zrel, al = rho * Z, -rho, T * (1 - rho)
                        else:
                            beta, zrel, al = rho, -rho * Z, T * (1 - rho)
                        X.append((al, beta)); Y.append(al - zrel)
                        W.append(zw[i] * tw[j] * (1 - rho) * rw[q] * rho ** (1 + 2 * s - van))
    elif topo == "te":
        kk = max(2, (k + 1) // 2 + 1)
        sq, sw = gl(kk)
        rq, rw = gj(4, 1 - 2 * s)
        for pieceB in (False, True):
            for q in range(4):
                xi = rq[q]
                for i in range(kk):
                    for j in range(kk):
                        S, Wv = sq[i], sq[j]
                        ru, ap, jac = (xi * Wv, xi, Wv) if pieceB else (xi, xi * Wv, 1.0)
                        X.append((ru * (1 - S), ru * S)); Y.append(ap)
                        W.append(sw[i] * sw[j] * jac * rw[q] * xi ** (1 + 2 * s))
    else:
        raise ValueError(topo)
    return np.array(X, float), np.array(Y, float), np.array(W, float)


# =================================================================== kernel constants
def normalisation(d, s):
    """assembly.py:57-63"""
    return float(2.0 ** (2 * s) * s * math.exp(gammaln(s + d / 2) - gammaln(1.0 - s)) / math.pi ** (d / 2))


@dataclass
class Params:
    """quadrature.py:115-131"""
    rho1: float = 2.0
    rho2: float = 2.0
    rho3: float = 2.0
    rho4: float = 2.0
    C_offset: float = 1.0
    alpha: float | None = None

    def alpha_for(self, d, s):
        return self.alpha if self.alpha is not None else (2.0 - s if d == 1 else 1.0)


def order_touch(h, n, s, d, p: Params, boundary=False):
    """quadrature.py:150-155 (+ clip :169-179)"""
    lead = p.alpha_for(d, s) / 2 + (0.25 if boundary else 0.5)
    rho = p.rho3 if boundary else p.rho1
    k = (lead * np.log(max(float(n), 2.0)) + s * np.abs(np.log(h))) / np.log(rho) - p.C_offset
    return np.clip(np.ceil(k), 2, K_MAX).astype(np.int64)


def order_far(hA, hB, dist, n, s, d, p: Params):
    """quadrature.py:157-179"""
    lead = p.alpha_for(d, s) / 2 + 0.5
    lnn = np.log(max(float(n), 2.0))
    mx = np.maximum(np.abs(np.log(hA)), np.abs(np.log(hB)))

    def br(ha, hb):
        num = lead * lnn + (s - 1) * np.abs(np.log(hb)) + mx - s * np.log(dist / hb) - p.C_offset
        return num / (np.maximum(np.log(np.maximum(dist / ha, 1e-300)), 0.0) + np.log(p.rho2))

    k = np.ceil(np.maximum(br(hA, hB), br(hB, hA)))
    return np.clip(k, 2, 9 if d == 2 else K_MAX).astype(np.int64)


# =================================================================== geometry
class Geo:
    def __init__(self, mesh, dofmap, s):
        self.d = d = mesh.vertices.shape[1]
        self.V = np.asarray(mesh.vertices, float)
        self.cells = np.asarray(mesh.cells, np.int64)
        self.P = self.V[self.cells]
        self.nc = len(self.cells)
        self.v2d = np.asarray(dofmap.vertex_to_dof, np.int64)
        self.gd = self.v2d[self.cells]
        self.n = int(dofmap.n)
        self.be = np.asarray(mesh.boundary_edges, np.int64).reshape(-1, d)
        self.bn = np.asarray(mesh.boundary_normals, float).reshape(-1, d)
        P = self.P
        if d == 1:
            self.h = np.abs(P[:, 1, 0] - P[:, 0, 0])          # mesh.py:80
            self.J = self.h.copy()
        else:
            e = [np.linalg.norm(P[:, (i + 1) % 3] - P[:, i], axis=1) for i in range(3)]
            self.h = np.maximum(e[0], np.maximum(e[1], e[2]))
            a, b = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
            self.J = np.abs(a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0])
            self.cen = P.mean(axis=1)
            self.rad = np.linalg.norm(P - self.cen[:, None, :], axis=2).max(axis=1)
        # vertex patches + cell neighbourhoods
        flat = self.cells.ravel()
        order = np.argsort(flat, kind="stable")
        self.pdata = np.repeat(np.arange(self.nc), d + 1)[order]
        self.poffs = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=len(self.V)))])
        self.s = s
        # cell quadrature (assembly.py:282-298)
        pts, w = simplex(d, XQ[d])
        self.lam = np.stack([1 - pts[:, 0], pts[:, 0]], 1) if d == 1 else \
            np.stack([1 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1)
        self.X = P[:, 0:1, :] + pts @ (P[:, 1:] - P[:, 0:1])
        self.W = np.outer(self.J, w)

    def patch(self, v):
        return self.pdata[self.poffs[v]:self.poffs[v + 1]]

    def neigh(self, c):
        return np.unique(np.concatenate([self.patch(v) for v in self.cells[c]]))

    def dist(self, a, b):
        """assembly.py:737-781, orientation (Pa, Pb) = (a, b) index arrays."""
        Pa, Pb = self.P[a], self.P[b]
        if self.d == 1:
            lo_a, hi_a = Pa[:, :, 0].min(1), Pa[:, :, 0].max(1)
            lo_b, hi_b = Pb[:, :, 0].min(1), Pb[:, :, 0].max(1)
            return np.maximum(np.maximum(lo_b - hi_a, lo_a - hi_b), 0.0)
        ra, rb = self.rad[a], self.rad[b]
        dc = np.linalg.norm(self.cen[a] - self.cen[b], axis=1)
        lower = dc - ra - rb
        out = np.maximum(lower, 0.0)
        close = np.nonzero(lower < 2.0 * (ra + rb))[0]
        if len(close):
            A_, B_ = Pa[close], Pb[close]
            best = np.full(len(close), np.inf)

            def psd(Pp, A0, B0):
                AB = B0 - A0
                t = np.sum((Pp - A0) * AB, axis=1) / np.maximum(np.sum(AB * AB, axis=1), 1e-300)
                t = np.clip(t, 0.0, 1.0)
                return np.linalg.norm(Pp - (A0 + t[:, None] * AB), axis=1)
            ed = [(0, 1), (1, 2), (2, 0)]
            for a0, a1 in ed:
                for b0, b1 in ed:
                    best = np.minimum(best, psd(A_[:, a0], B_[:, b0], B_[:, b1]))
                    best = np.minimum(best, psd(A_[:, a1], B_[:, b0], B_[:, b1]))
                    best = np.minimum(best, psd(B_[:, b0], A_[:, a0], A_[:, a1]))
                    best = np.minimum(best, psd(B_[:, b1], A_[:, a0], A_[:, a1]))
            out[close] = best
        return out

    def map(self, cells_or_P, u):
        P = self.P[cells_or_P] if not isinstance(cells_or_P, np.ndarray) or cells_or_P.ndim == 1 else cells_or_P
        return P[..., 0:1, :] + u @ (P[..., 1:, :] - P[..., 0:1, :])


# =================================================================== per-pair integrals
def hat_diff(topo, d, x, y):
    """assembly.py:99-126"""
    if d == 1:
        if topo == "ident":
            return np.stack([(1 - x) - (1 - y), x - y], 1)
        return np.stack([(1 - x) - (1 - y), x, -y], 1)
    lx = np.stack([1 - x[:, 0] - x[:, 1], x[:, 0], x[:, 1]], 1)
    ly = np.stack([1 - y[:, 0] - y[:, 1], y[:, 0], y[:, 1]], 1)
    if topo == "ident":
        return lx - ly
    if topo == "ce":
        return np.stack([lx[:, 0] - ly[:, 0], lx[:, 1] - ly[:, 1], lx[:, 2], -ly[:, 2]], 1)
    return np.stack([lx[:, 0] - ly[:, 0], lx[:, 1], lx[:, 2], -ly[:, 1], -ly[:, 2]], 1)


def jac(P):
    if P.shape[-1] == 1:
        return np.abs(P[..., 1, 0] - P[..., 0, 0])
    a, b = P[..., 1, :] - P[..., 0, :], P[..., 2, :] - P[..., 0, :]
    return np.abs(a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0])


def touching_matrix(topo, PK, PK2, s, k):
    """pair_matrices (assembly.py:143-169): absolute coordinates, then the difference."""
    d = PK.shape[-1]
    x, y, w = rule(topo, k, s, d)
    xh = x.reshape(len(w), d)
    yh = y.reshape(len(w), d)
    X = PK[0] + xh @ (PK[1:] - PK[0])
    Y = PK2[0] + yh @ (PK2[1:] - PK2[0])
    kern = np.sum((X - Y) ** 2, axis=-1) ** (-(d / 2.0 + s))
    D = hat_diff(topo, d, x if d == 1 else xh, y if d == 1 else yh)
    return (D * (kern * w)[:, None]).T @ D * (jac(PK) * jac(PK2))


def cross_block(Pa, Pb, s, k, fp32=False):
    """cross_matrices (assembly.py:172-229) for B pairs (Pa, Pb): (B, d+1, d+1)."""
    d = Pa.shape[-1]
    pts, w = simplex(d, k)
    lam = np.stack([1 - pts[:, 0], pts[:, 0]], 1) if d == 1 else \
        np.stack([1 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1)
    LW = lam * w[:, None]
    X = Pa[:, 0:1, :] + pts @ (Pa[:, 1:] - Pa[:, 0:1])
    Y = Pb[:, 0:1, :] + pts @ (Pb[:, 1:] - Pb[:, 0:1])
    r2 = np.sum((X[:, :, None, :] - Y[:, None, :, :]) ** 2, axis=-1)
    ex = -(d / 2.0 + s)
    if fp32 and len(w) ** 2 >= 1000:
        kern = (np.maximum(r2, 1e-300).astype(np.float32) ** np.float32(ex)).astype(np.float64)
    else:
        kern = r2 ** ex
    M = np.einsum("xa,bxy,yc->bac", LW, kern, LW, optimize=True)
    return M * (jac(Pa) * jac(Pb))[:, None, None]


def boundary_matrix(topo, PK, PE, ne, s, k, van):
    """boundary_pair_matrices (assembly.py:232-277), one pair; ne INWARD."""
    d = PK.shape[-1]
    ex = -(d / 2.0 + s)
    if d == 1:
        x, _, w = rule("eoc", 0, s, 1, van)
        pnt, far = PE[0, 0], PK[1, 0]
        diff = (pnt + x * (far - pnt)) - pnt
        kern = np.abs(diff) ** (2 * ex) * (ne[0] * diff)
        lam = np.stack([1 - x, x], 1)
        return (lam * (kern * w)[:, None]).T @ lam * jac(PK)
    x, a, w = rule(topo, k, s, 2, van)
    X = PK[0] + x @ (PK[1:] - PK[0])
    Y = PE[0] + a[:, None] * (PE[1] - PE[0])
    diff = X - Y
    kern = np.sum(diff ** 2, -1) ** ex * (diff @ ne)
    lam = np.stack([1 - x[:, 0] - x[:, 1], x[:, 0], x[:, 1]], 1)
    return (lam * (kern * w)[:, None]).T @ lam * jac(PK) * np.linalg.norm(PE[1] - PE[0])


def edge_flux(Xq, p0, p1, nrm, s, d):
    """edge_flux_potential (assembly.py:303-333) at points Xq (q, d)."""
    ex = -(d / 2.0 + s)
    if d == 1:
        diff = Xq[:, None, :] - p0[None, :, :]
        return np.sum(np.sum(diff * nrm[None], -1) * np.sum(diff ** 2, -1) ** ex, axis=1)
    t, w = gl(EDGE_GL)
    Y = p0[:, None, :] + t[None, :, None] * (p1 - p0)[:, None, :]
    L = np.linalg.norm(p1 - p0, axis=1)
    diff = Xq[:, None, None, :] - Y[None]
    val = np.einsum("xeqd,ed->xeq", diff, nrm) * np.sum(diff ** 2, -1) ** ex
    return np.einsum("xeq,q,e->x", val, w, L)


# =================================================================== per-cell rows
class Oracle:
    def __init__(self, mesh, dofmap, s, params: Params | None = None, integral=True, cross_fp32=False):
        self.g = Geo(mesh, dofmap, s)
        self.s = s
        self.p = params or Params()
        self.C = normalisation(self.g.d, s)
        self.integral = integral
        self.fp32 = cross_fp32
        self._touch = None
        self._bnd = None
        self.stats = dict(pairs=0, evals=0)

    # ---------------------------------------------------------------- touching pairs
    def touching_pairs(self):
        """assembly.py:412-473 + :672-680: sorted unordered pairs, canonical orders, k."""
        if self._touch is not None:
            return self._touch
        g = self.g
        out = []
        for K in range(g.nc):
            for K2 in g.neigh(K):
                if K2 <= K:
                    continue
                A, B = list(g.cells[K]), list(g.cells[K2])
                common = sorted(set(A) & set(B))
                if g.d == 1:
                    sh = common[0]
                    vK = [sh] + [v for v in A if v != sh]
                    vK2 = [sh] + [v for v in B if v != sh]
                    topo, locs = "cv", [sh, vK[1], vK2[1]]
                else:
                    vK = common + [v for v in A if v not in common]
                    vK2 = common + [v for v in B if v not in common]
                    if len(common) == 2:
                        topo, locs = "ce", vK + [vK2[2]]
                    else:
                        topo, locs = "cv", vK + vK2[1:]
                k = int(order_touch(min(g.h[K], g.h[K2]), g.n, self.s, g.d, self.p))
                out.append((K, K2, topo, k, vK, vK2, locs))
        self._touch = out
        return out

    def boundary_items(self):
        """assembly.py:796-841: (cell, edge) singular pairs in canonical order."""
        if self._bnd is not None:
            return self._bnd
        g = self.g
        items = []
        for e in range(len(g.be)):
            ev = list(g.be[e])
            cs = np.unique(np.concatenate([g.patch(v) for v in ev]))
            for c in cs:
                cv = list(g.cells[c])
                shared = sorted(set(ev) & set(cv))
                if g.d == 1:
                    topo, order, pe = "eoc", [ev[0]] + [v for v in cv if v != ev[0]], [ev[0]]
                elif len(shared) == 2:
                    topo, order, pe = "eoc", ev + [v for v in cv if v not in ev], ev
                else:
                    sv = shared[0]
                    topo, order, pe = "te", [sv] + [v for v in cv if v != sv], [sv] + [v for v in ev if v != sv]
                k = int(order_touch(g.h[c], g.n, self.s, g.d, self.p, boundary=True))
                items.append((c, e, topo, k, order, pe))
        self._bnd = items
        return items

    # ---------------------------------------------------------------- tail
    def psi(self, K):
        """Psi_K at the cell nodes (direct_tail_potential, assembly.py:985-1025), one target."""
        g = self.g
        keep = np.ones(g.nc, bool)
        keep[g.neigh(K)] = False
        src = np.nonzero(keep)[0]
        if not len(src):
            return np.zeros(g.X.shape[1])
        tgt = np.full(len(src), K)
        hi = replace(self.p, C_offset=self.p.C_offset - 4)
        ks = order_far(g.h[tgt], g.h[src], np.maximum(g.dist(tgt, src), 1e-300), g.n, self.s, g.d, hi)
        ex = -(g.d / 2.0 + self.s)
        out = np.zeros(g.X.shape[1])
        for k in np.unique(ks):
            sel = src[ks == k]
            pts, w = simplex(g.d, int(k))
            Y = g.P[sel][:, 0:1, :] + pts @ (g.P[sel][:, 1:] - g.P[sel][:, 0:1])
            r2 = np.sum((g.X[K][None, :, None, :] - Y[:, None, :, :]) ** 2, axis=-1)
            out += np.einsum("bxq,q,b->x", r2 ** ex, w, g.J[sel], optimize=True)
            self.stats["evals"] += r2.size
        self.stats["pairs"] += len(src)
        return out

    def w_in(self, K):
        """touch_T - V at the nodes of K = inward flux of the non-touching edges (:1082-1092)."""
        g = self.g
        if not len(g.be):
            return np.zeros(g.X.shape[1])
        far = ~np.isin(g.be, g.cells[K]).any(axis=1)
        e = g.be[far]
        if not len(e):
            return np.zeros(g.X.shape[1])
        p0 = g.V[e[:, 0]]
        p1 = g.V[e[:, 1]] if g.d == 2 else None
        return -edge_flux(g.X[K], p0, p1, g.bn[far], self.s, g.d)

    # ---------------------------------------------------------------- row block of one cell
    def add_cell(self, K, A, rowmap, symmetric):
        """Add to A every contribution whose row is a DoF of cell K (owner-computes).
        rowmap[i] = row of A for dof i (or -1).  symmetric: process disjoint pairs K < K2
        only and scatter both (i, j) and (j, i) (full assembly)."""
        g, C, s, d = self.g, self.C, self.s, self.g.d
        gK = g.gd[K]
        rows = [(a, rowmap[gK[a]]) for a in range(d + 1) if gK[a] >= 0 and rowmap[gK[a]] >= 0]
        ex = -(d / 2.0 + s)
        # identical pair (assembly.py:658-667)
        kT = int(order_touch(g.h[K], g.n, s, d, self.p))
        S = touching_matrix("ident", g.P[K], g.P[K], s, kT)
        # tail + boundary flux as weighted masses (assembly.py:399-407, :1079-1080, :1093-1094)
        lam, W = g.lam, g.W[K]
        Mp = np.einsum("q,qa,qb->ab", W * self.psi(K), lam, lam)
        Mb = np.einsum("q,qa,qb->ab", W * self.w_in(K), lam, lam) if self.integral else 0 * Mp
        L = 0.5 * C * S + C * Mp + C / (2 * s) * Mb
        for a, r in rows:
            for b in range(d + 1):
                if gK[b] >= 0:
                    A[r, gK[b]] += L[a, b]
        # disjoint cross term (assembly.py:693-725), reference (min, max) orientation
        keep = np.ones(g.nc, bool)
        keep[g.neigh(K)] = False
        if symmetric:
            keep[:K] = False
        src = np.nonzero(keep)[0]
        if len(src) and (rows or symmetric):
            lo, hi_ = np.minimum(src, K), np.maximum(src, K)
            ks = order_far(g.h[lo], g.h[hi_], np.maximum(g.dist(lo, hi_), 1e-300), g.n, s, d, self.p)
            for k in np.unique(ks):
                m = ks == k
                for c0 in range(0, int(m.sum()), 2048):
                    sl = np.nonzero(m)[0][c0:c0 + 2048]
                    M = cross_block(g.P[lo[sl]], g.P[hi_[sl]], s, int(k), self.fp32)
                    self.stats["evals"] += len(sl) * len(simplex(d, int(k))[1]) ** 2
                    kmin = lo[sl] == K
                    blk = np.where(kmin[:, None, None], M, M.transpose(0, 2, 1))   # [a of K, b of K2]
                    J2 = g.gd[src[sl]]
                    for a in range(d + 1):
                        ia = gK[a]
                        if ia < 0:
                            continue
                        for b in range(d + 1):
                            jb = J2[:, b]
                            ok = jb >= 0
                            if rowmap[ia] >= 0:
                                np.add.at(A, (np.full(ok.sum(), rowmap[ia]), jb[ok]), -C * blk[ok, a, b])
                            if symmetric:
                                rr = rowmap[jb[ok]]
                                good = rr >= 0
                                np.add.at(A, (rr[good], np.full(good.sum(), ia)), -C * blk[ok, a, b][good])
            self.stats["pairs"] += len(src)

    def add_touching(self, A, rowmap, cells_filter=None):
        """Touching distinct pairs, weight C = (C/2)*2 (assembly.py:690)."""
        g, C = self.g, self.C
        for (K, K2, topo, k, vK, vK2, locs) in self.touching_pairs():
            if cells_filter is not None and not (cells_filter[K] or cells_filter[K2]):
                continue
            T = touching_matrix(topo, g.V[vK], g.V[vK2], self.s, k)
            dofs = g.v2d[locs]
            for a in range(len(locs)):
                if dofs[a] < 0 or rowmap[dofs[a]] < 0:
                    continue
                for b in range(len(locs)):
                    if dofs[b] >= 0:
                        A[rowmap[dofs[a]], dofs[b]] += C * T[a, b]

    def add_boundary(self, A, rowmap):
        """Singular (cell, edge) pairs, weight C/(2s) (assembly.py:850, :1103)."""
        if not self.integral:
            return
        g, C, s = self.g, self.C, self.s
        van = 0 if s < 0.5 else 2
        for (c, e, topo, k, order, pe) in self.boundary_items():
            B = boundary_matrix(topo, g.V[order], g.V[pe], -g.bn[e], s, k, van if topo == "eoc" else 0)
            dofs = g.v2d[order]
            for a in range(len(order)):
                if dofs[a] < 0 or rowmap[dofs[a]] < 0:
                    continue
                for b in range(len(order)):
                    if dofs[b] >= 0:
                        A[rowmap[dofs[a]], dofs[b]] += C / (2 * s) * B[a, b]

    # ---------------------------------------------------------------- drivers
    def assemble(self, rows=None):
        """Dense A (rows=None) or the rows `rows` of A, as an array (len(rows), n)."""
        g = self.g
        if rows is None:
            rowmap = np.arange(g.n)
            A = np.zeros((g.n, g.n))
            for K in range(g.nc):
                self.add_cell(K, A, rowmap, symmetric=True)
            self.add_touching(A, rowmap)
            self.add_boundary(A, rowmap)
            return A
        rows = np.asarray(rows, np.int64)
        rowmap = np.full(g.n, -1, np.int64)
        rowmap[rows] = np.arange(len(rows))
        A = np.zeros((len(rows), g.n))
        need = np.zeros(g.nc, bool)
        dofs = np.nonzero(np.isin(g.v2d, rows))[0]
        for v in dofs:
            need[g.patch(v)] = True
        for K in np.nonzero(need)[0]:
            self.add_cell(K, A, rowmap, symmetric=False)
        self.add_touching(A, rowmap, cells_filter=need)
        self.add_boundary(A, rowmap)
        return A


def assemble_dense(mesh, dofmap, s, **kw):
    return Oracle(mesh, dofmap, s, **kw).assemble()


def assemble_rows(mesh, dofmap, s, rows, **kw):
    return Oracle(mesh, dofmap, s, **kw).assemble(rows)


def load_vector(mesh, dofmap, f=None, order=4):
    """assembly.py:550-570, f = 1 by default."""
    V, cells = np.asarray(mesh.vertices, float), np.asarray(mesh.cells)
    d = V.shape[1]
    pts, w = simplex(d, order)
    lam = np.stack([1 - pts[:, 0], pts[:, 0]], 1) if d == 1 else \
        np.stack([1 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1)
    P = V[cells]
    X = P[:, 0:1, :] + pts @ (P[:, 1:] - P[:, 0:1])
    fv = np.ones(X.shape[:2]) if f is None else np.asarray(f(X.reshape(-1, d))).reshape(len(P), -1)
    loc = np.einsum("cq,qa->ca", np.outer(jac(P), w) * fv, lam)
    b = np.zeros(dofmap.n)
    gd = np.asarray(dofmap.vertex_to_dof)[cells]
    np.add.at(b, gd[gd >= 0], loc[gd >= 0])
    return b


def pcg(A, b, tol=1e-8, max_iter=None, precond="jacobi"):
    """solve.py:52-109 (dense A, x0 = 0): returns (x, iterations, residual, converged)."""
    n = len(b)
    max_iter = int(10 * np.sqrt(n) + 100) if max_iter is None else max_iter
    Minv = 1.0 / np.diag(A) if precond == "jacobi" else np.ones(n)
    x = np.zeros(n)
    r = np.array(b, float)
    z = Minv * r
    p = z.copy()
    rz = r @ z
    norm0 = np.sqrt(abs(rz))
    if norm0 == 0:
        return x, 0, 0.0, True
    it, conv = 0, False
    while it < max_iter:
        Ap = A @ p
        pAp = p @ Ap
        if pAp <= 0:
            raise RuntimeError("p^T A p <= 0")
        al = rz / pAp
        x += al * p
        r -= al * Ap
        z = Minv * r
        rzn = r @ z
        it += 1
        if np.sqrt(abs(rzn)) <= tol * norm0:
            conv, rz = True, rzn
            break
        rz, p = rzn, z + (rzn / rz) * p
    return x, it, float(np.sqrt(abs(rz)) / norm0), conv


def timed_sample(mesh, dofmap, s, n_cells=16, seed=0, **kw):
    """CPU baseline: owner-computes rows of `n_cells` random target cells; returns
    (element-pair quadratures, seconds) — pairs counted like the device (tail + cross)."""
    o = Oracle(mesh, dofmap, s, **kw)
    rng = np.random.default_rng(seed)
    cells = rng.choice(o.g.nc, size=min(n_cells, o.g.nc), replace=False)
    rowmap = np.arange(o.g.n)
    A = np.zeros((o.g.n, o.g.n)) if o.g.n <= 20000 else None
    t0 = time.perf_counter()
    for K in cells:
        if A is None:
            o.psi(K)
        else:
            o.add_cell(int(K), A, rowmap, symmetric=False)
    return o.stats["pairs"], time.perf_counter() - t0
