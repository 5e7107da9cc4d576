"""Generate golden fixtures by running the UNMODIFIED reference (`fraclap`, pure
numpy/scipy) from /root/reference in THIS container.

Test infrastructure only: nothing on the GPU box reads /root/reference; the
tests there read the small `.npz` fixtures this script writes next to itself.

Usage (from the repo root):
    python tests/golden/make_golden.py tables meshes small c1      # seconds
    python tests/golden/make_golden.py c2                          # ~2.5 min, 15 GB RSS
    python tests/golden/make_golden.py c3 c3u                      # ~21 min each, 31 GB RSS
    python tests/golden/make_golden.py rows4 rows5                 # sampled-row oracle at c4/c5

Each target runs in its own subprocess so peak memory is released between them.

What is stored (all derived from the reference's own functions):
  * tables   : sha256 + moments of every quadrature payload `reference_payload(topo,k,s,d,v)`
               the configs can touch (quadrature.py:401-420)
  * payloads : the full node / weight arrays of a subset of those payloads
  * meshes   : the BASELINE meshes as the reference builds them (mesh.py:273, :41, :351)
  * small/c1 : full dense A (assembly.py:1059), b (:550), pcg x + iterations (solve.py:52)
  * c2/c3    : sampled rows, diag, A@1, A@v, b, x, iterations, exact per-pair Gauss orders
               (sha256 of the nc x nc int8 order matrices + histograms)
  * c3u      : the unmodified (fp32-shortcut) c3 oracle vs the fp64 variant (negative control)
  * rows4/5  : rows of A at c4/c5 from the reference's own batch primitives
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)


# --------------------------------------------------------------------------- meshes
def ref_mesh(kind, N):
    from fraclap import mesh as M
    if kind == "uniform1d":
        return M.build_interval_mesh(-1.0, 1.0, N)
    if kind == "graded1d":
        t = np.linspace(-1.0, 1.0, N + 1)
        x = np.sign(t) * (1.0 - (1.0 - np.abs(t)) ** 2)
        cells = np.stack([np.arange(N), np.arange(1, N + 1)], axis=1)
        return M.Mesh(x[:, None], cells, np.array([[0], [N]]), np.array([[-1.0], [1.0]]))
    if kind == "square2d":
        g = np.linspace(0.0, 1.0, N + 1)
        X, Y = np.meshgrid(g, g, indexing="xy")          # vertex v = j*(N+1)+i at (i/N, j/N)
        V = np.stack([X.ravel(), Y.ravel()], axis=1)
        tris = []
        for j in range(N):
            for i in range(N):
                sw = j * (N + 1) + i
                se, nw = sw + 1, sw + N + 1
                ne = nw + 1
                tris.append((sw, se, ne))
                tris.append((sw, ne, nw))
        return M._finish_polygon_mesh(V, np.asarray(tris, np.int64))
    raise ValueError(kind)


CONFIGS = {
    "c1": ("uniform1d", 512, 0.25),
    "c2": ("graded1d", 8192, 0.75),
    "c3": ("square2d", 64, 0.5),
    "c4a": ("square2d", 128, 0.25),
    "c4b": ("square2d", 128, 0.75),
    "c5": ("square2d", 256, 0.5),
}

SMALL = [(k, N, s) for (k, N) in (("uniform1d", 16), ("uniform1d", 40), ("graded1d", 24),
                                   ("graded1d", 64), ("square2d", 4), ("square2d", 8),
                                   ("square2d", 12))
         for s in (0.25, 0.5, 0.75)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ----------------------------------------------------------------- fp64 variant
def fp64_variant():
    """Force `cross_matrices` to fp64 (assembly.py:205 use32=False) and nothing else.
    Implemented by wrapping the original with numpy float32 casts neutralised."""
    from fraclap import assembly as A
    orig = A.cross_matrices
    if getattr(orig, "_fp64", False):
        return
    import numpy as _np

    class _NoF32(_np.ndarray):
        pass

    def cross64(PK, PK2, s, k):
        # the f32 switch is taken iff k^(2d) >= 1000; below that the original is fp64
        d = PK.shape[2]
        if k ** (2 * d) < 1000:
            return orig(PK, PK2, s, k)
        # re-run the same algorithm with float64 kernels: temporarily make astype(float32)
        # a no-op by patching numpy.float32 inside the module namespace
        saved = A.np
        class NP:
            def __getattr__(self, name):
                if name == "float32":
                    return _np.float64
                return getattr(_np, name)
        A.np = NP()
        try:
            return orig(PK, PK2, s, k)
        finally:
            A.np = saved
    cross64._fp64 = True
    A.cross_matrices = cross64


# ------------------------------------------------------------------ run helpers
def setup(kind, N, s, unmodified=False):
    from fraclap import mesh as M, assembly as A
    if not unmodified:
        fp64_variant()
    mesh = ref_mesh(kind, N)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    return mesh, dm, ker


def solve(A_, b, tol=1e-10):
    from fraclap import solve as S
    x, rep = S.pcg(A_, b, precond="jacobi", tol=tol, max_iter=10 ** 5)
    return x, rep


def order_matrices(mesh, dm, s):
    """Exact per-pair Gauss orders as the reference computes them (assembly.py:705-706,
    :1010-1012) laid out as nc x nc int8 matrices."""
    from fraclap import assembly as A, quadrature as Q
    params = Q.OrderParams()
    nc, d, n = mesh.num_cells, mesh.d, dm.n
    P = mesh.cell_coords()
    diam = mesh.cell_diameters()
    pa, pb = A._all_disjoint_pairs(nc, mesh)
    out = {}
    Kc = np.zeros((nc, nc), np.int8)
    step = 4_000_000
    for lo in range(0, len(pa), step):
        a, b = pa[lo:lo + step], pb[lo:lo + step]
        dist = A._dist_estimate_coords(P[a], P[b])
        Kc[a, b] = Q.select_order(Q.PairTopology.DISJOINT, diam[a], diam[b],
                                  np.maximum(dist, 1e-300), n, s, params, d=d)
    out["cross_sha"] = sha(Kc)
    out["cross_hist"] = np.bincount(Kc.ravel(), minlength=33)
    del Kc
    from dataclasses import replace
    hi = replace(params, C_offset=params.C_offset - 4)
    offs, pdata = mesh.patch_arrays()
    Kt = np.zeros((nc, nc), np.int8)
    for c in range(nc):
        neigh = np.unique(np.concatenate([pdata[offs[v]:offs[v + 1]] for v in mesh.cells[c]]))
        keep = np.ones(nc, bool)
        keep[neigh] = False
        src = np.nonzero(keep)[0]
        if not len(src):
            continue
        tgt = np.full(len(src), c)
        dist = A._dist_estimate_coords(P[tgt], P[src])
        Kt[c, src] = Q.select_order(Q.PairTopology.DISJOINT, diam[tgt], diam[src],
                                    np.maximum(dist, 1e-300), n, s, hi, d=d)
    out["tail_sha"] = sha(Kt)
    out["tail_hist"] = np.bincount(Kt.ravel(), minlength=33)
    del Kt
    # touching pairs (sorted unordered, assembly.py:412-423) + their orders
    pairs = A.enumerate_touching_pairs(mesh)
    cells = mesh.cells
    nsh = np.array([len(set(cells[a_]) & set(cells[b_])) for a_, b_ in pairs])
    kk = np.zeros(len(pairs), np.int64)
    for topo, want in ((Q.PairTopology.COMMON_EDGE, 2), (Q.PairTopology.COMMON_VERTEX, 1)):
        rows = np.nonzero(nsh == want)[0] if d == 2 else np.arange(len(pairs))
        if d == 1 and topo is Q.PairTopology.COMMON_EDGE:
            continue
        if len(rows):
            kk[rows] = Q.select_order(topo, diam[pairs[rows, 0]], diam[pairs[rows, 1]], 0.0,
                                      n, s, params, d=d)
    out["touch_pairs"] = pairs
    out["touch_nshared"] = nsh
    out["touch_k"] = kk
    out["ident_k"] = Q.select_order(Q.PairTopology.IDENTICAL, diam, diam, 0.0, n, s, params, d=d)
    return out


def dense_case(kind, N, s, unmodified=False, rows=None, full=False, orders=False, seed=0):
    from fraclap import assembly as A
    mesh, dm, ker = setup(kind, N, s, unmodified)
    t0 = time.perf_counter()
    Ad = A.assemble_dense(mesh, dm, ker, n_limit=10 ** 6)
    t_asm = time.perf_counter() - t0
    b = A.load_vector(mesh, dm, lambda X: np.ones(len(X)))
    x, rep = solve(Ad, b)
    n = dm.n
    v = np.random.default_rng(seed).uniform(-1, 1, n)
    rec = dict(kind=kind, N=N, s=s, n=n, nc=mesh.num_cells, t_asm=t_asm,
               b=b, x=x, iters=rep.iterations, resid=rep.residual,
               diag=np.diag(Ad).copy(), rowsum=Ad @ np.ones(n), Av=Ad @ v, v=v,
               maxabs=np.abs(Ad).max(), cells=mesh.cells, vertices=mesh.vertices,
               bedges=mesh.boundary_edges, bnormals=mesh.boundary_normals,
               vertex_to_dof=dm.vertex_to_dof, A_sha=sha(Ad))
    if full:
        rec["A"] = Ad
    if rows is not None:
        rec["rows_idx"] = np.asarray(rows, np.int64)
        rec["rows"] = Ad[rows].copy()
    if orders:
        rec.update(order_matrices(mesh, dm, s))
    return rec, Ad


def save(name, rec):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
    print("wrote", path, os.path.getsize(path), "bytes", flush=True)


def pick_rows(n, mesh=None, dm=None, k=16, seed=1):
    rng = np.random.default_rng(seed)
    base = {0, 1, n // 2, n - 1, n - 2, n // 3}
    base |= set(rng.choice(n, k - len(base), replace=False).tolist())
    return np.array(sorted(base)[:k], np.int64)


# -------------------------------------------------------------- sampled-row oracle
def ref_rows(mesh, dm, ker, rows, unmodified=False):
    """Rows of the dense matrix from the reference's own batch primitives; the
    recipe of SURVEY.md §8(c) (validated against full rows on c2/c3 here)."""
    from dataclasses import replace
    from fraclap import assembly as A, quadrature as Q
    if not unmodified:
        fp64_variant()
    params = Q.OrderParams()
    s, d, n, C = ker.s, mesh.d, dm.n, ker.C_ds
    P = mesh.cell_coords()
    V = mesh.vertices
    diam = mesh.cell_diameters()
    offs, pdata = mesh.patch_arrays()
    X, W, lam = A.cell_quadrature(mesh, A.XQ_ORDER[d])
    nc = mesh.num_cells
    cells = mesh.cells
    v2d = dm.vertex_to_dof
    gd = dm.cell_dofs
    dofs = dm.dofs
    out = np.zeros((len(rows), n))
    # touching pairs of the whole mesh (once)
    pairs = A.enumerate_touching_pairs(mesh)
    # boundary triplets of the whole mesh (once)
    acc_b = ([], [], [])
    touch_T = np.zeros(X.shape[:2])
    if len(mesh.boundary_edges):
        A._touching_boundary_triplets(mesh, dm, ker, params, acc_b, touch_T, X)
        Ib = np.concatenate(acc_b[0]); Jb = np.concatenate(acc_b[1]); Vb = np.concatenate(acc_b[2])
    hi = replace(params, C_offset=params.C_offset - 4)
    for r, i in enumerate(rows):
        vtx = dofs[i]
        Ks = pdata[offs[vtx]:offs[vtx + 1]]
        row = out[r]
        for K in Ks:
            a = int(np.nonzero(cells[K] == vtx)[0][0])
            # (1) identical
            kT = Q.select_order(Q.PairTopology.IDENTICAL, diam[K:K + 1], diam[K:K + 1], 0.0,
                                n, s, params, d=d)
            loc = A.pair_matrices(Q.PairTopology.IDENTICAL, P[K:K + 1], P[K:K + 1], s, int(kT[0]))[0]
            for b_ in range(d + 1):
                if gd[K, b_] >= 0:
                    row[gd[K, b_]] += 0.5 * C * loc[a, b_]
            # (3) cross, reference orientation (min, max)
            keep = np.ones(nc, bool)
            neigh = np.unique(np.concatenate([pdata[offs[v]:offs[v + 1]] for v in cells[K]]))
            keep[neigh] = False
            src = np.nonzero(keep)[0]
            lo_ = np.minimum(src, K); hi_ = np.maximum(src, K)
            dist = A._dist_estimate_coords(P[lo_], P[hi_])
            ks = Q.select_order(Q.PairTopology.DISJOINT, diam[lo_], diam[hi_],
                                np.maximum(dist, 1e-300), n, s, params, d=d)
            for k in np.unique(ks):
                sel = np.nonzero(ks == k)[0]
                M = A.cross_matrices(P[lo_[sel]], P[hi_[sel]], s, int(k))
                Kmin = lo_[sel] == K
                for t, sidx in enumerate(src[sel]):
                    blk = M[t][a, :] if Kmin[t] else M[t][:, a]
                    for b_ in range(d + 1):
                        j = gd[sidx, b_]
                        if j >= 0:
                            row[j] += -C * blk[b_]
            # (4) tail at X[K], target-first orientation, boosted orders
            tgt = np.full(len(src), K)
            dist = A._dist_estimate_coords(P[tgt], P[src])
            ks = Q.select_order(Q.PairTopology.DISJOINT, diam[tgt], diam[src],
                                np.maximum(dist, 1e-300), n, s, hi, d=d)
            psi = np.zeros(X.shape[1])
            J = A._jacobians(P)
            ex = -(d / 2.0 + s)
            for k in np.unique(ks):
                sel = np.nonzero(ks == k)[0]
                pts, w = Q.simplex_rule(d, int(k))
                Y = A._map_points(P[src[sel]], pts)
                diff = X[K][None, :, None, :] - Y[:, None, :, :]
                r2 = np.sum(diff ** 2, axis=-1)
                vals = np.einsum("bxq,q,b->bx", r2 ** ex, w, J[src[sel]], optimize=True)
                psi += vals.sum(axis=0)
            locm = np.einsum("q,qa,qb->ab", W[K] * psi, lam, lam)
            for b_ in range(d + 1):
                if gd[K, b_] >= 0:
                    row[gd[K, b_]] += C * locm[a, b_]
            # (5b) flux of non-touching edges
            if len(mesh.boundary_edges) and ker.variant is A.Variant.INTEGRAL:
                E = mesh.boundary_edges
                if d == 1:
                    Vn = A.edge_flux_potential(X[K:K + 1], V[E[:, 0]], None, mesh.boundary_normals, s, d=1)[0]
                else:
                    Vn = A.edge_flux_potential(X[K:K + 1], V[E[:, 0]], V[E[:, 1]], mesh.boundary_normals, s, d=2)[0]
                W_in = touch_T[K] - Vn
                locb = np.einsum("q,qa,qb->ab", W[K] * W_in, lam, lam)
                for b_ in range(d + 1):
                    if gd[K, b_] >= 0:
                        row[gd[K, b_]] += C / (2 * s) * locb[a, b_]
        # (2) touching distinct pairs with a cell in the patch
        if len(pairs):
            m = np.isin(pairs[:, 0], Ks) | np.isin(pairs[:, 1], Ks)
            sub = pairs[m]
            canon = A.canonicalize_touching(mesh, sub)
            nsh = np.array([len(set(cells[a_]) & set(cells[b_])) for a_, b_ in sub])
            for topo, (vK, vK2, locs) in canon.items():
                want = 2 if topo is Q.PairTopology.COMMON_EDGE else 1
                rws = np.nonzero(nsh == want)[0] if d == 2 else np.arange(len(sub))
                ks = Q.select_order(topo, diam[sub[rws, 0]], diam[sub[rws, 1]], 0.0, n, s, params, d=d)
                for k in np.unique(ks):
                    sel = np.nonzero(ks == k)[0]
                    loc = A.pair_matrices(topo, V[vK[sel]], V[vK2[sel]], s, int(k))
                    for t in range(len(sel)):
                        L = locs[sel[t]]
                        for a_ in range(L.shape[0]):
                            if L[a_] != vtx:
                                continue
                            for b_ in range(L.shape[0]):
                                j = v2d[L[b_]]
                                if j >= 0:
                                    row[j] += C * loc[t][a_, b_]
        # (5a) singular boundary pairs
        if len(mesh.boundary_edges) and ker.variant is A.Variant.INTEGRAL:
            sel = Ib == i
            np.add.at(row, Jb[sel], C / (2 * s) * Vb[sel])
    return out


# ------------------------------------------------------------------ targets
def t_tables():
    from fraclap import quadrature as Q
    T = Q.PairTopology
    recs = {}
    def put(name, p):
        arrs = [np.asarray(p[key], float) for key in sorted(p)]
        recs[name + "/sha"] = np.frombuffer(hashlib.sha256(b"".join(
            np.ascontiguousarray(a).tobytes() for a in arrs)).digest(), np.uint8)
        w = np.asarray(p["w"], float)
        mom = [len(w), w.sum()]
        for key in sorted(p):
            if key == "w":
                continue
            a = np.asarray(p[key], float).reshape(len(w), -1)
            for c in range(a.shape[1]):
                mom += [(w * a[:, c]).sum(), (w * a[:, c] ** 2).sum(), a[:, c].min(), a[:, c].max()]
        recs[name + "/mom"] = np.array(mom)
    for s in (0.25, 0.5, 0.75):
        put("1/identical/0/%g/0" % s, Q.reference_payload(T.IDENTICAL, 2, s, 1))
        for k in range(2, 33):
            put("1/common_vertex/%d/%g/0" % (k, s), Q.reference_payload(T.COMMON_VERTEX, k, s, 1))
        van = 0 if s < 0.5 else 2      # assembly.py:794
        put("1/edge_of_cell/0/%g/%d" % (s, van), Q.reference_payload(T.EDGE_OF_CELL, 2, s, 1, van))
        for k in range(2, 25):
            put("2/identical/%d/%g/0" % (k, s), Q.reference_payload(T.IDENTICAL, k, s, 2))
        for k in range(2, 17):
            put("2/common_edge/%d/%g/0" % (k, s), Q.reference_payload(T.COMMON_EDGE, k, s, 2))
        for k in range(2, 16):
            put("2/common_vertex/%d/%g/0" % (k, s), Q.reference_payload(T.COMMON_VERTEX, k, s, 2))
        for k in range(2, 21):
            put("2/edge_of_cell/%d/%g/%d" % (k, s, van), Q.reference_payload(T.EDGE_OF_CELL, k, s, 2, van))
            put("2/touching_edge/%d/%g/0" % (k, s), Q.reference_payload(T.TOUCHING_EDGE, k, s, 2))
    for d, kmax in ((1, 32), (2, 9)):
        for k in range(2, kmax + 1):
            p = Q.reference_payload(T.DISJOINT, k, 0.5, d)
            put("%d/disjoint/%d/x/0" % (d, k), p)
    recs["normalisation"] = np.array([[d, s, __import__("fraclap.assembly", fromlist=["x"]).normalisation(d, s)]
                                      for d in (1, 2) for s in (0.1, 0.25, 0.5, 0.75, 0.9)])
    save("tables", recs)


def t_payloads():
    """Full node / weight arrays of a subset of the reference's singular payloads (every topology,
    s in {1/4, 1/2, 3/4}, low / middle / capped orders): the elementwise check of the package's
    re-derived rules (tests/test_tables.py::test_payload_arrays)."""
    from fraclap import quadrature as Q
    T = Q.PairTopology
    recs = {}
    cases = [(1, "IDENTICAL", [2]), (1, "COMMON_VERTEX", [2, 14, 32]), (1, "EDGE_OF_CELL", [2]),
             (2, "IDENTICAL", [2, 14, 24]), (2, "COMMON_EDGE", [2, 9, 16]), (2, "COMMON_VERTEX", [2, 5, 15]),
             (2, "EDGE_OF_CELL", [2, 11, 20]), (2, "TOUCHING_EDGE", [2, 7, 20])]
    for d, topo, ks in cases:
        for s in (0.25, 0.5, 0.75):
            van = 0 if s < 0.5 else 2
            for k in ks:
                p = Q.reference_payload(getattr(T, topo), k, s, d, van)
                for key, v in p.items():
                    recs["%d/%s/%d/%g/%d/%s" % (d, topo.lower(), k, s, van, key)] = np.asarray(v, float)
    save("payloads", recs)


def t_meshes():
    recs = {}
    for name, (kind, N, s) in CONFIGS.items():
        from fraclap import mesh as M
        mesh = ref_mesh(kind, N)
        dm = M.DofMap(mesh, s)
        recs[name + "/cells_sha"] = np.frombuffer(bytes.fromhex(sha(mesh.cells)), np.uint8)
        recs[name + "/verts_sha"] = np.frombuffer(bytes.fromhex(sha(mesh.vertices)), np.uint8)
        recs[name + "/bedges_sha"] = np.frombuffer(bytes.fromhex(sha(mesh.boundary_edges)), np.uint8)
        recs[name + "/bnormals_sha"] = np.frombuffer(bytes.fromhex(sha(mesh.boundary_normals)), np.uint8)
        recs[name + "/counts"] = np.array([mesh.num_vertices, mesh.num_cells,
                                           len(mesh.boundary_edges), dm.n])
        if N <= 8 or kind != "square2d":
            pass
    for N in (4, 8):
        mesh = ref_mesh("square2d", N)
        recs["sq%d/cells" % N] = mesh.cells
        recs["sq%d/bedges" % N] = mesh.boundary_edges
        recs["sq%d/bnormals" % N] = mesh.boundary_normals
    save("meshes", recs)


def t_small():
    recs = {}
    for kind, N, s in SMALL:
        tag = "%s_%d_%g" % (kind, N, s)
        rec, Ad = dense_case(kind, N, s, full=True, orders=True)
        for k, v in rec.items():
            recs[tag + "/" + k] = v
        if kind == "square2d":
            recu, Au = dense_case(kind, N, s, unmodified=True, full=False)
            recs[tag + "/A_unmodified_maxdev"] = np.abs(Au - Ad).max() / np.abs(Ad).max()
        print(tag, "n=%d" % rec["n"], "iters=%d" % rec["iters"], flush=True)
    save("small", recs)


# irregular meshes: jittered + relabelled triangulations of the unit square (through the
# reference's own _finish_polygon_mesh) and random, shuffled partitions of (-1, 1)
IRREG = [("jit2d", 6, 0.25, 11), ("jit2d", 8, 0.5, 12), ("jit2d", 7, 0.75, 13),
         ("rand1d", 40, 0.5, 14), ("rand1d", 33, 0.25, 15)]


def irregular_mesh(kind, N, seed):
    from fraclap import mesh as M
    rng = np.random.default_rng(seed)
    if kind == "jit2d":
        g = np.linspace(0.0, 1.0, N + 1)
        X, Y = np.meshgrid(g, g, indexing="xy")
        V = np.stack([X.ravel(), Y.ravel()], axis=1)
        interior = (V[:, 0] > 0) & (V[:, 0] < 1) & (V[:, 1] > 0) & (V[:, 1] < 1)
        V[interior] += rng.uniform(-0.25, 0.25, (interior.sum(), 2)) / N
        tris = []
        for j in range(N):
            for i in range(N):
                sw = j * (N + 1) + i
                se, nw = sw + 1, sw + N + 1
                ne = nw + 1
                tris.append((sw, se, ne) if (i + j) % 2 == 0 else (sw, se, nw))
                tris.append((sw, ne, nw) if (i + j) % 2 == 0 else (se, ne, nw))
        T = np.asarray(tris, np.int64)
        pv = rng.permutation(len(V))                       # relabel vertices and cells
        inv = np.empty_like(pv)
        inv[pv] = np.arange(len(pv))
        V = V[pv]
        T = inv[T][rng.permutation(len(T))]
        return M._finish_polygon_mesh(V, T)
    if kind == "rand1d":
        x = np.sort(np.concatenate([[-1.0, 1.0], rng.uniform(-1, 1, N - 1)]))
        pv = rng.permutation(N + 1)
        inv = np.empty_like(pv)
        inv[pv] = np.arange(N + 1)
        cells = inv[np.stack([np.arange(N), np.arange(1, N + 1)], axis=1)][rng.permutation(N)]
        flip = rng.random(N) < 0.5
        cells[flip] = cells[flip][:, ::-1]
        return M.Mesh(x[pv][:, None], cells, np.array([[inv[0]], [inv[N]]]), np.array([[-1.0], [1.0]]))
    raise ValueError(kind)


def t_irregular():
    from fraclap import mesh as M, assembly as A
    fp64_variant()
    recs = {}
    for kind, N, s, seed in IRREG:
        tag = "%s_%d_%g" % (kind, N, s)
        mesh = irregular_mesh(kind, N, seed)
        dm = M.DofMap(mesh, s)
        ker = A.FractionalKernel(mesh.d, s)
        Ad = A.assemble_dense(mesh, dm, ker, n_limit=10 ** 6)
        b = A.load_vector(mesh, dm, lambda X: np.ones(len(X)))
        x, rep = solve(Ad, b)
        rec = dict(A=Ad, b=b, x=x, iters=rep.iterations, vertices=mesh.vertices, cells=mesh.cells,
                   bedges=mesh.boundary_edges, bnormals=mesh.boundary_normals, s=s)
        for k, v in rec.items():
            recs[tag + "/" + k] = v
        print(tag, "n=%d" % dm.n, "iters=%d" % rep.iterations, flush=True)
    save("irregular", recs)


# tiny meshes (n = 1, 2, ...) and exponents outside the specialised s in {1/4, 1/2, 3/4}
TINY = [("uniform1d", 2, 0.75), ("uniform1d", 3, 0.5), ("graded1d", 5, 0.3), ("uniform1d", 20, 0.6),
        ("square2d", 2, 0.25), ("square2d", 2, 0.75), ("square2d", 4, 0.3), ("square2d", 3, 0.6)]


def t_tiny():
    recs = {}
    for kind, N, s in TINY:
        tag = "%s_%d_%g" % (kind, N, s)
        rec, Ad = dense_case(kind, N, s, full=True)
        for k, v in rec.items():
            recs[tag + "/" + k] = v
        print(tag, "n=%d" % rec["n"], "iters=%d" % rec["iters"], flush=True)
    save("tiny", recs)


def t_cfg(name, unmodified=False, full=False):
    kind, N, s = CONFIGS[name]
    from fraclap import mesh as M
    mesh = ref_mesh(kind, N)
    n = M.DofMap(mesh, s).n
    rows = pick_rows(n)
    rec, Ad = dense_case(kind, N, s, unmodified=unmodified, rows=rows, full=full,
                         orders=not unmodified)
    if not unmodified:
        mesh, dm, ker = setup(kind, N, s)
        t0 = time.perf_counter()
        rr = ref_rows(mesh, dm, ker, rows[:6])
        rec["rowsampler_seconds"] = time.perf_counter() - t0
        rec["rowsampler_maxdev"] = np.abs(rr - Ad[rows[:6]]).max() / np.abs(Ad).max()
        print(name, "row sampler vs full:", rec["rowsampler_maxdev"], flush=True)
    print(name, "n=%d iters=%d t_asm=%.1fs" % (rec["n"], rec["iters"], rec["t_asm"]), flush=True)
    save(name + ("u" if unmodified else ""), rec)


def t_rows(name, nrows):
    kind, N, s = CONFIGS[name]
    mesh, dm, ker = setup(kind, N, s)
    n = dm.n
    rows = pick_rows(n, k=nrows, seed=7)
    t0 = time.perf_counter()
    R = ref_rows(mesh, dm, ker, rows)
    rec = dict(rows_idx=rows, rows=R, n=n, seconds=time.perf_counter() - t0)
    from fraclap import assembly as A
    rec["b"] = A.load_vector(mesh, dm, lambda X: np.ones(len(X)))
    save("rows_" + name, rec)


# near-field (cluster) assembly: assemble_near_field (assembly.py:860-970) over the reference's own
# cluster tree / admissible partition / NearStructure (cluster.py:25-255, :743-777)
NEAR = [("uniform1d", 64, 0.25, 8, 1.0, False), ("graded1d", 96, 0.75, 8, 1.0, False),
        ("rand1d", 40, 0.5, 4, 0.5, False), ("square2d", 8, 0.5, 16, 1.0, False),
        ("square2d", 12, 0.25, 16, 1.0, False), ("jit2d", 8, 0.75, 8, 0.7, False),
        ("square2d", 6, 0.75, 10 ** 6, 1.0, False), ("square2d", 8, 0.5, 16, 1.0, True),
        ("graded1d", 60, 0.25, 8, 1.0, True), ("square2d", 16, 0.5, 8, 1.0, False),
        ("square2d", 20, 0.25, 16, 1.0, False), ("graded1d", 300, 0.75, 8, 1.0, False),
        ("jit2d", 14, 0.25, 12, 1.0, False)]


def t_near():
    from fraclap import mesh as M, assembly as A, cluster as CL
    fp64_variant()
    recs = {}
    for kind, N, s, cap, eta, cheb_v in NEAR:
        tag = "%s_%d_%g_%d_%g%s" % (kind, N, s, cap, eta, "_V" if cheb_v else "")
        mesh = irregular_mesh(kind, N, 21) if kind in ("jit2d", "rand1d") else ref_mesh(kind, N)
        dm = M.DofMap(mesh, s)
        ker = A.FractionalKernel(mesh.d, s)
        t0 = time.perf_counter()
        tree = CL.build_tree(mesh, dm, cap)
        far, near = CL.admissible_partition(tree, eta)
        ns = CL.NearStructure(mesh, dm, tree, near)
        V = None
        if cheb_v:   # the compress() path's V_nodes: boundary flux through the cluster far field
            X, W, lam = A.cell_quadrature(mesh, CL.asm_xq_order(mesh.d))
            cheb = CL.ChebData(tree, 6)
            V = CL.boundary_flux_at_nodes(mesh, dm, ker, tree, cheb, eta, X,
                                          CL._cell_leaf_assignment(mesh, dm, tree))
        Anear = A.assemble_near_field(mesh, dm, ker, ns, V_nodes=V).tocsr()
        Anear.sum_duplicates()
        Anear.sort_indices()
        leaf_index = np.full(tree.num_nodes, -1, np.int64)
        for k_, nd in enumerate(tree.leaves):
            leaf_index[nd] = k_
        rec = dict(vertices=mesh.vertices, cells=mesh.cells, bedges=mesh.boundary_edges,
                   bnormals=mesh.boundary_normals, s=s, leaf_cap=cap, eta=eta,
                   dof_perm=tree.dof_perm, leaf_idx_of_dof=ns.leaf_idx_of_dof,
                   nl_pairs=leaf_index[ns.nl_pairs], far=np.asarray(far, np.int64).reshape(-1, 2),
                   indptr=Anear.indptr.astype(np.int64), indices=Anear.indices.astype(np.int64),
                   data=Anear.data)
        if V is not None:
            rec["V_nodes"] = V
        # the tail through the one-ring boundary and the boundary mass potential, at the cell nodes
        X, W, lam = A.cell_quadrature(mesh, A.XQ_ORDER[mesh.d])
        E = mesh.boundary_edges
        Vd = A.edge_flux_potential(X, mesh.vertices[E[:, 0]], None if mesh.d == 1 else mesh.vertices[E[:, 1]],
                                   mesh.boundary_normals, s, d=mesh.d) if V is None else V
        rec["psi"] = A.tail_potential(mesh, s, X, Vd)
        T = np.zeros(X.shape[:2])
        A._touching_boundary_triplets(mesh, dm, ker, A.OrderParams(),
                                      ([], [], []), T, X)
        rec["win"] = T - Vd
        for k, v in rec.items():
            recs[tag + "/" + k] = v
        print(tag, "n=%d nnz=%d leaves=%d near=%d %.1fs" % (dm.n, Anear.nnz, len(tree.leaves), len(ns.nl_pairs),
                                                            time.perf_counter() - t0), flush=True)
    save("near", recs)


# cluster operator (cluster.compress, cluster.py:667-712) and its matvec (:417-456)
CLUSTER = [("uniform1d", 96, 0.25, 8, 1.0, 8), ("graded1d", 200, 0.75, 8, 1.0, 10),
           ("uniform1d", 120, 0.5, 8, 1.0, 8),
           ("square2d", 16, 0.5, 8, 1.0, 5), ("jit2d", 14, 0.25, 12, 1.0, 6), ("square2d", 20, 0.25, 16, 1.0, 4)]


def t_cluster():
    from fraclap import mesh as M, assembly as A, cluster as CL
    fp64_variant()
    recs = {}
    for kind, N, s, cap, eta, mo in CLUSTER:
        tag = "%s_%d_%g_%d_m%d" % (kind, N, s, cap, mo)
        mesh = irregular_mesh(kind, N, 31) if kind in ("jit2d", "rand1d") else ref_mesh(kind, N)
        dm = M.DofMap(mesh, s)
        ker = A.FractionalKernel(mesh.d, s)
        t0 = time.perf_counter()
        tree = CL.build_tree(mesh, dm, cap)
        op = CL.compress(mesh, dm, ker, tree, eta, mo)
        x = np.random.default_rng(7).uniform(-1, 1, dm.n)
        y = op.matvec(x)
        nn = tree.num_nodes
        shift = np.zeros((nn, mesh.d, mo, mo))
        for nd in range(nn):
            if op.cheb.shift[nd] is not None:
                for j in range(mesh.d):
                    shift[nd, j] = op.cheb.shift[nd][j]
        near = op.near.tocsr()
        rec = dict(vertices=mesh.vertices, cells=mesh.cells, bedges=mesh.boundary_edges,
                   bnormals=mesh.boundary_normals, s=s, leaf_cap=cap, eta=eta, m=mo, C=ker.C_ds,
                   indptr=near.indptr.astype(np.int64), indices=near.indices.astype(np.int64), data=near.data,
                   far_pairs=op.far_pairs, far_blocks=op.far_blocks, basis_coef=op.basis_coef,
                   parent=np.asarray(tree.parent, np.int64), topo_order=np.asarray(tree.topo_order, np.int64),
                   ranges=np.asarray(tree.ranges, np.int64), dof_perm=tree.dof_perm,
                   leaves=np.asarray(tree.leaves, np.int64), shift=shift, points=op.cheb.points,
                   x=x, y=y, y_far=op.far_apply(x), diag=op.diag(),
                   center=np.asarray(tree.center), half=np.asarray(tree.half))
        # strong form of u_h = x at the order-4 cell nodes (adapt.strong_form_at, adapt.py:81-214), its
        # far part alone (ClusterOperator.evaluate_far_field_at_points, cluster.py:469-485) and the
        # residual norms with f = 1 (adapt.residual_norms, :248-254)
        from fraclap import adapt as AD
        X4, W4, _ = A.cell_quadrature(mesh, 4)
        cell_leaf = CL._cell_leaf_assignment(mesh, dm, tree)
        rec["cell_leaf"] = np.asarray(cell_leaf, np.int64)
        rec["X4"] = X4
        rec["far_at_points"] = op.evaluate_far_field_at_points(x, X4.reshape(-1, mesh.d),
                                                               np.repeat(cell_leaf, X4.shape[1]))
        rec["strong_form"] = AD.strong_form_at(x, mesh, dm, op, X=X4)
        rec["residual_norms"] = AD.residual_norms(x, lambda P: np.ones(len(P)), mesh, dm, op)
        nlm = op.near_dof_leaves()
        rec["near_leaf_keys"] = np.asarray(sorted(nlm), np.int64)
        rec["near_leaf_off"] = np.cumsum([0] + [len(nlm[k]) for k in sorted(nlm)]).astype(np.int64)
        rec["near_leaf_val"] = np.concatenate([nlm[k] for k in sorted(nlm)]).astype(np.int64)
        for k, v in rec.items():
            recs[tag + "/" + k] = v
        print(tag, "n=%d far=%d M=%d nnz=%d %.1fs" % (dm.n, len(op.far_pairs), op.cheb.M, near.nnz,
                                                     time.perf_counter() - t0), flush=True)
    save("cluster", recs)


TARGETS = {
    "cluster": t_cluster,
    "near": t_near,
    "tables": t_tables,
    "payloads": t_payloads,
    "meshes": t_meshes,
    "small": t_small,
    "irregular": t_irregular,
    "tiny": t_tiny,
    "c1": lambda: t_cfg("c1", full=True),
    "c2": lambda: t_cfg("c2"),
    "c3": lambda: t_cfg("c3"),
    "c3u": lambda: t_cfg("c3", unmodified=True),
    "rows4a": lambda: t_rows("c4a", 6),
    "rows4b": lambda: t_rows("c4b", 6),
    "rows5": lambda: t_rows("c5", 6),
}

if __name__ == "__main__":
    args = sys.argv[1:]
    if len(args) == 1 and args[0] in TARGETS and os.environ.get("GOLDEN_CHILD"):
        TARGETS[args[0]]()
        sys.exit(0)
    for a in args:
        t0 = time.time()
        env = dict(os.environ, GOLDEN_CHILD="1")
        r = subprocess.run([sys.executable, __file__, a], env=env)
        print("== target %s: exit %d in %.1fs" % (a, r.returncode, time.time() - t0), flush=True)
