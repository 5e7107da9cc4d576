"""Build the reference's cluster operator (cluster.compress, unmodified reference, THIS container)
for a BASELINE mesh and save its arrays for tools/bench_cluster.py (timing only; parity is
tests/test_gpu_parity.py::test_cluster_matvec_matches_reference on committed fixtures).
Usage: python tools/make_cluster_op.py c2 [m]  ->  bench_data/cluster_<cfg>.npz (git-ignored)"""
import os, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden"))
import numpy as np
from make_golden import ref_mesh, fp64_variant
from fraclap import mesh as M, assembly as A, cluster as CL

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
kind, N, s = {"c1": ("uniform1d", 512, 0.25), "c2": ("graded1d", 8192, 0.75), "c3": ("square2d", 64, 0.5)}[cfg]
fp64_variant()
mesh = ref_mesh(kind, N)
dm = M.DofMap(mesh, s)
ker = A.FractionalKernel(mesh.d, s)
cap = 8 if mesh.d == 1 else 16
t0 = time.perf_counter()
tree = CL.build_tree(mesh, dm, cap)
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8
op = CL.compress(mesh, dm, ker, tree, 1.0, m)
t1 = time.perf_counter()
x = np.random.default_rng(0).uniform(-1, 1, dm.n)
ts = []
for i in range(5):
    a = time.perf_counter(); y = op.matvec(x); ts.append(time.perf_counter() - a)
from fraclap import adapt as AD
a = time.perf_counter(); sf = AD.strong_form_at(x, mesh, dm, op); ref_sf_s = time.perf_counter() - a
nlm = op.near_dof_leaves()
nn = tree.num_nodes
shift = np.zeros((nn, mesh.d, m, m))
for nd in range(nn):
    if op.cheb.shift[nd] is not None:
        for j in range(mesh.d):
            shift[nd, j] = op.cheb.shift[nd][j]
near = op.near.tocsr()
os.makedirs("bench_data", exist_ok=True)
np.savez("bench_data/cluster_%s.npz" % cfg, d=mesh.d, m=m, s=s, C=ker.C_ds, parent=np.asarray(tree.parent),
         topo_order=np.asarray(tree.topo_order), ranges=np.asarray(tree.ranges), dof_perm=tree.dof_perm,
         shift=shift, basis_coef=op.basis_coef, far_pairs=op.far_pairs, points=op.cheb.points,
         indptr=near.indptr, indices=near.indices, data=near.data, x=x, y=y,
         ref_matvec_s=np.median(ts), ref_compress_s=t1 - t0, cores=os.cpu_count(),
         center=np.asarray(tree.center), half=np.asarray(tree.half), strong_form=sf, ref_strong_form_s=ref_sf_s,
         near_leaf_keys=np.asarray(sorted(nlm), np.int64),
         near_leaf_off=np.cumsum([0] + [len(nlm[k]) for k in sorted(nlm)]).astype(np.int64),
         near_leaf_val=np.concatenate([nlm[k] for k in sorted(nlm)]).astype(np.int64),
         vertices=mesh.vertices, cells=mesh.cells, bedges=mesh.boundary_edges, bnormals=mesh.boundary_normals)
print(cfg, "n", dm.n, "far pairs", len(op.far_pairs), "nnz", near.nnz, "compress %.1f s" % (t1 - t0),
      "reference matvec %.2f ms" % (1e3 * np.median(ts)), "strong form %.2f s" % ref_sf_s)
