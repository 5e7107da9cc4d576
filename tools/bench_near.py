"""GPU box: time the near-field (cluster) assembly, assemble_near_field, on BASELINE meshes.
Usage: python tools/bench_near.py c2 c3 [c4a ...]   (leaf_cap 8 in 1D / 16 in 2D, eta 1: SPEC defaults)"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1708_03912_b200 import mesh as M, assembly as A, cluster as CL

for cfg in sys.argv[1:] or ["c2", "c3"]:
    mesh, s = M.baseline_mesh(cfg)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    t0 = time.perf_counter()
    tree = CL.build_tree(mesh, dm, 8 if mesh.d == 1 else 16)
    far, near = CL.admissible_partition(tree, 1.0)
    ns = CL.NearStructure(mesh, dm, tree, near)
    t1 = time.perf_counter()
    ts = []
    for i in range(4):
        a = time.perf_counter()
        An = A.assemble_near_field(mesh, dm, ker, ns)
        ts.append(time.perf_counter() - a)
    print("%s n=%d nnz=%d (%.3f of n^2) near leaf pairs=%d far=%d | host tree+partition %.2f s | "
          "assemble_near_field %.1f ms (min %.1f)" % (cfg, dm.n, An.nnz, An.nnz / dm.n ** 2, len(ns.nl_pairs), len(far),
                                                      t1 - t0, 1e3 * np.median(ts[1:]), 1e3 * min(ts)), flush=True)
