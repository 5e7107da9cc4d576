import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import golden
from scipy.sparse import csr_matrix
from paper_1708_03912_b200 import mesh as M, adapt as AD
from paper_1708_03912_b200.cluster import ClusterOperatorDevice
G = golden("cluster")
for key in sorted({k.split("/")[0] for k in G.files}):
    g = lambda k: G[key + "/" + k]
    mesh = M.Mesh(g("vertices"), g("cells"), g("bedges"), g("bnormals")); s = float(g("s")); dm = M.DofMap(mesh, s); n = dm.n
    keys, off, val = g("near_leaf_keys"), g("near_leaf_off"), g("near_leaf_val")
    nlm = {int(k): val[off[i]:off[i + 1]] for i, k in enumerate(keys)}
    near = csr_matrix((g("data"), g("indices"), g("indptr")), shape=(n, n))
    op = ClusterOperatorDevice.from_arrays(mesh.d, int(g("m")), g("parent"), g("topo_order"), g("ranges"), g("dof_perm"), g("shift"), g("basis_coef"), g("far_pairs"), g("far_blocks"), g("points"), s, float(g("C")), near, center=g("center"), half=g("half"), near_leaf_map=nlm)
    sf, far = AD.strong_form_at(g("x"), mesh, dm, op, X=g("X4"), return_far=True)
    rf = g("far_at_points").reshape(far.shape); ref = g("strong_form")
    bad = np.nonzero(~np.isfinite(far).all(axis=1))[0]
    print(key, "far err %.2e" % np.nanmax(np.abs(far - rf) / np.abs(rf).max()), "sf err %.2e" % np.nanmax(np.abs(sf - ref) / np.abs(ref).max()), "nan cells", bad[:10], len(bad))
    if len(bad):
        cl = op.tree_info["cell_leaf"]; print("   leaves of bad cells", cl[bad[:10]], "half", g("half")[cl[bad[:5]]], "nn", len(g("parent")))
    bad2 = np.nonzero(np.abs(sf - ref).max(axis=1) > 1e-10 * np.abs(ref).max())[0]
    if len(bad2): print("   sf bad cells", bad2[:10], len(bad2), sf[bad2[0], :2], ref[bad2[0], :2], far[bad2[0], :2], rf[bad2[0], :2])
