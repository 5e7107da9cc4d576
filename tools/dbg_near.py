import sys, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import golden
from paper_1708_03912_b200 import mesh as M, assembly as A, cluster as CL, _lib
G = golden("near")
for key in sorted({k.split("/")[0] for k in G.files}):
    mesh = M.Mesh(G[key + "/vertices"], G[key + "/cells"], G[key + "/bedges"], G[key + "/bnormals"])
    s = float(G[key + "/s"]); dm = M.DofMap(mesh, s); ker = A.FractionalKernel(mesh.d, s)
    V = G[key + "/V_nodes"] if key + "/V_nodes" in G.files else None
    m = _lib.Marshal(mesh, dm, ker, None); _, _, tb = A._tables(mesh, dm, s, None)
    q = 6 if mesh.d == 1 else 16
    psi = np.empty((mesh.num_cells, q)); win = np.empty((mesh.num_cells, q))
    _lib.check(_lib.load().fl_debug_ring_tail(C.byref(m.mesh), C.byref(m.dofmap), C.byref(m.kernel), C.byref(m.params), C.byref(tb),
               None if V is None else np.ascontiguousarray(V).ctypes.data, 0, psi.ctypes.data, win.ctypes.data))
    rp, rw = G[key + "/psi"], G[key + "/win"]
    ep = np.abs(psi - rp).max() / np.abs(rp).max(); ew = np.abs(win - rw).max() / max(np.abs(rw).max(), 1e-300)
    bad = np.nonzero(np.abs(psi - rp).max(axis=1) > 1e-9 * np.abs(rp).max())[0]
    print(key, "psi rel %.2e win rel %.2e" % (ep, ew), "bad cells", bad[:12], len(bad))
    if len(bad):
        c = bad[0]; print("   cell", c, mesh.cells[c], "ours", psi[c, :3], "ref", rp[c, :3])
