"""GPU box: time the device cluster matvec (ClusterOperatorDevice) on an operator saved by
tools/make_cluster_op.py, against the reference's host matvec time and the dense matvec."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from scipy.sparse import csr_matrix
from paper_1708_03912_b200 import _lib
from paper_1708_03912_b200.cluster import ClusterOperatorDevice

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
Z = np.load("bench_data/cluster_%s.npz" % cfg)
n = len(Z["x"])
near = csr_matrix((Z["data"], Z["indices"], Z["indptr"]), shape=(n, n))
keys, off, val = Z["near_leaf_keys"], Z["near_leaf_off"], Z["near_leaf_val"]
nlm = {int(k): val[off[i]:off[i + 1]] for i, k in enumerate(keys)}
op = ClusterOperatorDevice.from_arrays(int(Z["d"]), int(Z["m"]), Z["parent"], Z["topo_order"], Z["ranges"],
                                       Z["dof_perm"], Z["shift"], Z["basis_coef"], Z["far_pairs"], None, Z["points"],
                                       float(Z["s"]), float(Z["C"]), near, center=Z["center"], half=Z["half"],
                                       near_leaf_map=nlm)
y = op.matvec(Z["x"])
print("rel diff vs reference y: %.2e" % (np.abs(y - Z["y"]).max() / np.abs(Z["y"]).max()))
ts = []
for i in range(20):
    a = time.perf_counter(); op.matvec(Z["x"]); ts.append(time.perf_counter() - a)
xd = torch.from_numpy(Z["x"]).cuda(); yd = torch.empty_like(xd)
L = _lib.load()
ev = []
for i in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    _lib.check(L.fl_cluster_matvec(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, 1))
    e1.record(); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1))
print("%s n=%d far pairs=%d: device matvec %.1f us (events), host-array matvec %.1f us; reference host matvec %.2f ms "
      "(%d cores) -> %.0fx" % (cfg, n, len(Z["far_pairs"]), 1e3 * np.median(ev[5:]), 1e6 * np.median(ts[3:]),
                               1e3 * float(Z["ref_matvec_s"]), int(Z["cores"]),
                               float(Z["ref_matvec_s"]) / (1e-3 * np.median(ev[5:]))))
# strong form of u_h = x at the order-4 cell nodes (adapt.strong_form_at)
from paper_1708_03912_b200 import mesh as Mm, adapt as AD
mesh = Mm.Mesh(Z["vertices"], Z["cells"], Z["bedges"], Z["bnormals"])
dm = Mm.DofMap(mesh, float(Z["s"]))
X4, _ = AD.cell_nodes(mesh, 4)
sf = AD.strong_form_at(Z["x"], mesh, dm, op, X=X4)
print("strong form rel diff vs reference: %.2e" % (np.abs(sf - Z["strong_form"]).max() / np.abs(Z["strong_form"]).max()))
ts = []
for i in range(5):
    a = time.perf_counter(); AD.strong_form_at(Z["x"], mesh, dm, op, X=X4); ts.append(time.perf_counter() - a)
print("%s strong form: %.2f ms (public call) vs reference %.2f s -> %.0fx" % (
    cfg, 1e3 * np.median(ts[1:]), float(Z["ref_strong_form_s"]), float(Z["ref_strong_form_s"]) / np.median(ts[1:])))
