"""GPU box: cluster matvec at a BASELINE config through compress (SPEC defaults), timed with CUDA
events; FRACLAP_COOP_PER_SM=0 selects the per-phase launches instead of the cooperative kernel."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_1708_03912_b200 import mesh as M, assembly as A, cluster as CL, _lib


class Stats:
    pass


cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
mesh, s = M.baseline_mesh(cfg)
dm = M.DofMap(mesh, s)
st = Stats(); st.h_min = float(mesh.cell_diameters().min()); st.dim = mesh.d
op = CL.compress(mesh, dm, A.FractionalKernel(mesh.d, s), CL.build_tree(mesh, dm, 8 if mesh.d == 1 else 16), 1.0,
                 CL.choose_order(st))
xd = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, dm.n)).cuda(); yd = torch.empty_like(xd)
L = _lib.load()
ev = []
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    _lib.check(L.fl_cluster_matvec(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, 1))
    e1.record(); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1))
print("%s coop_per_sm=%s matvec %.1f us (median of %d)" % (cfg, os.environ.get("FRACLAP_COOP_PER_SM", "1"),
                                                        1e3 * np.median(ev[min(5, reps - 1):]), reps))
if len(sys.argv) > 3:                      # bitwise: cooperative schedule vs per-level launches
    y1 = yd.cpu().numpy()
    ok = np.array_equal(y1, np.load(sys.argv[3])) if os.path.exists(sys.argv[3]) else np.save(sys.argv[3], y1)
    print("bitwise equal to %s: %s" % (sys.argv[3], ok))
