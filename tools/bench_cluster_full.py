"""GPU box: the whole cluster path with this package only — tree, compress (device near field and
far blocks), matvec, strong form — on BASELINE meshes (SPEC defaults: leaf cap 8 / 16, eta 1,
m = choose_order)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_1708_03912_b200 import mesh as M, assembly as A, cluster as CL, adapt as AD, _lib


class Stats:
    pass


for cfg in sys.argv[1:] or ["c2", "c3"]:
    mesh, s = M.baseline_mesh(cfg)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    st = Stats(); st.h_min = float(mesh.cell_diameters().min()); st.dim = mesh.d
    m = CL.choose_order(st)
    t0 = time.perf_counter()
    tree = CL.build_tree(mesh, dm, 8 if mesh.d == 1 else 16)
    t1 = time.perf_counter()
    op = CL.compress(mesh, dm, ker, tree, 1.0, m)
    t2 = time.perf_counter()
    op.free()                                   # the first call carries the CUDA context set-up
    tw = time.perf_counter()
    op = CL.compress(mesh, dm, ker, tree, 1.0, m)
    t_cold, t_warm = t2 - t1, time.perf_counter() - tw
    x = np.random.default_rng(0).uniform(-1, 1, dm.n)
    xd = torch.from_numpy(x).cuda(); yd = torch.empty_like(xd)
    L = _lib.load()
    ev = []
    for i in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        _lib.check(L.fl_cluster_matvec(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, 1))
        e1.record(); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1))
    X4, _ = AD.cell_nodes(mesh, 4)
    AD.strong_form_at(x, mesh, dm, op, X=X4)
    a = time.perf_counter(); AD.strong_form_at(x, mesh, dm, op, X=X4); t_sf = time.perf_counter() - a
    print("%s n=%d m=%d far pairs=%d near nnz=%d | tree %.2f s, compress %.2f s (first call %.2f s) | matvec %.1f us | strong form %.1f ms"
          % (cfg, dm.n, m, len(op.far_pairs), op.near.nnz, t1 - t0, t_warm, t_cold, 1e3 * np.median(ev[5:]), 1e3 * t_sf),
          flush=True)
    op.free()
