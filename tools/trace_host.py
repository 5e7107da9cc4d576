import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FRACLAP_TRACE"] = "1"
import torch
from paper_1708_03912_b200 import mesh as M, assembly as A
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for cfg in ["c2", "c3"]:
    mesh, s = M.baseline_mesh(cfg); dm = M.DofMap(mesh, s); ker = A.FractionalKernel(mesh.d, s)
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = A.assemble_dense_device(mesh, dm, ker, stream=st.cuda_stream)
        t1 = time.perf_counter()
        st_ = op.stats()
        t2 = time.perf_counter()
        op.free()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(cfg, "call %.3f ms, stats %.3f ms, free %.3f ms, lib ms_total %.3f" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, st_["ms_total"]), flush=True)
