import os, sys, time
os.environ["FRACLAP_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_1708_03912_b200 import mesh as M, assembly as A
mesh, s = M.baseline_mesh("c2"); dm = M.DofMap(mesh, s); ker = A.FractionalKernel(1, s); n = dm.n
out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
for i in range(4):
    t0 = time.perf_counter(); A.assemble_dense(mesh, dm, ker, n_limit=10 ** 7, out=out)
    print("e2e ms %.2f" % (1e3 * (time.perf_counter() - t0)), file=sys.stderr, flush=True)
