"""GPU box: e2e (assemble_dense into pinned host memory) at c2 against FRACLAP_HOST_BANDS."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_1708_03912_b200 import mesh as M, assembly as A

mesh, s = M.baseline_mesh(sys.argv[1] if len(sys.argv) > 1 else "c2")
dm = M.DofMap(mesh, s); ker = A.FractionalKernel(mesh.d, s); n = dm.n
out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
for nb in ["1", "4", "6", "8", "12", "16", "24"]:
    os.environ["FRACLAP_HOST_BANDS"] = nb
    ts = []
    for i in range(6):
        t0 = time.perf_counter(); A.assemble_dense(mesh, dm, ker, n_limit=10 ** 7, out=out); ts.append(time.perf_counter() - t0)
    print("bands", nb, "e2e ms %.2f (min %.2f)" % (1e3 * np.median(ts[1:]), 1e3 * min(ts)), flush=True)
