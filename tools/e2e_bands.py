"""GPU box: e2e (assemble_dense into pinned host memory) at c2 against FRACLAP_HOST_BANDS, with and
without an L2 flush between calls (the bench flushes), plus the raw D2H copy rate."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_1708_03912_b200 import mesh as M, assembly as A

mesh, s = M.baseline_mesh(sys.argv[1] if len(sys.argv) > 1 else "c2")
dm = M.DofMap(mesh, s); ker = A.FractionalKernel(mesh.d, s); n = dm.n
out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for nb in ["1", "8"]:
    os.environ["FRACLAP_HOST_BANDS"] = nb
    for fl in (False, True):
        ts = []
        for i in range(7):
            if fl:
                flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter(); A.assemble_dense(mesh, dm, ker, n_limit=10 ** 7, out=out); ts.append(time.perf_counter() - t0)
        print("bands", nb, "flush", fl, "e2e ms %.2f (min %.2f)" % (1e3 * np.median(ts[1:]), 1e3 * min(ts)), flush=True)
op = A.assemble_dense_device(mesh, dm, ker)
for i in range(3):
    t0 = time.perf_counter(); op.to_host(out); dt = time.perf_counter() - t0
    print("to_host ms %.2f = %.1f GB/s" % (1e3 * dt, 8.0 * n * n / dt / 1e9), flush=True)
