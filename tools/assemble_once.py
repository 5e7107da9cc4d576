"""Assemble one BASELINE configuration on cuda:0 `--reps` times (profiling driver: ncu / launch
lists); prints the assembly stats of the last run as JSON."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c5", nargs="?")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--hist", action="store_true", help="also print the cross / tail order histograms")
    ap.add_argument("--square", type=int, default=0, help="unit square N x N (SW-NE) instead of a config")
    ap.add_argument("--s", type=float, default=0.5)
    a = ap.parse_args()
    from paper_1708_03912_b200 import mesh as M, assembly as A, _lib
    if a.square:
        mesh, s = M.build_unit_square_mesh(a.square), a.s
    else:
        mesh, s = M.baseline_mesh(a.config)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    st = None
    for _ in range(a.reps):
        with A.assemble_dense_device(mesh, dm, ker) as op:
            st = op.stats()
    print(json.dumps(st))
    if a.hist:
        import ctypes as C
        import numpy as np
        m = _lib.Marshal(mesh, dm, ker, None)
        hc = np.zeros(33, np.uint64)
        ht = np.zeros(33, np.uint64)
        _lib.check(_lib.load().fl_debug_order_hist(C.byref(m.mesh), C.byref(m.dofmap), C.byref(m.kernel),
                                                   C.byref(m.params), 0, hc.ctypes.data, ht.ctypes.data))
        print(json.dumps({"cross_hist": {int(k): int(v) for k, v in enumerate(hc) if v},
                          "tail_hist": {int(k): int(v) for k, v in enumerate(ht) if v}}))


if __name__ == "__main__":
    main()
