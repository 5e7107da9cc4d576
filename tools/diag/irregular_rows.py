"""Diagnostic: sampled rows of irregular 2D meshes vs the oracle (deviation, cross path taken)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from conftest import make_mesh
from paper_1708_03912_b200 import mesh as M, assembly as A
from oracle import fraclap_oracle as O
CASES = (("jitter2d", 32, 0.5), ("jitter2d", 40, 0.75), ("graded2d", 32, 0.5), ("graded2d", 40, 0.25),
         ("graded2d", 48, 0.75), ("square2d", 40, 0.5))
if len(sys.argv) > 1:          # kind:N:s ...
    CASES = tuple((a.split(":")[0], int(a.split(":")[1]), float(a.split(":")[2])) for a in sys.argv[1:])
for kind, N, s in CASES:
    mesh = make_mesh(kind, N)
    dm = M.DofMap(mesh, s)
    rows = [0, 3, dm.n // 3, dm.n // 2 + 1, dm.n - 2]
    with A.assemble_dense_device(mesh, dm, A.FractionalKernel(2, s)) as op:
        got = op.rows(np.array(rows)); st = op.stats()
    ref = O.assemble_rows(mesh, dm, s, rows)
    d = np.abs(got - ref).max() / np.abs(ref).max()
    print("%-9s N=%d s=%.2f: rel dev %.2e  fallback %d scale_exp %d  tail block evals %.2e of %.2e" %
          (kind, N, s, d, st["cross_fallback"], st["cross_scale_exp"], st["evals_tail_block"], st["evals_tail"]))
