"""Diagnostic: sampled rows of a jittered mesh under the cross / tail path switches vs the oracle."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
from conftest import make_mesh
from paper_1708_03912_b200 import mesh as M, assembly as A
mesh = make_mesh('jitter2d', int(sys.argv[2])); s = float(sys.argv[3])
dm = M.DofMap(mesh, s)
rows = [3, dm.n // 3, dm.n // 2 + 1, dm.n - 2]
with A.assemble_dense_device(mesh, dm, A.FractionalKernel(2, s)) as op:
    np.save(sys.argv[4], op.rows(np.array(rows)))
    st = op.stats()
    print('scale_exp', st['cross_scale_exp'], 'fallback', st['cross_fallback'])
"""
N, s = int(sys.argv[1]), float(sys.argv[2])
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from conftest import make_mesh
from paper_1708_03912_b200 import mesh as M
from oracle import fraclap_oracle as O
mesh = make_mesh("jitter2d", N)
dm = M.DofMap(mesh, s)
rows = [3, dm.n // 3, dm.n // 2 + 1, dm.n - 2]
ref = O.assemble_rows(mesh, dm, s, rows)
scale = np.abs(ref).max()
for env in ("", "FRACLAP_CROSS2D_FALLBACK=1", "FRACLAP_CROSS2D=tiles"):
    e = dict(os.environ)
    if env:
        k, v = env.split("=")
        e[k] = v
    out = "/tmp/jr.npy"
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(N), str(s), out], env=e, capture_output=True, text=True)
    if r.returncode:
        print(env, "FAILED", r.stderr[-500:])
        continue
    print(r.stdout.strip())
    got = np.load(out)
    d = np.abs(got - ref)
    i, j = np.unravel_index(d.argmax(), d.shape)
    nbad = int((d > 1e-10 * scale).sum())
    print("%-24s max dev %.3e (rel max %.3e) at row %d col %d: got %.10e ref %.10e; entries over tol: %d" %
          (env or "default", d.max(), d.max() / scale, rows[i], j, got[i, j], ref[i, j], nbad))
