"""GPU box: where cluster.compress spends its time (cProfile, top entries)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1708_03912_b200 import mesh as M, assembly as A, cluster as CL
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
mesh, s = M.baseline_mesh(cfg); dm = M.DofMap(mesh, s); ker = A.FractionalKernel(mesh.d, s)
tree = CL.build_tree(mesh, dm, 8 if mesh.d == 1 else 16)
m = int(sys.argv[2]) if len(sys.argv) > 2 else 5
CL.compress(mesh, dm, ker, tree, 1.0, m)          # warm-up (library load, JIT of nothing)
pr = cProfile.Profile(); pr.enable()
op = CL.compress(mesh, dm, ker, tree, 1.0, m)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
