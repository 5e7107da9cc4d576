"""B200-native dense hot path of Ainsworth & Glusa's FEM for the integral fractional Laplacian.

Drop-in entry points mirroring the reference package `fraclap`:
  assembly.assemble_dense(mesh, dofmap, kernel, params=None, n_limit=DENSE_LIMIT)
  solve.pcg(op, b, precond="jacobi", tol=1e-8, max_iter=None, x0=None)
plus assembly.assemble_dense_device (matrix kept in HBM) and distributed.* (row-block
sharding over torch.distributed / NCCL).
"""
from .quadrature import OrderParams, PairTopology, QuadratureError, select_order  # noqa: F401
from .mesh import Mesh, DofMap, MeshError  # noqa: F401
from .assembly import (AssemblyError, FractionalKernel, Variant, normalisation,  # noqa: F401
                       assemble_dense, assemble_dense_device, load_vector, DENSE_LIMIT)
from .solve import SolverError, SolveReport, pcg  # noqa: F401
from .operator import DenseDeviceOperator  # noqa: F401

__version__ = "0.1.0"
