"""Jacobi-preconditioned CG — drop-in for `fraclap.solve.pcg` (solve.py:52-109).

For a DenseDeviceOperator (or a dense array, which is uploaded once) the whole loop runs in
libfraclap_b200.so: fused matvec / dot / vector kernels captured in a CUDA graph, scalars on
the device, the same stopping rule sqrt|r.z| <= tol * sqrt|r0.z0| (solve.py:96) and the
same iteration count.  Operators that live only on the host are not part of the dense device
path and are refused (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .operator import DenseDeviceOperator


class SolverError(RuntimeError):
    """solve.py:15."""


@dataclass
class SolveReport:
    """solve.py:38-45 (+ the true relative residual ||b - Ax|| / ||b||)."""
    iterations: int
    residual: float
    seconds: float
    converged: bool = True
    lanczos_alpha: tuple = ()
    lanczos_beta: tuple = ()
    true_residual: float = float("nan")


class LinearOperatorHandle:
    """solve.py:19-35: apply + exact diagonal."""

    def __init__(self, apply, diag, n=None):
        self.apply = apply
        self._diag = np.asarray(diag, float)
        self.n = len(self._diag) if n is None else n

    @classmethod
    def from_matrix(cls, A):
        if hasattr(A, "matvec"):
            return cls(A.matvec, A.diag())
        raise TypeError("host matrices are uploaded by pcg(); wrap other operators yourself")

    def diag(self):
        return self._diag


def pcg(op, b, precond="jacobi", tol=1e-8, max_iter=None, x0=None, record_lanczos=False):
    """Conjugate gradients with Jacobi preconditioning; returns (x, SolveReport)."""
    if record_lanczos:
        raise NotImplementedError("record_lanczos is outside the dense device path")
    if isinstance(op, np.ndarray):
        with DenseDeviceOperator.from_host(op) as dev:      # Ad @ x of solve.py:31-32, on the GPU
            return pcg(dev, b, precond, tol, max_iter, x0)
    from .cluster import ClusterOperatorDevice
    if isinstance(op, ClusterOperatorDevice):
        return _pcg_cluster(op, b, precond, tol, max_iter, x0)
    if not isinstance(op, DenseDeviceOperator):
        raise TypeError("pcg expects a DenseDeviceOperator (assemble_dense_device), a "
                        "ClusterOperatorDevice or a dense ndarray; host operators are not on the device path")
    if not op.full:
        raise ValueError("a row-block operator needs distributed.pcg_sharded")
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    if n != op.n:
        raise ValueError("b has length %d, operator is %d x %d" % (n, op.n, op.n))
    if max_iter is None:
        max_iter = int(10 * np.sqrt(n) + 100)                    # solve.py:61-62
    if precond in (None, "none"):
        pc = 0
    elif precond == "jacobi":
        pc = 1
    else:
        raise ValueError("precond must be 'jacobi' or None on the device path")
    x = np.empty(n)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    rep = _lib.fl_solve_report()
    t0 = time.perf_counter()
    _lib.check(_lib.load().fl_pcg(op.handle, b.ctypes.data, None if x0a is None else x0a.ctypes.data,
                                  float(tol), int(max_iter), pc, x.ctypes.data, C.byref(rep)))
    return x, SolveReport(int(rep.iterations), float(rep.residual), time.perf_counter() - t0,
                          bool(rep.converged), true_residual=float(rep.true_residual))


class _OneRank:
    """torch.distributed stand-in for a single process (pcg_sharded's exchange steps are identities)."""

    class ReduceOp:
        MAX = SUM = None

    @staticmethod
    def get_rank(group=None):
        return 0

    @staticmethod
    def get_world_size(group=None):
        return 1

    @staticmethod
    def all_reduce(t, op=None, group=None):
        return None

    @staticmethod
    def all_gather_into_tensor(out, inp, group=None, async_op=False):
        out.copy_(inp)


def _pcg_cluster(op, b, precond, tol, max_iter, x0=None):
    """The same Jacobi PCG (solve.py:52-109) on a ClusterOperatorDevice: device vectors, the
    device-scalar CG steps of libfraclap_b200 (fl_cg_*) and the H-matrix matvec
    (fl_cluster_matvec_async on torch's stream), run on the operator's own device."""
    import torch
    from .distributed import TorchDeviceBackend, pcg_sharded

    class _Backend(TorchDeviceBackend):
        def __init__(self, cop):
            super().__init__(None)
            self.cop = cop

        def matvec_diag(self, p_local):
            pass                                  # one rank: nothing to overlap

        def matvec_rest(self, p_full, p_local, Ap):
            # enqueued on torch's current stream, no host synchronisation
            _lib.check(self.lib.fl_cluster_matvec_async(self.cop.handle, self._p(p_full), self._p(Ap), self.stream))
            _lib.check(self.lib.fl_cg_dot_parts(self.S, self._p(p_local), self._p(Ap), self.stream))

    b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    if n != op.n:
        raise ValueError("b has length %d, operator is %d x %d" % (n, op.n, op.n))
    if precond not in ("jacobi", None, "none"):
        raise ValueError("precond must be 'jacobi' or None on the device path")
    if x0 is not None and np.shape(x0) != (n,):
        raise ValueError("x0 must have shape (%d,)" % n)
    t0 = time.perf_counter()
    with torch.cuda.device(op.device):
        x, rep = pcg_sharded(_Backend(op), b, op.diag(), [(0, n)], n, _OneRank, tol=tol, max_iter=max_iter,
                             precond="jacobi" if precond == "jacobi" else None, x0_local=x0)
        x = x.cpu().numpy()
    return x, SolveReport(int(rep["iterations"]), float(rep.get("residual", float("nan"))),
                          time.perf_counter() - t0, bool(rep["converged"]))
