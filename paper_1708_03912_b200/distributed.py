"""Row-block sharding over the GPUs of one box (torch.distributed / NCCL plumbing).

Assembly is owner-computes: rank g assembles the DoF rows R_g = [r0, r1) of A on its own
GPU (fl_assemble_dense with a row range); nothing is exchanged.  The CG solve
(solve.py:52-109) runs the sharded matvec y_g = A[R_g, :] p with one all-gather of the
search direction p per iteration and one all-reduce of the two CG dot products; the
vector updates are fused device kernels of libfraclap_b200.so.

`pcg_sharded` is written against a tiny backend interface so the same control logic is
exercised on CPU with gloo in tests/test_distributed.py.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib


def shard_rows(n: int, world: int, weights=None):
    """Contiguous row blocks [(r0, r1)] for `world` ranks, balanced by `weights` (per-row
    work estimate; default uniform)."""
    if world <= 0:
        raise ValueError("world must be positive")
    if weights is None:
        cuts = [round(n * g / world) for g in range(world + 1)]
    else:
        w = np.cumsum(np.asarray(weights, float))
        tot = w[-1] if len(w) else 0.0
        cuts = [0] + [min(n, int(np.searchsorted(w, tot * g / world)) + 1) for g in range(1, world)] + [n]
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


class TorchDeviceBackend:
    """Device vectors as torch CUDA tensors; matvec and fused updates in libfraclap_b200."""

    def __init__(self, op, stream=None):
        import torch
        self.torch = torch
        self.op = op
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream().cuda_stream
        self.lib = _lib.load()

    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64, device=self.dev)

    def from_numpy(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a), dtype=self.torch.float64).to(self.dev)

    def matvec(self, p_full, out_local):
        self.op.matvec_device(p_full.data_ptr(), out_local.data_ptr(), self.stream)

    def dot(self, a, b):
        out = self.zeros(1)
        _lib.check(self.lib.fl_dot_async(a.numel(), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(self.stream)))
        return out

    def update(self, alpha, x, r, z, p, Ap, minv):
        out = self.zeros(1)
        _lib.check(self.lib.fl_cg_update_async(x.numel(), float(alpha), C.c_void_p(x.data_ptr()),
                                               C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()),
                                               C.c_void_p(p.data_ptr()), C.c_void_p(Ap.data_ptr()),
                                               C.c_void_p(minv.data_ptr()), C.c_void_p(out.data_ptr()),
                                               C.c_void_p(self.stream)))
        return out

    def xpby(self, z, beta, p):
        _lib.check(self.lib.fl_xpby_async(z.numel(), C.c_void_p(z.data_ptr()), float(beta),
                                          C.c_void_p(p.data_ptr()), C.c_void_p(self.stream)))

    def item(self, t):
        return float(t.item())


def pcg_sharded(backend, b_local, diag_local, rows, n, dist, group=None, tol=1e-8, max_iter=None,
                precond="jacobi"):
    """Jacobi PCG with A distributed by contiguous row blocks `rows` = [(r0, r1)] per rank.
    Same recurrences and stopping rule as solve.py:52-109.  Returns (x_local, report dict)."""
    import torch
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    r0, r1 = rows[rank]
    m = r1 - r0
    if max_iter is None:
        max_iter = int(10 * np.sqrt(n) + 100)
    d = np.asarray(diag_local, float)
    if precond == "jacobi":
        bad = torch.tensor([float(np.any(d <= 0))], dtype=torch.float64)
        bad = backend.from_numpy(bad.numpy())
        dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
        if backend.item(bad) > 0:
            from .solve import SolverError
            raise SolverError("nonpositive diagonal; operator not SPD")
        minv = backend.from_numpy(1.0 / np.where(d > 0, d, 1.0))
    else:
        minv = backend.from_numpy(np.ones(m))
    blk = max(r1_ - r0_ for r0_, r1_ in rows)
    lda = ((n + 31) // 32) * 32
    t0 = time.perf_counter()
    x = backend.zeros(m)
    r = backend.from_numpy(b_local)
    z = backend.zeros(m)
    p_local = backend.zeros(m)
    Ap = backend.zeros(m)
    # z = minv r, p = z, rz = r.z  (alpha = 0 leaves x, r unchanged)
    rz_t = backend.update(0.0, x, r, z, p_local, Ap, minv)
    dist.all_reduce(rz_t, group=group)
    rz = backend.item(rz_t)
    p_local.copy_(z)
    norm0 = np.sqrt(abs(rz))
    if norm0 == 0:
        return x, dict(iterations=0, residual=0.0, seconds=time.perf_counter() - t0, converged=True)
    gather_in = backend.zeros(blk)
    gather_out = backend.zeros(blk * world)
    p_full = backend.zeros(lda)
    it, converged = 0, False
    while it < max_iter:
        gather_in[:m].copy_(p_local)
        dist.all_gather_into_tensor(gather_out, gather_in, group=group)
        for g, (a, e) in enumerate(rows):
            p_full[a:e].copy_(gather_out[g * blk:g * blk + (e - a)])
        backend.matvec(p_full, Ap)
        pAp_t = backend.dot(p_local, Ap)
        dist.all_reduce(pAp_t, group=group)
        pAp = backend.item(pAp_t)
        if pAp <= 0:
            from .solve import SolverError
            raise SolverError("p^T A p <= 0: operator not SPD")
        alpha = rz / pAp
        rzn_t = backend.update(alpha, x, r, z, p_local, Ap, minv)
        dist.all_reduce(rzn_t, group=group)
        rzn = backend.item(rzn_t)
        it += 1
        if np.sqrt(abs(rzn)) <= tol * norm0:
            converged, rz = True, rzn
            break
        beta = rzn / rz
        rz = rzn
        backend.xpby(z, beta, p_local)
    return x, dict(iterations=it, residual=float(np.sqrt(abs(rz)) / norm0),
                   seconds=time.perf_counter() - t0, converged=converged)
