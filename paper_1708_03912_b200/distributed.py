"""Row-block sharding over the GPUs of one box (torch.distributed / NCCL plumbing).

Assembly is owner-computes: rank g assembles the DoF rows R_g = [g*B, min(n, (g+1)*B)) of A on
its own GPU (fl_assemble_dense with a row range); nothing is exchanged.  The block size B is
the same for every rank and a multiple of 512 (the fixed reduction chunk of the solver), so the
search direction can be all-gathered straight into one padded vector and every reduction of
the solve is independent of the number of ranks.

`pcg_sharded` is Jacobi-PCG (solve.py:52-109) on the row blocks.  Per iteration:

    all-gather p  ||  diagonal-block chunks of A[R_g, :] p     (overlapped: NCCL stream vs compute stream)
    rest of the matvec + chunk sums of p.Ap      -> all-gather of the chunk sums
    alpha (folded on the device), x/r/z update + chunk sums of r.z  -> all-gather
    beta, stopping test (solve.py:96), p = z + beta p

The scalars never leave the device; the host reads a `done` flag every CHUNK_ITERS iterations
(all ranks fold the same gathered sums in the same order, so they stop together).  The control
logic is written against a small backend interface so the same code runs on CPU with gloo in
tests/test_distributed.py.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib

VCH = 512            # fixed global reduction chunk (csrc/fl_solve.cu); row blocks are multiples of it
CHUNK_ITERS = 8      # iterations enqueued between two reads of the device `done` flag


def block_rows(n: int, world: int, align: int = VCH) -> int:
    """Rows per rank: ceil(n / world) rounded up to a multiple of `align`."""
    if world <= 0:
        raise ValueError("world must be positive")
    per = -(-int(n) // world)
    return max(align, -(-per // align) * align)


def shard_rows(n: int, world: int, align: int = VCH):
    """Contiguous row blocks [(r0, r1)] for `world` ranks: equal blocks of block_rows(n, world)
    rows (the last one shorter).  Work per row is nearly uniform on the BASELINE meshes (the
    tail and cross terms of every row run over all cells), so the blocks are not weighted."""
    b = block_rows(n, world, align)
    return [(min(n, g * b), min(n, (g + 1) * b)) for g in range(world)]


class TorchDeviceBackend:
    """Device vectors as torch CUDA tensors; every step is one libfraclap_b200 call enqueued on
    torch's current stream (fl_cg_*, include/fraclap_b200.h)."""

    def __init__(self, op, stream=None):
        import torch
        self.torch = torch
        self.op = op
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._stream = stream
        self.lib = _lib.load()
        self.S = None

    @property
    def stream(self):
        s = self._stream if self._stream is not None else self.torch.cuda.current_stream().cuda_stream
        return C.c_void_p(int(s))

    # ---- vectors
    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64, device=self.dev)

    def from_numpy(self, a, length=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        t = self.zeros(len(a) if length is None else length)
        t[:len(a)] = self.torch.from_numpy(a).to(self.dev)
        return t

    def to_numpy(self, t):
        return t.cpu().numpy()

    def scalar(self, v):
        return self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)

    def item(self, t):
        return float(t.item())

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    # ---- solver state
    def setup(self, n, m, blk, world, rank, tol, max_iter):
        h = C.c_void_p()
        _lib.check(self.lib.fl_cg_create(n, m, blk, world, rank, float(tol), int(max_iter),
                                         self.dev.index, self.stream, C.byref(h)))
        self.S = h
        L = C.c_int64()
        _lib.check(self.lib.fl_cg_buffers(h, None, None, C.byref(L)))
        # the chunk sums live in torch tensors (the all-gather needs them); the library only
        # ever sees their pointers
        self.local = self.zeros(L.value)
        self.all = self.local if world == 1 else self.zeros(L.value * world)
        _lib.check(self.lib.fl_cg_bind_parts(h, self._p(self.local)))
        return self.local, self.all

    def free(self):
        if self.S is not None:
            self.lib.fl_cg_free(self.S)
            self.S = None

    def begin(self, r, minv, z, p):
        _lib.check(self.lib.fl_cg_begin(self.S, self._p(r), self._p(minv), self._p(z), self._p(p), self.stream))

    def init(self, allp):
        _lib.check(self.lib.fl_cg_init(self.S, self._p(allp), self.stream))

    def matvec_diag(self, p_local):
        _lib.check(self.lib.fl_cg_matvec_diag(self.S, self.op.handle, self._p(p_local), self.stream))

    def matvec_rest(self, p_full, p_local, Ap):
        _lib.check(self.lib.fl_cg_matvec_rest(self.S, self.op.handle, self._p(p_full), self._p(p_local),
                                              self._p(Ap), self.stream))

    def alpha_update(self, allp, x, r, z, p, Ap, minv):
        _lib.check(self.lib.fl_cg_alpha_update(self.S, self._p(allp), self._p(x), self._p(r), self._p(z),
                                               self._p(p), self._p(Ap), self._p(minv), self.stream))

    def beta_xpby(self, allp, z, p):
        _lib.check(self.lib.fl_cg_beta_xpby(self.S, self._p(allp), self._p(z), self._p(p), self.stream))

    def poll(self):
        st = _lib.fl_cg_status()
        _lib.check(self.lib.fl_cg_poll(self.S, C.byref(st), self.stream))
        return dict(iterations=int(st.iterations), rz=float(st.rz), norm0=float(st.norm0), done=bool(st.done),
                    converged=bool(st.converged), error=int(st.error))


def pcg_sharded(backend, b_local, diag_local, rows, n, dist, group=None, tol=1e-8, max_iter=None,
                precond="jacobi", x0_local=None):
    """Jacobi PCG with A distributed by the row blocks `rows` = shard_rows(n, world).  Same
    recurrences, stopping rule and iteration count as solve.py:52-109; the iterates are bitwise
    independent of the number of ranks.  Returns (x_local, report dict)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if [tuple(r) for r in rows] != shard_rows(n, world):
        raise ValueError("rows must be shard_rows(n, world): equal blocks of block_rows(n, world) rows")
    r0, r1 = rows[rank]
    m = r1 - r0
    blk = block_rows(n, world)
    if max_iter is None:
        max_iter = int(10 * np.sqrt(n) + 100)                    # solve.py:61-62
    be = backend
    t0 = time.perf_counter()
    d = np.asarray(diag_local, float)
    if precond == "jacobi":
        bad = be.scalar(float(np.any(d <= 0)))
        dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
        if be.item(bad) > 0:
            from .solve import SolverError
            raise SolverError("nonpositive diagonal; operator not SPD")      # solve.py:67-68
        minv = be.from_numpy(1.0 / np.where(d > 0, d, 1.0), blk)
    elif precond in (None, "none"):
        minv = be.from_numpy(np.ones(m), blk)
    else:
        raise ValueError("precond must be 'jacobi' or None")
    local, allp = be.setup(n, m, blk, world, rank, tol, max_iter)

    def gather(out, inp):
        if world > 1:
            dist.all_gather_into_tensor(out, inp, group=group)

    x = be.from_numpy(np.zeros(m) if x0_local is None else np.asarray(x0_local, float), blk)
    r = be.from_numpy(b_local, blk)
    z = be.zeros(blk)
    p_local = be.zeros(blk)
    Ap = be.zeros(blk)
    p_full = p_local if world == 1 else be.zeros(world * blk)
    try:
        if x0_local is not None:                                  # r = b - A x0 (solve.py:74)
            if world > 1:
                dist.all_gather_into_tensor(p_full, x, group=group)
            be.matvec_diag(x)
            be.matvec_rest(x if world == 1 else p_full, x, Ap)
            r.sub_(Ap)
        be.begin(r, minv, z, p_local)                              # z = M^-1 r, p = z (:75-77)
        gather(allp, local)
        be.init(allp)
        st = be.poll()
        while not st["done"]:
            for _ in range(CHUNK_ITERS):
                if world > 1:
                    # the all-gather runs on the NCCL stream while the diagonal block's chunks
                    # are computed from the rank's own slice of p
                    work = dist.all_gather_into_tensor(p_full, p_local, group=group, async_op=True)
                    be.matvec_diag(p_local)
                    work.wait()
                be.matvec_rest(p_full, p_local, Ap)
                gather(allp, local)
                be.alpha_update(allp, x, r, z, p_local, Ap, minv)
                gather(allp, local)
                be.beta_xpby(allp, z, p_local)
            st = be.poll()
        if st["error"]:
            from .solve import SolverError
            raise SolverError("p^T A p <= 0: operator not SPD")          # solve.py:87-88
    finally:
        if hasattr(be, "free"):
            be.free()
    norm0 = st["norm0"]
    return x[:m], dict(iterations=st["iterations"], residual=0.0 if norm0 == 0 else float(np.sqrt(abs(st["rz"])) / norm0),
                       seconds=time.perf_counter() - t0, converged=bool(st["converged"]) or norm0 == 0)
