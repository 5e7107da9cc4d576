"""Row-block sharded CG (paper_1708_03912_b200.distributed) over torch.distributed with the
gloo backend, world_size 2, on CPU: the same control logic the NCCL/GPU path runs, with a
host backend standing in for the device kernels.  Checked against the single-process
Jacobi-PCG of the oracle on the reference's own c1 matrix (tests/golden/c1.npz)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN


class HostBackend:
    """The device steps of fl_cg_* (csrc/fl_solve.cu) restated on CPU tensors: chunk sums over
    fixed global chunks of 512 entries, gathered and folded in global order on every rank."""
    VCH = 512

    def __init__(self, A_rows, r0):
        self.A = torch.as_tensor(A_rows)
        self.r0 = r0

    def zeros(self, m):
        return torch.zeros(m, dtype=torch.float64)

    def from_numpy(self, a, length=None):
        a = np.asarray(a, dtype=np.float64)
        t = self.zeros(len(a) if length is None else length)
        t[:len(a)] = torch.from_numpy(a)
        return t

    def scalar(self, v):
        return torch.tensor([float(v)], dtype=torch.float64)

    def item(self, t):
        return float(t.item())

    def setup(self, n, m, blk, world, rank, tol, max_iter):
        self.n, self.m, self.blk, self.world, self.tol, self.max_iter = n, m, blk, world, tol, max_iter
        self.L = blk // self.VCH
        self.local = self.zeros(self.L)
        self.all = self.local if world == 1 else self.zeros(self.L * world)
        self.sc = dict(it=0, done=False, converged=False, error=0, rz=0.0, norm0=0.0, alpha=0.0, beta=0.0)
        return self.local, self.all

    def _parts(self, v):
        self.local.zero_()
        for c in range(-(-self.m // self.VCH)):
            self.local[c] = float(v[c * self.VCH:min(self.m, (c + 1) * self.VCH)].sum())

    def _fold(self, allp):
        t = 0.0
        for g in range(self.world):
            rows = max(0, min(self.n, (g + 1) * self.blk) - g * self.blk)
            for c in range(-(-rows // self.VCH)):
                t += float(allp[g * self.L + c])
        return t

    def begin(self, r, minv, z, p):
        m = self.m
        z[:m] = minv[:m] * r[:m]
        p[:m] = z[:m]
        self._parts(r[:m] * z[:m])

    def init(self, allp):
        rz = self._fold(allp)
        self.sc.update(rz=rz, norm0=float(np.sqrt(abs(rz))))
        if self.sc["norm0"] == 0:
            self.sc.update(done=True, converged=True)

    def matvec_diag(self, p_local):
        pass

    def matvec_rest(self, p_full, p_local, Ap):
        if self.sc["done"]:
            return
        Ap[:self.m] = self.A @ p_full[:self.A.shape[1]]
        self._parts(p_local[:self.m] * Ap[:self.m])

    def alpha_update(self, allp, x, r, z, p, Ap, minv):
        if self.sc["done"]:
            return
        pAp = self._fold(allp)
        if not pAp > 0:
            self.sc.update(error=1, done=True)
            return
        a = self.sc["rz"] / pAp
        m = self.m
        x[:m] += a * p[:m]
        r[:m] -= a * Ap[:m]
        z[:m] = minv[:m] * r[:m]
        self._parts(r[:m] * z[:m])

    def beta_xpby(self, allp, z, p):
        if self.sc["done"]:
            return
        rzn = self._fold(allp)
        self.sc["it"] += 1
        if np.sqrt(abs(rzn)) <= self.tol * self.sc["norm0"]:
            self.sc.update(converged=True, done=True, rz=rzn)
            return
        beta = rzn / self.sc["rz"]
        self.sc["rz"] = rzn
        if self.sc["it"] >= self.max_iter:
            self.sc["done"] = True
        p[:self.m] = z[:self.m] + beta * p[:self.m]

    def poll(self):
        return dict(iterations=self.sc["it"], rz=self.sc["rz"], norm0=self.sc["norm0"], done=self.sc["done"],
                    converged=self.sc["converged"], error=self.sc["error"])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1708_03912_b200 import distributed as D
    G = np.load(path)
    A, b = G["A"], G["b"]
    n = len(b)
    rows = D.shard_rows(n, world)
    r0, r1 = rows[rank]
    be = HostBackend(A[r0:r1], r0)
    x, rep = D.pcg_sharded(be, b[r0:r1], np.diag(A)[r0:r1], rows, n, dist, tol=1e-10, max_iter=10 ** 5)
    parts = [None] * world
    dist.all_gather_object(parts, (r0, x.numpy(), rep["iterations"]))
    if rank == 0:
        xs = np.zeros(n)
        for a, xv, _ in parts:
            xs[a:a + len(xv)] = xv
        np.save(out, np.concatenate([[rep["iterations"]], xs]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pcg_gloo(tmp_path, world):
    """world 3 at n = 513 leaves the last rank without rows (blocks of 512 rows)."""
    from oracle import fraclap_oracle as O
    path = os.path.join(GOLDEN, "c1.npz")
    if not os.path.exists(path):
        pytest.skip("c1 golden missing")
    out = str(tmp_path / "x.npy")
    mp.spawn(_worker, args=(world, _free_port(), path, out), nprocs=world, join=True)
    res = np.load(out)
    it, x = int(res[0]), res[1:]
    G = np.load(path)
    xo, ito, _, _ = O.pcg(G["A"], G["b"], tol=1e-10, max_iter=10 ** 5)
    assert it == ito == int(G["iters"])
    assert np.linalg.norm(x - xo) <= 1e-12 * np.linalg.norm(xo)
    assert np.linalg.norm(x - G["x"]) <= 1e-9 * np.linalg.norm(G["x"])


def test_shard_rows():
    from paper_1708_03912_b200.distributed import shard_rows, block_rows
    assert shard_rows(10, 3, align=1) == [(0, 4), (4, 8), (8, 10)]
    assert shard_rows(65025, 8) == [(g * 8192, min(65025, (g + 1) * 8192)) for g in range(8)]
    assert block_rows(8191, 2) == 4096 and shard_rows(8191, 2) == [(0, 4096), (4096, 8191)]
    assert shard_rows(513, 1) == [(0, 513)]
    for n, w in [(1, 4), (513, 3), (16641, 8), (3969, 2)]:
        r = shard_rows(n, w)
        assert r[0][0] == 0 and r[-1][1] == n and all(a[1] == b[0] for a, b in zip(r, r[1:]))
        assert all(a % 512 == 0 for a, _ in r if a < n)
