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
    def __init__(self, A_rows):
        self.A = torch.as_tensor(A_rows)

    def zeros(self, m):
        return torch.zeros(m, dtype=torch.float64)

    def from_numpy(self, a):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).clone()

    def matvec(self, p_full, out):
        out.copy_(self.A @ p_full[: self.A.shape[1]])

    def dot(self, a, b):
        return torch.dot(a, b).reshape(1)

    def update(self, alpha, x, r, z, p, Ap, minv):
        x.add_(alpha * p)
        r.sub_(alpha * Ap)
        z.copy_(minv * r)
        return torch.dot(r, z).reshape(1)

    def xpby(self, z, beta, p):
        p.mul_(beta).add_(z)

    def item(self, t):
        return float(t.item())


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
    be = HostBackend(A[r0:r1])
    x, rep = D.pcg_sharded(be, b[r0:r1], np.diag(A)[r0:r1], rows, n, dist, tol=1e-10, max_iter=10 ** 5)
    parts = [None] * world
    dist.all_gather_object(parts, (r0, x.numpy(), rep["iterations"]))
    if rank == 0:
        xs = np.zeros(n)
        for a, xv, _ in parts:
            xs[a:a + len(xv)] = xv
        np.save(out, np.concatenate([[rep["iterations"]], xs]))
    dist.destroy_process_group()


def test_sharded_pcg_gloo_world2(tmp_path):
    from oracle import fraclap_oracle as O
    path = os.path.join(GOLDEN, "c1.npz")
    if not os.path.exists(path):
        pytest.skip("c1 golden missing")
    out = str(tmp_path / "x.npy")
    mp.spawn(_worker, args=(2, _free_port(), path, out), nprocs=2, join=True)
    res = np.load(out)
    it, x = int(res[0]), res[1:]
    G = np.load(path)
    xo, ito, _, _ = O.pcg(G["A"], G["b"], tol=1e-10, max_iter=10 ** 5)
    assert it == ito == int(G["iters"])
    assert np.linalg.norm(x - xo) <= 1e-12 * np.linalg.norm(xo)
    assert np.linalg.norm(x - G["x"]) <= 1e-9 * np.linalg.norm(G["x"])


def test_shard_rows():
    from paper_1708_03912_b200.distributed import shard_rows
    assert shard_rows(10, 3) == [(0, 3), (3, 7), (7, 10)]
    r = shard_rows(100, 4, weights=np.r_[np.ones(50), 3 * np.ones(50)])
    assert r[0][0] == 0 and r[-1][1] == 100 and all(a[1] == b[0] for a, b in zip(r, r[1:]))
    assert r[0][1] == 50 and r[1][1] == 67
