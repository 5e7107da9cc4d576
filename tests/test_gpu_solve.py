"""GPU: the row-block sharded Jacobi-PCG (distributed.pcg_sharded, fl_cg_*) against the
single-device solver fl_pcg (solve.pcg) and across rank counts.

* world 1 over a real NCCL process group: x and the iteration count bitwise equal to fl_pcg;
* 2 / 4 / 8 "ranks" emulated in lockstep on the one GPU (each rank's row block is its own
  fl_dense, the all-gathers are concatenations, every step in pcg_sharded's order — no kernel
  waits on another): bitwise the 1-rank iterates, and the split matvec of every row block
  equals the rows of the whole-matrix matvec bitwise.
Reference loop: solve.py:52-109; sharding: SURVEY.md §8(e)."""
import os
import socket

import numpy as np
import pytest

from conftest import make_mesh

pytestmark = pytest.mark.gpu


def _setup(kind, N, s):
    from paper_1708_03912_b200 import mesh as M, assembly as A
    mesh = make_mesh(kind, N)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    b = A.load_vector(mesh, dm, 1.0)
    return mesh, dm, ker, b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def lockstep_pcg(mesh, dm, ker, b, world, tol, max_iter, ops=None):
    """pcg_sharded's schedule for `world` ranks run one after another on one GPU."""
    import torch
    from paper_1708_03912_b200 import assembly as A, distributed as D
    n = dm.n
    rows = D.shard_rows(n, world)
    blk = D.block_rows(n, world)
    if ops is None:
        ops = [A.assemble_dense_device(mesh, dm, ker, rows=r) for r in rows]
    bes = [D.TorchDeviceBackend(op) for op in ops]
    st = []
    for g, ((r0, r1), be, op) in enumerate(zip(rows, bes, ops)):
        m = r1 - r0
        d = op.diag()
        loc, _ = be.setup(n, m, blk, world, g, tol, max_iter)
        v = dict(x=be.zeros(blk), r=be.from_numpy(b[r0:r1], blk), z=be.zeros(blk), p=be.zeros(blk),
                 Ap=be.zeros(blk), minv=be.from_numpy(1.0 / d, blk), loc=loc)
        st.append(v)
    allp = torch.zeros(world * bes[0].local.numel(), dtype=torch.float64, device="cuda")

    def gather():
        allp.copy_(torch.cat([v["loc"] for v in st]))

    for be, v in zip(bes, st):
        be.begin(v["r"], v["minv"], v["z"], v["p"])
    gather()
    for be in bes:
        be.init(allp)
    while True:
        for _ in range(D.CHUNK_ITERS):
            for be, v in zip(bes, st):
                if world > 1:
                    be.matvec_diag(v["p"])
            p_full = torch.cat([v["p"] for v in st]) if world > 1 else st[0]["p"]
            for be, v in zip(bes, st):
                be.matvec_rest(p_full, v["p"], v["Ap"])
            gather()
            for be, v in zip(bes, st):
                be.alpha_update(allp, v["x"], v["r"], v["z"], v["p"], v["Ap"], v["minv"])
            gather()
            for be, v in zip(bes, st):
                be.beta_xpby(allp, v["z"], v["p"])
        polls = [be.poll() for be in bes]
        assert all(p == polls[0] for p in polls)
        if polls[0]["done"]:
            break
    x = torch.cat([v["x"][:r1 - r0] for v, (r0, r1) in zip(st, rows)]).cpu().numpy()
    for be in bes:
        be.free()
    return x, polls[0], ops


@pytest.mark.parametrize("kind,N,s", [("graded1d", 2048, 0.75), ("uniform1d", 1500, 0.25), ("square2d", 40, 0.5),
                                      ("square2d", 48, 0.25)])
def test_lockstep_ranks_bitwise(cuda_lib, kind, N, s):
    """Row blocks are bitwise the whole matrix's rows (1D: canonical gather order; 2D: exact
    fixed-point cross accumulation), so 1/2/4/8 ranks give bitwise the same x and iteration
    count, equal to fl_pcg's."""
    from paper_1708_03912_b200 import solve as S, assembly as A
    mesh, dm, ker, b = _setup(kind, N, s)
    full = A.assemble_dense_device(mesh, dm, ker)
    x_ref, rep = S.pcg(full, b, tol=1e-10, max_iter=10 ** 5)
    for world in (1, 2, 4, 8):
        if world * 512 > dm.n + 511:
            continue
        x, st, ops = lockstep_pcg(mesh, dm, ker, b, world, 1e-10, 10 ** 5, ops=[full] if world == 1 else None)
        assert st["converged"] and st["iterations"] == rep.iterations, (world, st, rep.iterations)
        assert np.array_equal(x, x_ref), (world, np.abs(x - x_ref).max())
        for op in ops:
            if op is not full:
                op.free()
    full.free()


@pytest.mark.parametrize("kind,N,s", [("graded1d", 2048, 0.75), ("square2d", 24, 0.5)])
def test_split_matvec_rows_bitwise(cuda_lib, kind, N, s):
    """The split matvec (diagonal-block chunks from the rank's slice, then the rest) of a row
    block equals the same rows of the whole-matrix matvec bitwise, for any row blocks."""
    import ctypes as C
    import torch
    from paper_1708_03912_b200 import assembly as A, distributed as D, _lib
    from paper_1708_03912_b200.operator import DenseDeviceOperator
    mesh, dm, ker, _ = _setup(kind, N, s)
    n = dm.n
    full = A.assemble_dense_device(mesh, dm, ker)
    Ah = full.to_host()
    lib = _lib.load()
    x = np.random.default_rng(0).uniform(-1, 1, n)
    for world in (2, 3):
        rows = D.shard_rows(n, world, align=512)
        blk = D.block_rows(n, world)
        if rows[-1][0] >= rows[-1][1]:
            continue
        pf = torch.zeros(world * blk, dtype=torch.float64, device="cuda")
        pf[:n] = torch.from_numpy(x).cuda()
        y_full = torch.zeros(blk * world, dtype=torch.float64, device="cuda")
        full.matvec_device(pf.data_ptr(), y_full.data_ptr(), torch.cuda.current_stream().cuda_stream)
        for g, (r0, r1) in enumerate(rows):
            # a row-block operator holding exactly the whole matrix's rows (uploaded)
            blkop = DenseDeviceOperator.from_host_rows(Ah[r0:r1], n, r0)
            be = D.TorchDeviceBackend(blkop)
            be.setup(n, r1 - r0, blk, world, g, 1e-10, 10)
            Ap = be.zeros(blk)
            pl = pf[g * blk:(g + 1) * blk].clone()
            be.matvec_diag(pl)
            be.matvec_rest(pf, pl, Ap)
            assert torch.equal(Ap[:r1 - r0], y_full[r0:r1]), (world, g)
            be.free()
            blkop.free()
    full.free()
    del C, lib


def _nccl_worker(rank, world, port, kind, N, s, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from paper_1708_03912_b200 import assembly as A, distributed as D
    mesh, dm, ker, b = _setup(kind, N, s)
    rows = D.shard_rows(dm.n, world)
    r0, r1 = rows[rank]
    op = A.assemble_dense_device(mesh, dm, ker, rows=(r0, r1))
    x, rep = D.pcg_sharded(D.TorchDeviceBackend(op), b[r0:r1], op.diag(), rows, dm.n, dist, tol=1e-10,
                           max_iter=10 ** 5)
    np.save(out, np.concatenate([[rep["iterations"], float(rep["converged"])], x.cpu().numpy()]))
    op.free()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,N,s", [("graded1d", 2048, 0.75), ("square2d", 24, 0.5)])
def test_pcg_sharded_nccl_world1_equals_fl_pcg(cuda_lib, tmp_path, kind, N, s):
    """pcg_sharded on TorchDeviceBackend over a real NCCL group (world 1) reproduces fl_pcg's
    iterates bitwise (same kernels, same fold) and the same iteration count."""
    import torch.multiprocessing as mp
    from paper_1708_03912_b200 import solve as S, assembly as A
    mesh, dm, ker, b = _setup(kind, N, s)
    with A.assemble_dense_device(mesh, dm, ker) as op:
        x_ref, rep = S.pcg(op, b, tol=1e-10, max_iter=10 ** 5)
    out = str(tmp_path / "x.npy")
    mp.spawn(_nccl_worker, args=(1, _free_port(), kind, N, s, out), nprocs=1, join=True)
    res = np.load(out)
    assert int(res[0]) == rep.iterations and res[1] == 1.0
    assert np.array_equal(res[2:], x_ref)


def test_pcg_x0_and_breakdown(cuda_lib):
    """x0 warm start (solve.py:73-74) through the sharded path on one rank; SolverError on a
    non-SPD operator (solve.py:87-88)."""
    from paper_1708_03912_b200 import solve as S, assembly as A, distributed as D
    from paper_1708_03912_b200.solve import _OneRank, SolverError
    from paper_1708_03912_b200.operator import DenseDeviceOperator
    mesh, dm, ker, b = _setup("uniform1d", 300, 0.5)
    n = dm.n
    with A.assemble_dense_device(mesh, dm, ker) as op:
        x_ref, rep = S.pcg(op, b, tol=1e-12, max_iter=10 ** 5)
        x0 = x_ref + 1e-3 * np.random.default_rng(1).uniform(-1, 1, n)
        x, r = D.pcg_sharded(D.TorchDeviceBackend(op), b, op.diag(), [(0, n)], n, _OneRank, tol=1e-12,
                             max_iter=10 ** 5, x0_local=x0)
        xs, reps = S.pcg(op, b, tol=1e-12, max_iter=10 ** 5, x0=x0)
        assert r["iterations"] == reps.iterations
        assert np.array_equal(x.cpu().numpy(), xs)
        assert np.linalg.norm(xs - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
    Abad = np.diag(np.r_[np.ones(600), -np.ones(624)])
    with DenseDeviceOperator.from_host(Abad) as bad:
        with pytest.raises(SolverError):
            D.pcg_sharded(D.TorchDeviceBackend(bad), np.ones(1224), np.abs(np.diag(Abad)), [(0, 1224)], 1224,
                          _OneRank, tol=1e-10, max_iter=100)


@pytest.mark.parametrize("name,N,s,tol", [("c4a", 128, 0.25, 1e-10), ("c4b", 128, 0.75, 1e-10), ("c5", 256, 0.5, 1e-8)])
def test_cg_large_against_tight_solve(cuda_lib, name, N, s, tol):
    """BASELINE configs[3]/[4]: Jacobi-PCG on the whole device matrix to the BASELINE tolerance
    (c5: rel. residual 1e-8) lands within 1e-9 (relative l2) of a tol-1e-12 solve of the same
    matrix, the sharded solver on one rank gives the same iterates bitwise, and the true residual
    ||b - A x|| / ||b|| is small.  Iteration counts are printed for the record."""
    from paper_1708_03912_b200 import solve as S, assembly as A, distributed as D
    from paper_1708_03912_b200.solve import _OneRank
    mesh, dm, ker, b = _setup("square2d", N, s)
    n = dm.n
    with A.assemble_dense_device(mesh, dm, ker) as op:
        x, rep = S.pcg(op, b, tol=tol, max_iter=10 ** 5)
        xt, rept = S.pcg(op, b, tol=1e-12, max_iter=10 ** 5)
        xs, reps = D.pcg_sharded(D.TorchDeviceBackend(op), b, op.diag(), [(0, n)], n, _OneRank, tol=tol,
                                 max_iter=10 ** 5)
        res = np.linalg.norm(b - op.matvec(x)) / np.linalg.norm(b)
    rel = np.linalg.norm(x - xt) / np.linalg.norm(xt)
    print("%s: n=%d iterations %d (tol %g), %d (tol 1e-12), |x - x_tight| / |x_tight| = %.2e, true residual %.2e"
          % (name, n, rep.iterations, tol, rept.iterations, rel, res))
    assert rep.converged and rept.converged
    assert reps["iterations"] == rep.iterations and np.array_equal(xs.cpu().numpy(), x)
    assert rel <= 1e-9
    assert res <= 10 * tol
