#!/usr/bin/env python
"""Benchmark of the dense fractional-Laplacian hot path on B200.

Metric (BASELINE.json): element-pair quadratures/s of the dense assembly, with the dense
matvec GB/s (and the CG solve) reported beside it, against the FP64 / HBM rooflines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step = one full dense assembly (assembly.py:1059-1104) of the configuration: every
element pair K x K~ (identical, touching, disjoint cross, ordered tail, boundary) on the
device, timed with CUDA events on the launching stream.  N > 1: rows are sharded by
contiguous DoF blocks (owner computes, no collective in the assembly); value = total pairs /
max-over-ranks time (strong scaling: the mesh is fixed).  After the timed steps: 100
matvecs with x ~ U(-1,1) (seed 0) and one Jacobi-PCG to 1e-10 (sharded CG with NCCL when
N > 1).  `--impl reference` times the CPU oracle port of the reference (oracle/) on a bounded
sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "element-pair quadratures/s (assembly) and dense matvec GB/s vs fp64/HBM roofline"
CONFIG_TEXT = {
    "c1": "1D uniform 512 cells, s=0.25 (n=513)",
    "c2": "1D graded 8192 cells toward +-1, s=0.75 (n=8191)",
    "c3": "2D unit square 64x64 SW-NE, s=0.5 (n=3969)",
    "c4a": "2D unit square 128x128 SW-NE, s=0.25 (n=16641)",
    "c4b": "2D unit square 128x128 SW-NE, s=0.75 (n=16129)",
    "c5": "2D unit square 256x256 SW-NE, s=0.5 (n=65025)",
}
# per-evaluation algorithmic fp64 FLOPs excluding the power and the
# executed FLOPs of the specialised power r2^ex (ncu-measured)
ALG_FLOPS = {(1, "tail"): 4, (1, "cross"): 6, (2, "tail"): 7, (2, "cross"): 11}
POW_FLOPS = {6: 11, 8: 8, 10: 11, 12: 9, 14: 12, 0: 60}   # = kpow_flops() in csrc/fl_device.cuh (2D)
POW_FLOPS_1D = {6: 9, 8: 9, 10: 10, 0: 60}                  # = kpow_abs_flops() (1D far field)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def committed_traffic(cfg, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/r01/traffic.json,
    dram__bytes_read.sum + dram__bytes_write.sum), or None when that kernel was not captured."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "traffic.json")) as f:
            return json.load(f).get(cfg, {}).get(kernel)
    except (OSError, ValueError):
        return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_worker(job):
    """One host process of the CPU baseline: the oracle port on its share of target cells."""
    cfg, budget_s, w, nw = job
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    from paper_1708_03912_b200 import mesh as M
    from oracle import fraclap_oracle as O
    mesh, s = M.baseline_mesh(cfg)
    dm = M.DofMap(mesh, s)
    o = O.Oracle(mesh, dm, s)
    cells = np.random.default_rng(0).permutation(mesh.num_cells)[w::nw]
    A = np.zeros((1, dm.n))
    rowmap = np.full(dm.n, -1, np.int64)
    t0 = time.perf_counter()
    done = 0
    for K in cells:
        o.psi(int(K))                                   # ordered tail pairs of K
        o.add_cell(int(K), A, rowmap, symmetric=True)   # unordered cross pairs (K, K2 > K) + identical
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return o.stats["pairs"], time.perf_counter() - t0, done


def cpu_sample(cfg, budget_s=12.0, procs=None):
    """Oracle port on every host core (one process per core, BLAS pinned to one thread each):
    owner-computes rows of random target cells of the same mesh for ~budget_s seconds; returns
    the aggregate pairs/s and the description."""
    import multiprocessing as mp
    if procs is None:
        try:
            procs = len(os.sched_getaffinity(0))
        except AttributeError:
            procs = os.cpu_count() or 1
        procs = max(1, min(procs, 128))
    jobs = [(cfg, budget_s, w, procs) for w in range(procs)]
    if procs == 1:
        res = [_cpu_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_worker, jobs)
    pairs = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    return pairs / dt, dict(cells=sum(r[2] for r in res), seconds=dt, pairs=pairs, threads=procs)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, info = cpu_sample(args.config, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.median(vals))
    sample = ("oracle port (numpy restatement of assemble_dense), %d host processes, on %d random target "
              "cells of %s: their ordered tail pairs + unordered cross pairs, %.1f s per step"
              % (info["threads"], info["cells"], args.config, info["seconds"]))
    line = {"metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": 0, "steps": args.steps,
            "ms_per_step": 1e3 * info["seconds"],
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "impl": "reference",
            "dtype": "f64", "data": "synthetic", "vs_baseline": None,
            "config": {"workload": args.config, "mesh": CONFIG_TEXT[args.config]},
            "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": info["threads"], "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--matvecs", type=int, default=100)
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-near", action="store_true", help="skip the near-field (cluster path) timing")
    ap.add_argument("--ref-budget", type=float, default=8.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1708_03912_b200 import _lib, mesh as M, assembly as A, solve as S, distributed as D

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream

    mesh, s = M.baseline_mesh(args.config)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(mesh.d, s)
    n = dm.n
    rows = D.shard_rows(n, world)
    r0, r1 = rows[rank]

    def assemble():
        return A.assemble_dense_device(mesh, dm, ker, rows=(r0, r1), device=local, stream=sptr)

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")   # > L2 (126 MB)
    for _ in range(args.warmup):
        op = assemble()
        op.free()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = lib.fl_launch_count()
    times, stats = [], None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))                       # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            op = assemble()
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            times.append(ev[i][0].elapsed_time(ev[i][1]))
            stats = op.stats()
            if i < args.steps - 1:
                op.free()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = (lib.fl_launch_count() - launches0) // max(args.steps, 1)
    tot = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_step = float(tot.item()) / args.steps
    pairs = (stats["pairs_identical"] + stats["pairs_touching"] + stats["pairs_cross"] + stats["pairs_tail"]
             + stats["pairs_boundary_singular"] + stats["pairs_boundary_flux"])
    value = pairs / (ms_step / 1e3)

    # roofline of the dominant assembly kernel (fp64 pipe)
    fp64 = C_double = None
    import ctypes as C
    C_double = C.c_double()
    _lib.check(lib.fl_probe_fp64_peak(local, C.byref(C_double)))
    fp64 = C_double.value
    e4 = int(round(4 * (mesh.d + 2 * s))) if s in (0.25, 0.5, 0.75) else 0
    kern = {"tail": (stats["ms_tail"], stats["evals_tail"]), "cross": (stats["ms_cross"], stats["evals_cross"])}
    dom = max(kern, key=lambda k: kern[k][0])
    ms_k, ev_k = kern[dom]
    fl_per_eval = ALG_FLOPS[(mesh.d, dom)] + (POW_FLOPS_1D if mesh.d == 1 else POW_FLOPS).get(e4, 60)
    achieved = ev_k * fl_per_eval / (ms_k * 1e-3) / 1e12 if ms_k > 0 else 0.0
    kname = {("tail", 1): "tail1d_kernel", ("tail", 2): "tail_kernel", ("cross", 1): "cross1d_tile_kernel",
             ("cross", 2): "cross_tile_kernel"}[(dom, mesh.d)]
    roofline = {"bound": "fp64", "kernel": kname, "achieved": achieved, "peak": fp64,
                "unit": "TFLOP/s", "frac": achieved / fp64 if fp64 else None,
                "traffic": committed_traffic(args.config, kname),
                "peak_source": "fl_probe_fp64_peak (DFMA chains, this run)",
                "flops_per_eval": fl_per_eval, "evals_per_launch": ev_k, "ms_per_launch": ms_k}

    # dense matvec GB/s (100 matvecs, x ~ U(-1,1) seed 0), A (> L2) read once per matvec
    pk, pk_src = peaks()
    lda = ((n + 31) // 32) * 32
    x = torch.zeros(lda, dtype=torch.float64, device="cuda")
    x[:n] = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(max(r1 - r0, 1), dtype=torch.float64, device="cuda")
    mv = []
    for i in range(args.matvecs + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.matvec_device(x.data_ptr(), y.data_ptr(), sptr)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            mv.append(e0.elapsed_time(e1))
    mv_ms = float(np.median(mv))
    mv_bytes = 8.0 * (r1 - r0) * n + 8.0 * n + 8.0 * (r1 - r0)
    mvt = torch.tensor([mv_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(mvt, op=dist.ReduceOp.MAX)
    mv_gbs = (8.0 * n * n + 16.0 * n) / (float(mvt.item()) * 1e-3) / 1e9
    matvec = {"gbs": mv_gbs, "ms": float(mvt.item()), "bytes": 8.0 * n * n + 16.0 * n,
              "traffic": committed_traffic(args.config, "matvec_kernel"),
              "frac_of_measured_copy_peak": mv_gbs / (pk["hbm_gbs"] * world), "peak_source": pk_src}

    # CG (Jacobi PCG to 1e-10, solve.py:52-109)
    cg = None
    if not args.no_cg:
        b = A.load_vector(mesh, dm, lambda X: np.ones(len(X)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            xs, rep = S.pcg(op, b, tol=1e-10, max_iter=10 ** 5)
            cg = {"iterations": rep.iterations, "seconds": rep.seconds, "converged": rep.converged,
                  "true_residual": rep.true_residual}
        else:
            be = D.TorchDeviceBackend(op, sptr)
            xs, rep = D.pcg_sharded(be, b[r0:r1], op.diag(), rows, n, dist, tol=1e-10, max_iter=10 ** 5)
            cg = {"iterations": rep["iterations"], "seconds": time.perf_counter() - t0,
                  "converged": rep["converged"]}
        cg["ms_per_iteration"] = 1e3 * cg["seconds"] / max(cg["iterations"], 1)

    # e2e through the public API with host buffers: assemble_dense -> (n, n) ndarray (N = 1), or
    # each rank's row block assemble_dense_device(rows) -> to_host (N > 1); max over ranks
    e2e = None
    if 8.0 * (r1 - r0) * n <= 4e9:     # host copy of the rows must fit comfortably in pinned RAM
        Mh = A._lib.Marshal(mesh, dm, ker, None)
        tdir, tdata, _ = A._tables(mesh, dm, s, None)
        h2d = (Mh.vertices.nbytes + Mh.cells.nbytes + Mh.bedges.nbytes + Mh.bnormals.nbytes + Mh.v2d.nbytes
               + tdir.nbytes + tdata.nbytes)
        out = torch.empty((r1 - r0, n), dtype=torch.float64, pin_memory=True).numpy()
        et = []
        for i in range(max(2, args.steps)):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:
                A.assemble_dense(mesh, dm, ker, n_limit=10 ** 7, out=out)
            else:
                ope = A.assemble_dense_device(mesh, dm, ker, rows=(r0, r1), device=local, stream=sptr)
                ope.to_host(out)
                ope.free()
            tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et.append(float(tt.item()))
        e2e = {"value": pairs / float(np.median(et)), "unit": "pairs/s", "h2d_bytes_per_step": int(h2d * world),
               "d2h_bytes_per_step": int(8 * n * n), "seconds_per_step": float(np.median(et))}

    # near-field (cluster path) assembly of the same mesh, SPEC defaults (leaf cap 8 / 16, eta 1):
    # assemble_near_field through the public API (host tree + partition excluded, CSR returned to
    # the host included), median of 3 after one warm-up
    near = None
    if rank == 0 and world == 1 and not args.no_near:
        from paper_1708_03912_b200 import cluster as CL
        th = time.perf_counter()
        tree = CL.build_tree(mesh, dm, 8 if mesh.d == 1 else 16)
        far_nodes, near_nodes = CL.admissible_partition(tree, 1.0)
        ns = CL.NearStructure(mesh, dm, tree, near_nodes)
        host_s = time.perf_counter() - th
        nts = []
        for i in range(4):
            t0 = time.perf_counter()
            An = A.assemble_near_field(mesh, dm, ker, ns)
            nts.append(time.perf_counter() - t0)
        near = {"ms": 1e3 * float(np.median(nts[1:])), "nnz": int(An.nnz), "leaf_cap": 8 if mesh.d == 1 else 16,
                "eta": 1.0, "near_leaf_pairs": int(len(ns.nl_pairs)), "far_node_pairs": int(len(far_nodes)),
                "host_tree_partition_s": host_s}
        # the whole cluster path (compress -> H-matrix matvec -> residual strong form), m = choose_order
        try:
            from paper_1708_03912_b200 import adapt as AD

            class _St:
                pass
            st_ = _St()
            st_.h_min, st_.dim = float(mesh.cell_diameters().min()), mesh.d
            mo = CL.choose_order(st_)
            t0 = time.perf_counter()
            cop = CL.compress(mesh, dm, ker, tree, 1.0, mo)
            comp_s = time.perf_counter() - t0
            xv = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
            yv = torch.empty_like(xv)
            cev = []
            for i in range(23):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _lib.check(lib.fl_cluster_matvec(cop.handle, C.c_void_p(xv.data_ptr()), C.c_void_p(yv.data_ptr()),
                                                 None, 1))
                e1.record(stream)
                torch.cuda.synchronize()
                if i >= 3:
                    cev.append(e0.elapsed_time(e1))
            X4, _ = AD.cell_nodes(mesh, 4)
            AD.strong_form_at(xv.cpu().numpy(), mesh, dm, cop, X=X4)
            t0 = time.perf_counter()
            AD.strong_form_at(xv.cpu().numpy(), mesh, dm, cop, X=X4)
            sf_ms = 1e3 * (time.perf_counter() - t0)
            bc = A.load_vector(mesh, dm, 1.0)
            t0 = time.perf_counter()
            _, crep = S.pcg(cop, bc, tol=1e-10, max_iter=10 ** 5)
            cg_s = time.perf_counter() - t0
            near["cluster"] = {"cheb_order": mo, "far_pairs": int(len(cop.far_pairs)), "compress_s": comp_s,
                               "matvec_us": 1e3 * float(np.median(cev)), "strong_form_ms": sf_ms,
                               "cg_iterations": crep.iterations, "cg_ms_per_iteration": 1e3 * cg_s / max(crep.iterations, 1)}
            cop.free()
        except Exception as exc:     # reported, never fatal for the headline line
            near["cluster"] = {"error": repr(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, info = cpu_sample(args.config)
        cpu = {"value": v, "unit": "pairs/s", "cores": info["threads"], "kind": "port",
               "sample": "oracle port, %d host processes, on %d random target cells of %s (their ordered "
                         "tail + unordered cross pairs), %.1f s" % (info["threads"], info["cells"], args.config,
                                                                   info["seconds"])}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE mesh, f=1)",
                "config": {"workload": args.config, "mesh": CONFIG_TEXT[args.config], "n": n,
                           "cells": mesh.num_cells, "pairs_per_step": pairs,
                           "parallelism": "rows%d" % world, "l2": "flushed (256 MB write) between steps",
                           "phases_ms": {k: stats[k] for k in ("ms_prep", "ms_singular", "ms_tail", "ms_flux",
                                                               "ms_tiles", "ms_cross", "ms_discover", "ms_near",
                                                               "ms_cross_compute", "ms_local", "ms_total")},
                           "near_pairs": stats["near_pairs"], "evals_tail": stats["evals_tail"],
                           "evals_cross": stats["evals_cross"]},
                "roofline": roofline, "matvec": matvec, "cg": cg, "e2e": e2e, "near_field": near,
                "cpu_baseline": cpu,
                "clocks": clk.summary(), "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    op.free()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
