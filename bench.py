#!/usr/bin/env python
"""Benchmark of the dense fractional-Laplacian hot path on B200.

Metric (BASELINE.json): element-pair quadratures/s of the dense assembly, with the dense
matvec GB/s and the Jacobi-PCG solve reported beside it, against the FP64 / HBM rooflines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload: BASELINE configs[4] = c5 (2D unit square 256x256, s = 1/2, n = 65025, A = 33.8 GB),
the largest configuration that fits one GPU (configs[1] = c2 and configs[3] = c4a / c4b with their
100-matvec bandwidth runs are timed too, as `extra`).
A step = one full dense assembly (assembly.py:1059-1104) of the configuration: every element
pair K x K~ (identical, touching, disjoint cross, ordered tail, boundary) on the device, inputs
resident, timed with CUDA events on the launching stream.  N > 1 (`--gpus N` re-launches itself
under torch.distributed.run when WORLD_SIZE is unset): rank g assembles the DoF row block
shard_rows(n, N)[g] (owner computes, no collective); value = the whole matrix's pairs / max-over-
ranks time (strong scaling: the mesh is fixed).  After the timed steps: 100 matvecs with
x ~ U(-1,1) (seed 0), Jacobi-PCG to 1e-8 (c5) through the sharded solver (NCCL all-gathers when
N > 1), and the end-to-end public-API path (host mesh in -> assemble -> load_vector -> pcg -> x
to host).  `--impl reference` times the CPU oracle port of the reference (oracle/) on a bounded
sample of the same workload on the host cores (the reference itself cannot assemble c4/c5: its
nc^2 pair arrays need > 100 GB); beside it, `reference_own` times the UNMODIFIED reference
(baseline/_ref, its own assemble_dense + pcg) on c1 and a 512-cell 2D square with every host core.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    "c5": "2D unit square 256x256 SW-NE, s=0.5 (n=65025, A = 33.8 GB fp64)",
}
CG_TOL = {"c1": 1e-10, "c2": 1e-10, "c3": 1e-10, "c4a": 1e-10, "c4b": 1e-10, "c5": 1e-8}   # BASELINE.json configs
# per-evaluation algorithmic fp64 FLOPs excluding the power and the
# executed FLOPs of the specialised power r2^ex (ncu-measured)
ALG_FLOPS = {(1, "tail"): 4, (1, "cross"): 6, (2, "tail"): 7, (2, "cross"): 11}
POW_FLOPS = {6: 11, 8: 8, 10: 11, 12: 9, 14: 12, 0: 60}   # = kpow_flops() in csrc/fl_device.cuh (2D)
POW_FLOPS_1D = {6: 9, 8: 9, 10: 10, 0: 60}                  # = kpow_abs_flops() (1D far field)
KERNEL_NAME = {("tail", 1): "tail1d_kernel", ("tail", 2): "tail2d_block_kernel + tail_kernel",
               ("cross", 1): "cross1d_tile_kernel", ("cross", 2): "cross2d_kernel + near_block_kernel",
               ("tail_block", 2): "tail2d_block_kernel", ("tail_pairs", 2): "tail_kernel",
               ("cross_far", 2): "cross2d_kernel", ("near", 2): "near_block_kernel"}


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
                                       "--format=csv,noheader,nounits", "-lms", "200"],
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
    """DRAM bytes per launch of `kernel` from the committed ncu captures (profiles/*/traffic.json,
    dram__bytes_read.sum + dram__bytes_write.sum; the newest round that has it), or None."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                v = json.load(f).get(cfg, {}).get(kernel)
            if v is not None:
                return {"bytes": v, "source": "profiles/%s/traffic.json" % rnd}
        except (OSError, ValueError):
            continue
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n):
    """`--gpus N` without a torch.distributed launcher: re-run this script as N NCCL ranks."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # stderr shows nranks / NVLS for the record
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- CPU arm
def _cpu_worker(job):
    """One host process of the CPU baseline: the oracle port (numpy restatement of the reference's
    assemble_dense, pinned to its outputs) on its share of target cells — for each cell K every
    contribution the reference computes for K: identical pair, ordered tail pairs (Psi_K), the
    boundary flux at K's nodes, the unordered disjoint cross pairs (K, K2 > K), the touching pairs
    (K, K2 > K) and the singular (K, edge) pairs, all scattered into a dense row buffer with
    np.add.at as the reference does (rows folded modulo 64 so the buffer is (64, n) instead of (n, n);
    the scatter work is the reference's)."""
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
    g = o.g
    cells = np.random.default_rng(0).permutation(mesh.num_cells)[w::nw]
    R = 64
    A = np.zeros((R, dm.n))
    rowmap = np.arange(dm.n, dtype=np.int64) % R
    bitems = {}
    if len(g.be):
        for e in range(len(g.be)):
            for c in np.unique(np.concatenate([g.patch(v) for v in g.be[e]])):
                bitems.setdefault(int(c), []).append(e)
    extra = 0
    t0 = time.perf_counter()
    done = 0
    for K in cells:
        K = int(K)
        o.add_cell(K, A, rowmap, symmetric=True)            # identical + tail + flux + cross (K2 > K)
        for K2 in g.neigh(K):                               # touching pairs (K, K2 > K), assembly.py:644-690
            if K2 <= K:
                continue
            vA, vB = list(g.cells[K]), list(g.cells[K2])
            com = sorted(set(vA) & set(vB))
            vK = com + [v for v in vA if v not in com]
            vK2 = com + [v for v in vB if v not in com]
            topo = "cv" if (g.d == 1 or len(com) == 1) else "ce"
            locs = vK + ([vK2[2]] if topo == "ce" else vK2[1:]) if g.d == 2 else [com[0], vK[1], vK2[1]]
            k = int(O.order_touch(min(g.h[K], g.h[K2]), g.n, s, g.d, o.p))
            T = O.touching_matrix(topo, g.V[vK], g.V[vK2], s, k)
            dofs = g.v2d[locs]
            ok = dofs >= 0
            np.add.at(A, (rowmap[dofs[ok]][:, None], dofs[ok][None, :]), o.C * T[np.ix_(ok, ok)])
            extra += 1
        for e in bitems.get(K, ()):                          # singular (cell, edge) pairs, :784-857
            ev = list(g.be[e])
            cv = list(g.cells[K])
            shared = sorted(set(ev) & set(cv))
            if g.d == 1 or len(shared) == 2:
                topo, order, pe = "eoc", (ev + [v for v in cv if v not in ev]) if g.d == 2 else \
                    [ev[0]] + [v for v in cv if v != ev[0]], ev if g.d == 2 else [ev[0]]
            else:
                sv = shared[0]
                topo, order, pe = "te", [sv] + [v for v in cv if v != sv], [sv] + [v for v in ev if v != sv]
            kb = int(O.order_touch(g.h[K], g.n, s, g.d, o.p, boundary=True))
            van = (0 if s < 0.5 else 2) if topo == "eoc" else 0
            B = O.boundary_matrix(topo, g.V[order], g.V[pe], -g.bn[e], s, kb, van)
            dofs = g.v2d[order]
            ok = dofs >= 0
            np.add.at(A, (rowmap[dofs[ok]][:, None], dofs[ok][None, :]), o.C / (2 * s) * B[np.ix_(ok, ok)])
            extra += 1
        extra += 1 + len(g.be)                               # identical pair + nb boundary-flux pairs
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return o.stats["pairs"] + extra, time.perf_counter() - t0, done


def cpu_sample(cfg, budget_s=10.0, procs=None):
    """Oracle port on every host core (one process per core, BLAS pinned to one thread each):
    rows of random target cells of the same mesh for ~budget_s seconds; aggregate pairs/s."""
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


def cpu_sample_text(info, cfg):
    return ("oracle port (numpy restatement of assemble_dense, pinned to the reference's outputs), %d host "
            "processes, %d random target cells of %s: per cell its identical, ordered tail, boundary-flux, "
            "unordered cross (K2 > K), touching and boundary-singular pairs with the dense np.add.at scatter; "
            "%.1f s" % (info["threads"], info["cells"], cfg, info["seconds"]))


REF_DIR = os.path.join(ROOT, "baseline", "_ref")      # pip install --target of the unmodified reference
REF_OWN_CASES = {"c1": ("c1", None), "sq16": ("2D unit square 16x16 SW-NE, s=0.5 (512 cells, n=225)", 16)}


def _ref_own_child(cases):
    """Runs in a fresh interpreter (bench.py --ref-own): the UNMODIFIED reference's own
    assemble_dense (assembly.py:1059-1104) + Jacobi-PCG (solve.py:52-109), imported from
    baseline/_ref, on every host core its BLAS uses; the oracle port on the same job beside it
    (single process) so the port's speed relative to the reference is on record."""
    sys.path.insert(0, REF_DIR)
    import fraclap
    from fraclap import mesh as RM, assembly as RA, solve as RS
    from paper_1708_03912_b200 import mesh as M
    from oracle import fraclap_oracle as O
    out = {"module": os.path.dirname(fraclap.__file__).replace(ROOT + "/", ""), "cpu_count": os.cpu_count()}
    try:
        import threadpoolctl
        out["threadpool_info"] = [{k: i.get(k) for k in ("internal_api", "num_threads", "version")}
                                  for i in threadpoolctl.threadpool_info()]
    except Exception as e:                       # noqa: BLE001
        out["threadpool_info"] = "unavailable: %s" % e
    for name in cases:
        cfg, N = REF_OWN_CASES[name]
        if N is None:
            mesh, s = M.baseline_mesh(cfg)
        else:
            mesh, s = M.build_unit_square_mesh(N), 0.5
        rmesh = RM.Mesh(mesh.vertices, mesh.cells, mesh.boundary_edges, mesh.boundary_normals)
        rdm = RM.DofMap(rmesh, s)
        t0 = time.perf_counter()
        Ar = RA.assemble_dense(rmesh, rdm, RA.FractionalKernel(rmesh.d, s), n_limit=10 ** 6)
        t_asm = time.perf_counter() - t0
        b = RA.load_vector(rmesh, rdm, lambda X: np.ones(len(X)))
        t0 = time.perf_counter()
        x, rep = RS.pcg(Ar, b, precond="jacobi", tol=1e-10, max_iter=10 ** 5)
        t_cg = time.perf_counter() - t0
        dm = M.DofMap(mesh, s)
        o = O.Oracle(mesh, dm, s)
        t0 = time.perf_counter()
        Ao = o.assemble()
        t_port = time.perf_counter() - t0
        pairs = port_pair_total(o, mesh)
        out[name] = {"mesh": CONFIG_TEXT.get(cfg, cfg), "n": int(rdm.n), "pairs": int(pairs),
                     "assemble_s": t_asm, "pairs_per_s": pairs / t_asm, "cg_s": t_cg,
                     "cg_iterations": int(getattr(rep, "iterations", -1)),
                     "port_assemble_s_1proc": t_port, "port_max_rel_dev": float(np.abs(Ao - Ar).max() / np.abs(Ar).max())}
    print(json.dumps(out), flush=True)
    return 0


def port_pair_total(o, mesh):
    """Element pairs of one full oracle assembly, counted as the GPU arm counts them (pair_count)."""
    g = o.g
    nc, nb = mesh.num_cells, len(g.be)
    touching = len(o.touching_pairs())
    bsing = len(o.boundary_items())
    return nc + touching + (nc * (nc - 1) // 2 - touching) + (nc * (nc - 1) - 2 * touching) + bsing + nc * nb


def reference_own(cases=("c1", "sq16"), timeout=600):
    """The reference's own CPU path, timed in a child interpreter; None when baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "fraclap")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref /root/reference)"}
    try:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-own", ",".join(cases)],
                           capture_output=True, text=True, timeout=timeout)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:                       # noqa: BLE001
        return {"unavailable": "reference run failed: %s" % str(e)[:200]}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, info = cpu_sample(args.config, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.median(vals))
    own = None if args.no_ref_own else reference_own()
    line = {"metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": 0, "steps": args.steps,
            "ms_per_step": 1e3 * info["seconds"],
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "impl": "reference",
            "dtype": "f64", "data": "synthetic (BASELINE mesh, f=1)", "vs_baseline": None,
            "config": {"workload": args.config, "mesh": CONFIG_TEXT[args.config]},
            "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": info["threads"], "kind": "port",
                             "sample": cpu_sample_text(info, args.config), "reference_own": own},
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def roofline_of(stats, d, s, fp64, kind):
    """Algorithmic FP64 rate of one assembly kernel: its evaluations (device-counted) x FLOPs per
    evaluation / its device ms (CUDA events on the assembly stream).  kind: tail / cross (1D or
    the whole 2D phase), tail_block (2D block-pair tail kernel), tail_pairs (2D warp-per-target
    tail on the remaining source blocks), cross_far (2D cross2d_kernel compute pass), near (2D
    near blocks, k >= 5)."""
    e4 = int(round(4 * (d + 2 * s))) if s in (0.25, 0.5, 0.75) else 0
    base = "tail" if kind.startswith("tail") else "cross"
    if kind == "tail":
        ms, ev = stats["ms_tail"], stats["evals_tail"]
    elif kind == "tail_block":
        ms, ev = stats["ms_tail_block"], stats["evals_tail_block"]
    elif kind == "tail_pairs":
        ms, ev = stats["ms_tail"] - stats["ms_tail_block"], stats["evals_tail"] - stats["evals_tail_block"]
    elif kind == "cross":
        ms, ev = (stats["ms_cross_compute"] or stats["ms_cross"]), stats["evals_cross"]
    elif kind == "cross_far":
        ms, ev = stats["ms_cross_compute"], stats["evals_cross"] - stats["evals_near"]
    else:   # near
        ms, ev = stats["ms_near"], stats["evals_near"]
    fpe = ALG_FLOPS[(d, base)] + (POW_FLOPS_1D if d == 1 else POW_FLOPS).get(e4, 60)
    flops = ev * fpe
    extra = {}
    if kind in ("tail_block", "tail") and stats.get("evals_tail_sym", 0) > 0:
        # an order-4 block pair swept once for both directions: each of those evaluations also
        # accumulates into the partner cell's psi (one more FMA); it stands for two of the reference's
        sym = stats["evals_tail_sym"]
        flops += 2 * sym
        extra = {"evals_sym_both_directions": sym, "reference_equivalent_evals": ev + sym}
    ach = flops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    out = {"bound": "fp64", "kernel": KERNEL_NAME[(kind, d)], "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
           "frac": ach / fp64 if fp64 else None, "flops_per_eval": fpe, "evals_per_launch": ev,
           "ms_per_launch": ms}
    out.update(extra)
    return out


def pair_count(stats):
    return (stats["pairs_identical"] + stats["pairs_touching"] + stats["pairs_cross"] + stats["pairs_tail"]
            + stats["pairs_boundary_singular"] + stats["pairs_boundary_flux"])


def time_assembly(assemble, steps, warmup, stream, flush, world, dist):
    import torch
    for _ in range(warmup):
        op = assemble()
        op.free()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times, op = [], None
    for i in range(steps):
        if op is not None:
            op.free()
        flush.fill_(float(i))                       # L2 flush between timed steps (not timed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op = assemble()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return op, times


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--matvecs", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c2 line and the cluster-path timings")
    ap.add_argument("--ref-budget", type=float, default=6.0)
    ap.add_argument("--no-ref-own", action="store_true", help="skip timing the reference's own code (baseline/_ref)")
    ap.add_argument("--ref-own", default=None, help=argparse.SUPPRESS)    # internal: child of reference_own()
    args = ap.parse_args()
    if args.ref_own:
        return _ref_own_child(args.ref_own.split(","))
    if args.impl == "reference":
        return run_reference(args)
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)

    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_1708_03912_b200 import _lib, mesh as M, assembly as A, solve as S, distributed as D
    if torch.cuda.device_count() <= local:
        print(json.dumps({"error": "rank %d needs cuda:%d, %d visible" % (rank, local, torch.cuda.device_count())}))
        return 1
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

    def maxr(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def assemble():
        return A.assemble_dense_device(mesh, dm, ker, rows=(r0, r1), device=local, stream=sptr)

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")   # > L2 (126 MB)
    fp64c = C.c_double()
    _lib.check(lib.fl_probe_fp64_peak(local, C.byref(fp64c)))
    fp64 = fp64c.value

    # ---------------------------------------------------------------- timed assembly steps
    launches0 = lib.fl_launch_count()
    with ClockSampler(local) as clk:
        op, times = time_assembly(assemble, args.steps, args.warmup, stream, flush, world, dist)
    launches = (lib.fl_launch_count() - launches0) // max(args.steps + args.warmup, 1)
    stats = op.stats()
    ms_step = maxr(sum(times)) / args.steps
    # the whole matrix's element pairs (the classification is global, so every rank reports the
    # job's counts; a row block is a share of that job)
    pairs = pair_count(stats)
    value = pairs / (ms_step / 1e3)
    kinds = ("tail", "cross") if mesh.d == 1 or stats["ms_tail_block"] <= 0 else \
        ("tail_block", "tail_pairs", "cross_far", "near")
    roofs = [roofline_of(stats, mesh.d, s, fp64, k) for k in kinds]
    for r in roofs:
        r["traffic"] = committed_traffic(args.config, r["kernel"])
    roof = dict(max(roofs, key=lambda r: r["ms_per_launch"]))
    roof["traffic"] = committed_traffic(args.config, roof["kernel"])
    roof["peak_source"] = "fl_probe_fp64_peak (DFMA chains, this run, same GPU)"

    # ---------------------------------------------------------------- dense matvec GB/s
    pk, pk_src = peaks()
    blk = D.block_rows(n, world)
    xg = torch.zeros(world * blk, dtype=torch.float64, device="cuda")
    xg[:n] = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(max(r1 - r0, 1), dtype=torch.float64, device="cuda")
    mv = []
    for i in range(args.matvecs + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.matvec_device(xg.data_ptr(), y.data_ptr(), sptr)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            mv.append(e0.elapsed_time(e1))
    mv_ms = maxr(float(np.median(mv)))
    mv_bytes = 8.0 * n * n + 16.0 * n
    mv_gbs = mv_bytes / (mv_ms * 1e-3) / 1e9
    matvec = {"gbs": mv_gbs, "ms": mv_ms, "bytes": mv_bytes, "count": args.matvecs,
              "x": "U(-1,1) seed 0", "traffic": committed_traffic(args.config, "mv_rows_kernel")
              or committed_traffic(args.config, "matvec_kernel"),
              "frac_of_measured_copy_peak": mv_gbs / (pk["hbm_gbs"] * world), "peak_gbs": pk["hbm_gbs"] * world,
              "peak_source": pk_src}

    # ---------------------------------------------------------------- CG (solve.py:52-109)
    cg = None
    b = A.load_vector(mesh, dm, 1.0)
    tol = CG_TOL[args.config]
    if not args.no_cg:
        cg = {"tol": tol, "stopping": "sqrt(r.z) <= tol sqrt(r0.z0) (solve.py:96)"}
        be = D.TorchDeviceBackend(op)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        xs, rep = D.pcg_sharded(be, b[r0:r1], op.diag(), rows, n, dist if world > 1 else S._OneRank,
                                tol=tol, max_iter=10 ** 5)
        torch.cuda.synchronize()
        sec = maxr(time.perf_counter() - t0)
        cg.update({"path": "distributed.pcg_sharded (fl_cg_*, NCCL all-gathers)" if world > 1 else
                   "distributed.pcg_sharded (fl_cg_*, one rank)", "iterations": rep["iterations"],
                   "converged": rep["converged"], "seconds": sec,
                   "ms_per_iteration": 1e3 * sec / max(rep["iterations"], 1)})
        if world == 1:
            x1, rep1 = S.pcg(op, b, tol=tol, max_iter=10 ** 5)       # fl_pcg: CUDA-graph solver, same kernels
            cg["fl_pcg"] = {"iterations": rep1.iterations, "seconds": rep1.seconds,
                            "ms_per_iteration": 1e3 * rep1.seconds / max(rep1.iterations, 1),
                            "true_residual": rep1.true_residual}
            cg["sharded_equals_fl_pcg_bitwise"] = bool(np.array_equal(xs.cpu().numpy(), x1))
    op.free()

    # ---------------------------------------------------------------- end to end, public API
    e2e = None
    if not args.no_e2e:
        Mh = A._lib.Marshal(mesh, dm, ker, None)
        tdir, tdata, _ = A._tables(mesh, dm, s, None)
        h2d = (Mh.vertices.nbytes + Mh.cells.nbytes + Mh.bedges.nbytes + Mh.bnormals.nbytes + Mh.v2d.nbytes
               + tdir.nbytes + tdata.nbytes)
        et = []
        for i in range(max(1, args.e2e_steps)):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            ope = A.assemble_dense_device(mesh, dm, ker, rows=(r0, r1), device=local)
            bb = A.load_vector(mesh, dm, lambda X: np.ones(len(X)))          # f evaluated on the host
            if world == 1:
                xe, repe = S.pcg(ope, bb, tol=tol, max_iter=10 ** 5)
            else:
                xl, repe = D.pcg_sharded(D.TorchDeviceBackend(ope), bb[r0:r1], ope.diag(), rows, n, dist, tol=tol,
                                         max_iter=10 ** 5)
                xe = xl.cpu().numpy()
            torch.cuda.synchronize()
            et.append(maxr(time.perf_counter() - t0))
            ope.free()
        sec = float(np.median(et))
        q = 16 if mesh.d == 2 else 6
        e2e = {"value": pairs / sec, "unit": "pairs/s", "seconds_per_step": sec, "steps": len(et),
               "path": "host mesh -> assemble_dense_device -> load_vector -> pcg (tol %g) -> x on the host" % tol,
               # H2D: mesh + dofmap + quadrature tables (assembly), the same + f at the rule nodes
               # (load_vector), b and the diagonal (pcg); D2H: b (load_vector) and x
               "h2d_bytes_per_step": int(world * (2 * h2d + 8 * mesh.num_cells * q + 8 * n + 8 * (r1 - r0))),
               "d2h_bytes_per_step": int(world * 8 * n + 8 * n),
               "copies_declared": True}

    # ---------------------------------------------------------------- extra lines (rank 0, N = 1)
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra and args.config != "c2":
        extra["c2"] = extra_c2(lib, stream, flush, fp64)
        for c4 in ("c4a", "c4b"):
            extra[c4] = extra_c4(c4, lib, stream, flush, fp64)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, info = cpu_sample(args.config)
        cpu = {"value": v, "unit": "pairs/s", "cores": info["threads"], "kind": "port",
               "sample": cpu_sample_text(info, args.config),
               "reference_own": None if args.no_ref_own else reference_own()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE mesh, f=1)",
                "config": {"workload": args.config, "mesh": CONFIG_TEXT[args.config], "n": n,
                           "cells": mesh.num_cells, "pairs_per_step": pairs,
                           "parallelism": "rows%d" % world, "row_block": [r0, r1],
                           "l2": "flushed (256 MB write) between steps; A (%.1f GB) > L2" % (8e-9 * n * n),
                           "phases_ms_rank0": {k: stats[k] for k in ("ms_prep", "ms_singular", "ms_tail", "ms_flux",
                                                                     "ms_tiles", "ms_cross", "ms_discover", "ms_near",
                                                                     "ms_cross_compute", "ms_local", "ms_total")},
                           "near_pairs": stats["near_pairs"], "order_ties": stats["order_ties"],
                           "evals_tail": stats["evals_tail"],
                           "evals_cross": stats["evals_cross"]},
                "roofline": roof, "roofline_kernels": roofs, "matvec": matvec, "cg": cg, "e2e": e2e,
                "cpu_baseline": cpu, "extra": extra or None,
                "clocks": clk.summary(), "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def extra_c2(lib, stream, flush, fp64, steps=5):
    """configs[1] (c2, 1D graded, s = 3/4): device-timed assembly + its roofline, matvec, CG."""
    import torch
    from paper_1708_03912_b200 import mesh as M, assembly as A, solve as S
    mesh, s = M.baseline_mesh("c2")
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(1, s)
    sptr = stream.cuda_stream
    op, times = time_assembly(lambda: A.assemble_dense_device(mesh, dm, ker, stream=sptr), steps, 2, stream, flush,
                              1, None)
    st = op.stats()
    ms = float(np.mean(times))
    out = {"mesh": CONFIG_TEXT["c2"], "ms_per_step": ms, "value": pair_count(st) / (ms * 1e-3), "unit": "pairs/s",
           "roofline": roofline_of(st, 1, s, fp64, "tail"), "roofline_cross": roofline_of(st, 1, s, fp64, "cross")}
    x, rep = S.pcg(op, A.load_vector(mesh, dm, 1.0), tol=1e-10, max_iter=10 ** 5)
    out["cg"] = {"iterations": rep.iterations, "ms_per_iteration": 1e3 * rep.seconds / max(rep.iterations, 1)}
    op.free()
    return out


def extra_c4(name, lib, stream, flush, fp64, steps=3, matvecs=100):
    """configs[3] (c4a / c4b: 2D 128x128, s = 1/4 / 3/4): device-timed assembly with its kernel
    rooflines, 100 matvecs with x ~ U(-1,1) (seed 0) for the bandwidth, and Jacobi-PCG to 1e-10."""
    import torch
    from paper_1708_03912_b200 import mesh as M, assembly as A, solve as S
    mesh, s = M.baseline_mesh(name)
    dm = M.DofMap(mesh, s)
    ker = A.FractionalKernel(2, s)
    sptr = stream.cuda_stream
    op, times = time_assembly(lambda: A.assemble_dense_device(mesh, dm, ker, stream=sptr), steps, 2, stream, flush,
                              1, None)
    st = op.stats()
    ms = float(np.mean(times))
    kinds = ("tail_block", "tail_pairs", "cross_far", "near") if st["ms_tail_block"] > 0 else ("tail", "cross")
    out = {"mesh": CONFIG_TEXT[name], "ms_per_step": ms, "value": pair_count(st) / (ms * 1e-3), "unit": "pairs/s",
           "roofline_kernels": [roofline_of(st, 2, s, fp64, k) for k in kinds]}
    n = dm.n
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    mv = []
    for i in range(matvecs + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.matvec_device(x.data_ptr(), y.data_ptr(), sptr)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            mv.append(e0.elapsed_time(e1))
    mv_ms = float(np.median(mv))
    out["matvec"] = {"gbs": (8.0 * n * n + 16.0 * n) / (mv_ms * 1e-3) / 1e9, "ms": mv_ms, "count": matvecs,
                     "x": "U(-1,1) seed 0"}
    xs, rep = S.pcg(op, A.load_vector(mesh, dm, 1.0), tol=1e-10, max_iter=10 ** 5)
    out["cg"] = {"iterations": rep.iterations, "ms_per_iteration": 1e3 * rep.seconds / max(rep.iterations, 1)}
    op.free()
    return out


if __name__ == "__main__":
    sys.exit(main())
