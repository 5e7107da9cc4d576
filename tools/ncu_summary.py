#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py report <file.ncu-rep>      # per-kernel key metrics + top stalls
  python tools/ncu_summary.py launches <launches.csv>    # per-kernel share of the launch list
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe busy % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe busy % (elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA (thread inst)"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD (thread inst)"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL (thread inst)"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def report(path):
    hdr, units, rows = _raw(path)
    print("| kernel | metric | value |\n|---|---|---|")
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        short = name.split("(")[0].replace("void ", "")
        for k, label in KEYS:
            if k in d and d[k] != "":
                print("| %s | %s | %s %s |" % (short, label, d[k], u.get(k, "")))
        try:
            dfma = float(d["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"].replace(",", ""))
            dadd = float(d["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"].replace(",", ""))
            dmul = float(d["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"].replace(",", ""))
            t = float(d["gpu__time_duration.sum"].replace(",", ""))
            scale = {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}
            t *= scale.get(u.get("gpu__time_duration.sum", "ms"), 1e-3)
            print("| %s | executed fp64 TFLOP/s (2*DFMA+DADD+DMUL) | %.2f |" % (short, (2 * dfma + dadd + dmul) / t / 1e12))
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        st = []
        for k in hdr:
            if "smsp__average_warps_issue_stalled" in k and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        top = ", ".join("%s %.2f" % (n, v) for v, n in sorted(st, reverse=True)[:6])
        print("| %s | top stalls (warps per issue) | %s |" % (short, top))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("| %s | %d | %.1f | %.1f%% |" % (k, c, t, 100 * t / tot))


def flops(path):
    """Executed fp64 FLOPs from the per-instruction SASS counters (2*DFMA + DADD + DMUL, predicated-on
    thread instructions) and the kernel duration: the ncu-executed figure of SURVEY.md §8(d)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ip = hdr.index("Predicated-On Thread Instructions Executed")
    isrc = hdr.index("Source")
    cnt = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ip or not r[ip].isdigit():
            continue
        t = r[isrc].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        if op in ("DFMA", "DADD", "DMUL"):
            cnt[op] += int(r[ip])
    h, u, rr = _raw(path)
    d = dict(zip(h, rr[0]))
    t = float(d["gpu__time_duration.sum"].replace(",", ""))
    t *= {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}.get(
        dict(zip(h, u)).get("gpu__time_duration.sum", "ms"), 1e-3)
    fl = 2 * cnt["DFMA"] + cnt["DADD"] + cnt["DMUL"]
    name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
    print("| %s | executed fp64 FLOPs (2*DFMA+DADD+DMUL thread instructions) | %.4g |" % (name, fl))
    print("| %s | executed fp64 TFLOP/s (serialised ncu replay) | %.2f |" % (name, fl / t / 1e12))


if __name__ == "__main__":
    {"report": report, "launches": launches, "flops": flops}[sys.argv[1]](sys.argv[2])
