"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py gpurun_out/prof_dense_v1.ncu-rep dense_fpi_kernel profiles/r1_dense_ncu.md [tau]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r1_launches.md

Also merges per-kernel DRAM bytes per launch into profiles/ncu_summary.json,
which bench.py reads for the roofline ``traffic`` field.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
]
STALLS = ["wait", "math_pipe_throttle", "long_scoreboard", "short_scoreboard", "barrier", "selected",
          "not_selected", "branch_resolving", "mio_throttle", "lg_throttle", "dispatch_stall",
          "no_instruction"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return res


def summarise(rep, kernel, md_path, tau=None):
    rows = [r for r in raw(rep) if kernel in r.get("Kernel Name", ("", ""))[0]]
    if not rows:
        raise SystemExit(f"kernel {kernel} not in {rep}")
    r = rows[0]
    lines = [f"# ncu --set full: `{kernel}`", "", f"source: `{os.path.basename(rep)}` "
             "(ncu --set full --clock-control none --import-source on, one launch)", "",
             "| metric | value | unit |", "|---|---|---|"]
    vals = {}
    for m in METRICS:
        if m in r:
            v, u = r[m]
            vals[m] = (v, u)
            lines.append(f"| {m} | {v} | {u} |")
    lines += ["", "Warp stall reasons (average warps per issued instruction):", "",
              "| stall | per issue |", "|---|---|"]
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in r:
            lines.append(f"| {s} | {r[k][0]} |")
    with open(md_path, "w") as fh:
        fh.write("\n".join(lines) + "\n")

    def to_bytes(v, u):
        f = float(v.replace(",", ""))
        return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        js = json.load(open(js_path))
    except (OSError, ValueError):
        js = {}
    rd = to_bytes(*vals["dram__bytes_read.sum"])
    wr = to_bytes(*vals["dram__bytes_write.sum"])
    js[kernel] = {"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                  "duration": vals["gpu__time_duration.sum"][0] + " " + vals["gpu__time_duration.sum"][1],
                  "source": os.path.basename(rep)}
    if tau:
        js[kernel]["tau"] = int(tau)
    json.dump(js, open(js_path, "w"), indent=1, sort_keys=True)
    print(open(md_path).read())


def launches(csv_path, md_path):
    rows = list(csv.reader(open(csv_path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    lines = ["# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             f"source: `{os.path.basename(csv_path)}`; cold-cache, serialised: compare shares, not absolutes", "",
             "| # | kernel | duration | unit |", "|---|---|---|---|"]
    tot = {}
    for n, r in enumerate(rows[h + 1:]):
        name = r[ki].split("(")[0]
        lines.append(f"| {n} | {name} | {r[vi]} | {r[ui]} |")
        tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", ""))
    s = sum(tot.values())
    lines += ["", "| kernel | total | share |", "|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {k} | {v:.0f} | {v / s:.1%} |")
    with open(md_path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines[-len(tot) - 2:]))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarise(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
