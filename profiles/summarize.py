#!/usr/bin/env python
"""Summarise ncu outputs brought back from the B200 into committed text files.

    python profiles/summarize.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
    python profiles/summarize.py report gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>_ncu.txt
    python profiles/summarize.py traffic gpurun_out/prof.ncu-rep <kernel-key>   # -> profiles/traffic.json

`launches` aggregates an `ncu --metrics gpu__time_duration.sum --clock-control none`
launch list per kernel (count, total, share, mean): cold-cache and serialised, so the
SHARE is what compares with bench.py.  `report` prints the key `--set full` metrics and
the warp-stall breakdown of every kernel in a report.  `traffic` records the dram bytes
per launch of a kernel for bench.py's roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__block_size", "launch__grid_size", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    bscale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    agg = defaultdict(lambda: [0, 0.0, 0.0])  # launches, total us, total dram MB
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        v = float(r[vi].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v * scale.get(r[ui], 1e-3)
        elif metric.startswith("dram__bytes"):
            agg[name][2] += v * bscale.get(r[ui], 1e-6)
    tot = sum(v[1] for v in agg.values())
    print(f"# {os.path.basename(path)}: {sum(v[0] for v in agg.values())} launches, "
          f"total {tot:.1f} us (cold-cache, serialised; the SHARE is what compares with bench.py)")
    print(f"{'share':>7} {'count':>6} {'mean_us':>10} {'dram_MB':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1] / tot * 100:6.2f}% {v[0]:6d} {v[1] / v[0]:10.2f} {v[2] / max(v[0], 1):9.1f}  {k}")


def report(rep):
    recs, units = _raw(rep)
    for d in recs:
        print(f"## {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                print(f"  {k:66s} {d[k]:>16s} {units.get(k, '')}")
        st = []
        for k, v in d.items():
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(x for _, x in st) or 1.0
        print("  warp stalls (share of samples): " + ", ".join(
            f"{k} {x / tot * 100:.1f}%" for k, x in sorted(st, key=lambda t: -t[1])[:8]))
        print()


def traffic(rep, kernel, key=None):
    """dram bytes per launch of `kernel` (first launch in the report) -> traffic.json[key]
    (key: "<workload>/<path>/<kernel>", as bench.py looks it up)."""
    key = key or kernel
    recs, units = _raw(rep)
    d = [r for r in recs if kernel in r.get("Kernel Name", "")][0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[k].replace(",", "")) * scale.get(units.get(k, "byte"), 1)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur[key] = b
    json.dump(cur, open(path, "w"), indent=1)
    print(key, b)


if __name__ == "__main__":
    {"launches": lambda: launches(sys.argv[2]), "report": lambda: report(sys.argv[2]),
     "traffic": lambda: traffic(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)}[sys.argv[1]]()
