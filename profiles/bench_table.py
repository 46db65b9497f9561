#!/usr/bin/env python
"""Markdown table of committed bench lines:
    python profiles/bench_table.py profiles/r02/bench_c4_default.json profiles/r02/bench_configs.jsonl"""
import json
import sys

rows = []
for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            rows.append(json.loads(line))
print("| config | points | path | step ms | evals/s | bin / main / combine ms | roofline frac (useful) | executed MMA frac | e2e ms | oracle evals/s |")
print("|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c, r, ph = d["config"], d["roofline"], d.get("phases_ms", {})
    name = c["config"] + (f" h={c['h_px']:g}" if c.get("h_px") is not None else "")
    if c.get("dp_eps_m") is not None:
        name += f" DP ε={c['dp_eps_m']:g} m"
    if c.get("path") == "snap":
        print(f"| {name} | {c['n_points']} | snap (Alg. 3 + Eq. 7) | {d['ms_per_step']:.3f} | {d['value']:.3g} taps/s | whole call | {r['frac']:.3f} HBM | – | {d['e2e']['ms_per_step']:.2f} | – |")
        continue
    cpu = d.get("cpu_baseline", {}).get("value")
    print(f"| {name} | {c['n_points']} | {c['path']} | {d['ms_per_step']:.3f} | {d['value']:.3g} | "
          f"{ph.get('bin_ms', 0):.3f} / {ph.get('main_ms', 0):.3f} / {ph.get('combine_ms', 0):.3f} | "
          f"{r['frac']:.4f} {r['bound']} | {r.get('executed_frac', '–')} | {d['e2e']['ms_per_step']:.2f} | "
          f"{cpu:.3g} |" if cpu else "– |")
