#!/usr/bin/env python3
"""Markdown table of the bench lines under profiles/ (one row per JSON line): throughput, step kernel, the
roofline fields bench.py reports and the clocks seen. Run here, no GPU:  python tools/roofline_report.py [r2]"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
print("| file | workload | upd/s | e2e upd/s | step kernel ms | frac (algorithmic / measured copy peak) | "
      "frac of nominal 8 TB/s | DRAM / compulsory | SM MHz | exchange |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{tag}_bench_*.json"))):
    try:
        d = json.load(open(f))
    except (OSError, ValueError):
        continue
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    fmt = lambda x, p="%.3g": (p % x) if isinstance(x, (int, float)) else "—"
    print(f"| {os.path.basename(f)} | {d.get('config', {}).get('workload', '—')} | {fmt(d.get('value'))} | "
          f"{fmt(e2e)} | {fmt(r.get('avg_launch_ms'), '%.4f')} | {fmt(r.get('frac'), '%.2f')} | "
          f"{fmt(r.get('frac_nominal'), '%.2f')} | {fmt(r.get('dram_frac_vs_compulsory'), '%.2f')} | "
          f"{fmt((d.get('clocks') or {}).get('sm_mhz'), '%.0f')} | {d.get('config', {}).get('exchange', '—')} |")
