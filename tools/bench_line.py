#!/usr/bin/env python3
"""One-line summary of bench.py JSON lines: python tools/bench_line.py file.json [...] (or stdin)."""
import json
import sys

paths = sys.argv[1:] or ["-"]
for p in paths:
    lines = sys.stdin.read().splitlines() if p == "-" else open(p).read().splitlines()
    for ln in lines:
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        c = d.get("clocks") or {}
        print(f"{p}: {d['config'].get('workload')} value {d['value']:.4e} kernel_ms {r.get('avg_launch_ms', 0):.4f} "
              f"frac {r.get('frac', 0):.3f} traffic_frac {r.get('traffic_frac') or 0:.3f} e2e {e.get('value', 0):.4e} "
              f"sm_mhz {c.get('sm_mhz')} {c.get('reasons')}")
