#!/usr/bin/env python3
"""Summarise ncu output for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>      per-kernel count / time / share
  python tools/ncu_summary.py full <report.ncu-rep>         key metrics + SASS mix of the captured kernel
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = re.compile(r"^(gpu__time_duration.sum|dram__bytes_(read|write).sum|dram__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"lts__t_sector_hit_rate.pct|lts__t_sectors_srcunit_ltcfabric.sum|lts__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"l1tex__t_sector_hit_rate.pct|sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread|"
                  r"launch__grid_size|launch__block_size|launch__occupancy_limit_registers|smsp__inst_executed.sum|"
                  r"smsp__issue_active.avg.pct_of_peak_sustained_active|sm__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"smsp__average_warps_issue_stalled_(long_scoreboard|wait|short_scoreboard|not_selected|branch_resolving)_per_issue_active.ratio|"
                  r"sm__sass_inst_executed_op_global_ld.sum|sm__sass_inst_executed_op_global_st.sum|"
                  r"l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum|l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum|"
                  r"sm__maximum_warps_per_active_cycle_pct|sm__warps_active.avg.per_cycle_active)$")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iV:
            continue
        v = float(r[iV].replace(",", ""))
        ms = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[iU], 1e-6) * v
        a = agg.setdefault(r[iN].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: gpu__time_duration.sum per launch (ncu, --clock-control none, serialised, cold cache)")
    print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
    for k, (c, ms) in agg.items():
        print(f"{k:34s} {c:8d} {ms:10.3f} {ms / c * 1e3:10.2f} {100 * ms / tot:6.1f}%")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"# {path}: {r[hdr.index('Kernel Name')]}")
        for i, h in enumerate(hdr):
            if KEYS.search(h):
                print(f"{h:80s} {r[i]:>18s} {units[i]}")
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(sass.splitlines()))
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    c, cw, tot, totw = collections.Counter(), collections.Counter(), 0, 0
    for r in rows[2:]:
        try:
            e, w = int(r[iE]), int(r[iW])
        except (ValueError, IndexError):
            continue
        s = r[iS].strip()
        op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0] if s else "?"
        c[op] += e
        cw[op] += w
        tot += e
        totw += w
    print(f"# SASS mix: {tot} warp instructions; opcode: % of instructions / % of stall samples")
    print(" ".join(f"{op}:{100 * e / tot:.1f}%/{100 * cw[op] / max(totw, 1):.0f}%" for op, e in c.most_common(30)))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
