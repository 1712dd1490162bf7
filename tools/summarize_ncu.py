"""Summarise ncu raw-page CSV exports (tools/run_profiles.sh) into a
markdown table for profiles/: per kernel launch duration, DRAM bytes
(traffic), DRAM throughput, issue activity, occupancy, lane efficiency and
the top stall reasons.  Also summarises a --metrics gpu__time_duration launch
list into per-kernel shares.

    python tools/summarize_ncu.py launches gpurun_out/launches_c2.csv
    python tools/summarize_ncu.py raw gpurun_out/prof_c2_r1_raw.csv
"""

from __future__ import annotations

import csv
import sys
from collections import defaultdict

# time -> milliseconds, bytes -> bytes
UNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def _f(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return float("nan")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    k, v, u = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= v:
            continue
        name = r[k]
        tot[name] += _f(r[v]) * UNIT.get(r[u], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    print("| kernel | launches | total ms (ncu, serialised, cold) | share |")
    print("|---|---|---|---|")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{name}` | {cnt[name]} | {ms:.3f} | {ms / T:.3f} |")
    print(f"| **total** | {sum(cnt.values())} | {T:.3f} | 1.000 |")


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]

    def col(name):
        return h.index(name) if name in h else None

    def val(r, name):
        i = col(name)
        if i is None:
            return float("nan")
        return _f(r[i]) * UNIT.get(units[i], 1.0)

    stalls = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")]
    print("| kernel | time us | DRAM read MB | DRAM write MB | traffic GB/s | DRAM % peak | issue active % | warps active % | lanes/instr | regs | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        name = r[col("Kernel Name")]
        t_ms = val(r, "gpu__time_duration.sum")
        rd = val(r, "dram__bytes_read.sum") / 1e6
        wr = val(r, "dram__bytes_write.sum") / 1e6
        gbs = (rd + wr) * 1e6 / (t_ms * 1e-3) / 1e9 if t_ms else float("nan")
        st = sorted(((_f(r[i]), h[i]) for i in stalls), reverse=True)[:3]
        sts = ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}" for v, n in st)
        print(f"| `{name}` | {t_ms * 1e3:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | "
              f"{val(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{val(r, 'smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | "
              f"{val(r, 'launch__registers_per_thread'):.0f} | {sts} |")


if __name__ == "__main__":
    {"launches": launches, "raw": raw}[sys.argv[1]](sys.argv[2])
