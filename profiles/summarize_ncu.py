#!/usr/bin/env python
"""Summarise ncu exports into the markdown committed under profiles/.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv
    python profiles/summarize_ncu.py full raw.csv  > profiles/rNN_<cfg>_ncu_full.md
    python profiles/summarize_ncu.py launches launches.csv > profiles/rNN_<cfg>_launches.md
"""
import collections
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(lbl for _, lbl in KEYS) + " | top stall reasons |")
    print("|---|" + "---|" * (len(KEYS) + 1))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("galois::", "")
        cells = []
        for k, _ in KEYS:
            if k in h:
                i = h.index(k)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        st.sort(reverse=True)
        cells.append(", ".join(f"{k} {v / tot:.0%}" for v, k in st[:4]))
        print(f"| {name} | " + " | ".join(cells) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("galois::", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for k, v in agg.items():
        print(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.1%} |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
