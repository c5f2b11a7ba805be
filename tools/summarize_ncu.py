"""Summarise ncu outputs brought back from gpurun into profiles/ (tracked).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python tools/summarize_ncu.py full gpurun_out/prof_gemm.ncu-rep profiles/r01_gemm_full.md

`launches` aggregates the per-launch gpu__time_duration list (cold-cache,
serialised by ncu: compare SHARES, not absolute times) by kernel; `full`
extracts the counters the roofline uses (DRAM bytes, tensor-pipe activity,
duration) for every profiled launch of an `ncu --set full` report.
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def _kernel(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(src: str, dst: str) -> None:
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        k = _kernel(r[ki])
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    out = [f"# Launch list summary ({len(data)} launches, `{src}`)", "",
           "ncu `--metrics gpu__time_duration.sum --clock-control none`: per-launch times are cold-cache",
           "and serialised, so the SHARE column is the comparable quantity.", "",
           "| kernel | launches | total us | share | avg us |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / total:.1%} | {v / cnt[k]:.2f} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]


def full(src: str, dst: str) -> None:
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = [f"# ncu --set full summary (`{src}`)", "",
           "| launch | kernel | " + " | ".join(lbl for _, lbl in FULL_METRICS) + " |",
           "|---|---|" + "---:|" * len(FULL_METRICS)]
    for i, r in enumerate(data):
        cells = []
        for metric, _ in FULL_METRICS:
            if metric in hdr:
                j = hdr.index(metric)
                cells.append(f"{r[j]} {units[j]}".strip())
            else:
                cells.append("n/a")
        out.append(f"| {i} | `{_kernel(r[hdr.index('Kernel Name')])}` | " + " | ".join(cells) + " |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
