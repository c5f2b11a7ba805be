"""Summarise an ncu step CSV with DRAM bytes (tools/gpu_hbm_step.sh): the
second of two eager steps (profiler range around the steps), per kernel:
launches, total time, DRAM bytes read + written, achieved GB/s and the
fraction of the measured HBM peak.
Usage: python tools/hbm_summary.py CSV [title] > profiles/....md"""
import collections
import csv
import json
import os
import re
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(path)
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9}
L = {}
for r in data:
    d = L.setdefault(int(r[0]), {"k": r[ki]})
    v = float(r[vi].replace(",", ""))
    d[r[mi]] = v * scale.get(r[ui], 1)
ids = sorted(L)
# the capture holds exactly two steps (step_once.py brackets them with
# cudaProfilerStart/Stop, ncu --profile-from-start off): the second half
step = ids[len(ids) // 2:]


def short(k):
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", k)
    return (m.group(1) + (m.group(2) or "")) if m else k[:60]


peak = 6552.0
mp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")
if os.path.exists(mp):
    peak = json.load(open(mp))["hbm_gbs"]
agg = collections.OrderedDict()
for i in step:
    d = L[i]
    a = agg.setdefault(short(d["k"]), [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d["gpu__time_duration.sum"]
    a[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
tot_t = sum(a[1] for a in agg.values())
print(f"# {title}\n")
print("ncu `gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum` per launch, caches flushed "
      "before every kernel (ncu default), the second of two eager steps (profiler range around the steps only) "
      "(`tools/step_once.py 2`). ncu serialises "
      f"launches: compare shares and GB/s, not the absolute step time. HBM peak {peak:.0f} GB/s "
      "(MEASURED_PEAKS.json copy bandwidth).\n")
print("| kernel | launches | total us | share | DRAM MB | GB/s | frac of HBM peak |")
print("|---|---:|---:|---:|---:|---:|---:|")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = b / t / 1e9 if t else 0.0
    print(f"| `{k}` | {n} | {t * 1e6:.1f} | {t / tot_t:.1%} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")
print(f"\nStep total {tot_t * 1e6:.1f} us over {len(step)} launches.")
