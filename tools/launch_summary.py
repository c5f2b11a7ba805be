"""Per-kernel share of one bench step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none
--profile-from-start off --csv` over `bench.py --steps 2`; bench.py brackets
its timed steps with cudaProfilerStart/Stop, so the capture holds exactly the
timed graph replays).  The second step is summarised.
Usage: python tools/launch_summary.py CSV [title] > profiles/....md"""
import collections
import csv
import re
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
L = {}
for r in data:
    L.setdefault(int(r[0]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(L)
step = ids[len(ids) // 2:]


def short(k):
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", k)
    return (m.group(1) + (m.group(2) or "")) if m else k[:60]


agg = collections.OrderedDict()
for i in step:
    a = agg.setdefault(short(L[i]["k"]), [0, 0.0])
    a[0] += 1
    a[1] += L[i]["gpu__time_duration.sum"] / 1e3
tot = sum(a[1] for a in agg.values())
gemm = sum(a[1] for k, a in agg.items() if k.startswith("gemm_"))
print(f"# {title}\n")
print("`ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off` "
      "over `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (the capture holds the two timed CUDA-graph "
      "replays; the second is summarised).  ncu serialises kernels and its bench line is not a measurement: "
      "compare shares.\n")
print("| kernel | launches | total us | share | avg us |")
print("|---|---:|---:|---:|---:|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {t:.1f} | {t / tot:.1%} | {t / n:.1f} |")
print(f"\nStep total {tot:.1f} us over {len(step)} launches; tcgen05 GEMM launches {gemm / tot:.1%}.")
