"""GEMM DRAM traffic per train step from an ncu step CSV (tools/gpu_hbm_step.sh):
the second of two eager steps (profiler range around the steps), summed over
the tcgen05 GEMM launches (and the split-K reductions that complete them).  Writes the JSON bench.py reads for
`roofline.traffic`.  Usage: python tools/gemm_traffic.py CSV WORKLOAD OUT.json"""
import csv
import json
import sys

path, workload, out = sys.argv[1:4]
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
L = {}
for r in data:
    d = L.setdefault(int(r[0]), {"k": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
ids = sorted(L)
# the capture holds exactly two steps (step_once.py brackets them with
# cudaProfilerStart/Stop, ncu --profile-from-start off): the second half
step = ids[len(ids) // 2:]
gemm = [i for i in step if "gemm_tc" in L[i]["k"] or "split_reduce" in L[i]["k"]]
doc = {
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over "
              f"tools/step_once.py 2 ({workload}, N=1), second of two steps, profiler range around the steps only, "
              f"caches flushed before every kernel; {path.split('/')[-1]}",
    "workload": workload,
    "gemm_launches_per_step": len(gemm),
    "dram_read_bytes_per_step": sum(L[i]["dram__bytes_read.sum"] for i in gemm),
    "dram_write_bytes_per_step": sum(L[i]["dram__bytes_write.sum"] for i in gemm),
    "ncu_gemm_time_s_per_step": sum(L[i]["gpu__time_duration.sum"] for i in gemm),
}
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc))
