"""Print the second eager step of an ncu launch list (tools/step_once.py 2) in order."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/step_launches.csv')))
h = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
L = {}
for r in data:
    L.setdefault(int(r[0]), {})['k'] = r[ki]
    L[int(r[0])][r[mi]] = r[vi]
ids = sorted(L)
half = ids[len(ids) // 2:]
def short(k):
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", k)
    return (m.group(1) + (m.group(2) or '')) if m else k[:50]
t = lambda i: float(L[i]['gpu__time_duration.sum'].replace(',', '')) / 1e3
print(len(ids), 'step total us', round(sum(t(i) for i in half), 1), 'gemm us',
      round(sum(t(i) for i in half if 'gemm' in L[i]['k']), 1))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i in half[:n]:
    print(i, short(L[i]['k'])[:55], round(t(i), 1), L[i].get('launch__grid_size'))
