"""Sum an ncu launch list of tools/c4_all.py per kernel type (second call of every layer only)."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data, order = {}, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d['ID']
        if k not in data:
            data[k] = {'name': d['Kernel Name']}
            order.append(k)
        try:
            data[k][d['Metric Name']] = float(d['Metric Value'])
        except ValueError:
            pass
# split into calls: a call starts at the first quantize of side A after a GEMM
calls, cur = [], []
for k in order:
    n = data[k]['name']
    cur.append(k)
    if 'gemm_i8' in n or 'gemm_tc' in n:
        calls.append(cur)
        cur = []
second = [c for i, c in enumerate(calls) if i % 2 == 1]
tot = defaultdict(float)
for c in second:
    for k in c:
        n = re.sub(r'<.*', '', data[k]['name'].replace('void ', '').replace('lrqmm::', ''))
        n = re.sub(r'\(.*', '', n)
        tot[n] += data[k].get('gpu__time_duration.sum', 0) / 1e3
s = sum(tot.values())
print(f"{len(second)} layer calls, total {s / 1e3:.2f} ms")
for n, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{t / 1e3:8.2f} ms  {100 * t / s:5.1f}%  {n}")
