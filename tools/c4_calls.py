"""Per-position kernel totals over the c4 suite (second call of every layer): which step of the
LRQMM chain (by launch order within the call) costs what.   python tools/c4_calls.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data, order = None, {}, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['ID'] not in data:
            data[d['ID']] = {'name': d['Kernel Name']}
            order.append(d['ID'])
        try:
            data[d['ID']][d['Metric Name']] = float(d['Metric Value'])
        except ValueError:
            pass
calls, cur = [], []
for k in order:
    cur.append(k)
    if 'gemm_i8' in data[k]['name'] or 'gemm_tc' in data[k]['name']:
        calls.append(cur)
        cur = []
second = [c for i, c in enumerate(calls) if i % 2 == 1]
tot = defaultdict(float)
for c in second:
    seen = defaultdict(int)
    for k in c:
        n = re.sub(r'\(.*', '', re.sub(r'<.*', '', data[k]['name'].replace('void ', '').replace('lrqmm::', '')))
        seen[n] += 1
        tot[f"{n}#{seen[n]}"] += data[k].get('gpu__time_duration.sum', 0) / 1e3
s = sum(tot.values())
print(f"{len(second)} layer calls, total {s / 1e3:.2f} ms")
for n, t in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{t / 1e3:8.2f} ms  {100 * t / s:5.1f}%  {n}")
