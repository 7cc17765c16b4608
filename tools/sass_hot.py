"""Top stall-sampled SASS instructions of an ncu `--page source --csv --print-source sass` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = next(i for i, r in enumerate(rows) if 'Warp Stall Sampling (All Samples)' in r)
hdr = rows[k]
idx = hdr.index('Warp Stall Sampling (All Samples)')
ie = hdr.index('Instructions Executed')
data = [(int(r[idx] or 0), i, r[1].strip(), r[ie]) for i, r in enumerate(rows[k + 1:]) if len(r) == len(hdr)]
tot = sum(d[0] for d in data)
print('total samples', tot, 'instructions', len(data))
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for n, i, s, e in sorted(data, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{n:6d} {100.0 * n / max(tot, 1):5.1f}% @{i:5d} {s[:80]:80s} exec={e}")
    for j in range(max(0, i - ctx), i):
        print(f"{'':22s}   {data[j][2][:80]}")
