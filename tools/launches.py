"""Summarise an ncu --csv launch list: per-kernel time and DRAM bytes for the last step."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
skip_first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr = None; data = {}; order = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); k = d['ID']
        if k not in data: data[k] = {'name': d['Kernel Name'][:70]}; order.append(k)
        try: data[k][d['Metric Name']] = float(d['Metric Value'])
        except ValueError: pass
sel = order[skip_first:]
tot = 0
for k in sel:
    d = data[k]; t = d.get('gpu__time_duration.sum', 0) / 1e3; tot += t
    print(f"{t:9.1f} us  R {d.get('dram__bytes_read.sum', 0)/1e6:9.1f} MB  W {d.get('dram__bytes_write.sum', 0)/1e6:8.1f} MB  {d['name']}")
print(f"total {tot:.1f} us over {len(sel)} launches")
