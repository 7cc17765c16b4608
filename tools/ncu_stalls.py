"""Top warp-stall sites of one kernel in an ncu report (source page, SASS), with the mbarrier
offset each TRYWAIT polls, to tell which pipeline role waits on which barrier."""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]; idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
key = "Warp Stall Sampling (All Samples)"
val = lambda r: float(r[idx[key]] or 0)
tot = sum(val(r) for r in data)
print(f"total samples {tot:.0f}")
for i in sorted(range(len(data)), key=lambda i: -val(data[i]))[:n]:
    r = data[i]
    note = ""
    for j in range(max(0, i - 3), i + 1):
        m = re.search(r"TRYWAIT.*\+0x([0-9a-f]+)\]", data[j][1])
        if m: note = f"  <- waits bar +0x{m.group(1)}"
    print(f"{val(r):7.0f} {100 * val(r) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]}{note}")
