"""Hottest SASS instructions (by warp-stall samples and by executions) of one kernel in an
`ncu --page source --csv` export: python tools/ncu_hot.py file.csv kernel_substring [n]"""
import csv
import sys

path, kname = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(path)))
hdr = cur = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = r[1]
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) > 5 and cur and kname in cur:
        ex = int(r[5]) if r[5].isdigit() else 0
        out.append((int(r[0], 16), r[1].strip(), ex, int(r[2]) if r[2].isdigit() else 0))
base = out[0][0]
ts = sum(x[3] for x in out) or 1
te = sum(x[2] for x in out)
print("instructions executed", te, "stall samples", ts)
for a, s, ex, sm in sorted(sorted(out, key=lambda x: -x[3])[:n]):
    print("%6x %-66s %11d %5.1f%%" % (a - base, s[:66], ex, 100 * sm / ts))
