"""Stall samples per SASS instruction of a one-kernel .ncu-rep, grouped into address ranges
split at labels the user gives (or the top N instructions): python tools/ncu_stalls.py rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
ia, isrc, ist, ie = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), \
    hh.index("Instructions Executed")
# stall reason columns, if present
reason_cols = [(i, n) for i, n in enumerate(hh) if n.startswith("stall_") or n.startswith("Stall ")]
tot = sum(int(r[ist] or 0) for r in data)
base = int(data[0][ia], 16)
print(f"total samples {tot}; reason columns: {len(reason_cols)}")
recs = []
for k, r in enumerate(data):
    s = int(r[ist] or 0)
    recs.append((s, int(r[ia], 16) - base, r[isrc].strip(), int(r[ie] or 0), k))
# running window: print every instruction with >= 0.3 % of samples, in address order
for s, a, t, e, k in recs:
    if s >= tot * 0.003:
        print(f"{a:6x} {100 * s / tot:5.1f}% ex={e:>10d}  {t}")
if len(sys.argv) > 3:
    cuts = [int(x, 16) for x in sys.argv[3].split(",")]
    bounds = [0] + cuts + [1 << 40]
    for lo, hi in zip(bounds, bounds[1:]):
        s = sum(r[0] for r in recs if lo <= r[1] < hi)
        e = sum(r[3] for r in recs if lo <= r[1] < hi)
        print(f"[{lo:6x},{hi:6x}) samples {100 * s / tot:5.1f}%  inst {e}")
