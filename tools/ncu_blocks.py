"""Group SASS instructions of an .ncu-rep by execution count (basic-block frequency)."""
import collections
import csv
import io
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
g = collections.defaultdict(lambda: [0, 0, 0, ""])
for r in data:
    e = int(r[i_e])
    if e == 0:
        continue
    g[e][0] += 1
    g[e][1] += e
    g[e][2] += int(r[i_s])
    if not g[e][3]:
        g[e][3] = r[i_src].strip()[:50]
tot = sum(v[1] for v in g.values())
for e, (n, s, st, first) in sorted(g.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"count {e:>10} x {n:>4} instr = {s:>11} ({100*s/tot:5.1f}%)  stall {st:>6}  first: {first}")
