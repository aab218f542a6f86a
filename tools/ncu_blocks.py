"""Group the SASS of one kernel in an .ncu-rep by execution count (basic-block frequency):
    python tools/ncu_blocks.py rep.ncu-rep [kernel-substring] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1]]
        sections.append(cur)
    elif cur is not None:
        cur.append(r)
if not sections:  # single-kernel report: no "Kernel Name" rows
    sections = [["?"] + rows]
for sec in sections:
    if want not in sec[0]:
        continue
    h, data = sec[1], [x for x in sec[2:] if len(x) > 5]
    ie, isrc, isa = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    g = collections.defaultdict(lambda: [0, 0, 0, []])
    for x in data:
        n = int(x[ie] or 0)
        if n == 0:
            continue
        g[n][0] += 1
        g[n][1] += n
        g[n][2] += int(x[isa] or 0)
        g[n][3].append(x[isrc].strip())
    tot = sum(v[1] for v in g.values())
    print(f"{sec[0][:100]}: {tot} warp instructions")
    for n, v in sorted(g.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"exec {n:9d} x{v[0]:4d} = {v[1] / tot * 100:5.1f}%  samples {v[2]}")
        print("     ", " | ".join(v[3][:12])[:300])
