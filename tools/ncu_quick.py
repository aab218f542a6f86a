"""Quick look at one-kernel .ncu-rep: key metrics, stall reasons, instruction mix per opcode
and executed instructions per address block: python tools/ncu_quick.py rep [units]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for w in want:
    if w in h:
        print(f"{w:64s} {v[h.index(w)]} {u[h.index(w)]}")
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in n:
        try:
            st.append((float(v[i].replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in sorted(st, reverse=True)[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
i_src, i_e, i_a = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Address")
ops = collections.Counter()
tot = 0
for r in data:
    e = int(r[i_e] or 0)
    tot += e
    t = r[i_src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += e
print(f"instructions {tot} = {tot / units:.0f} per unit")
print("  " + ", ".join(f"{k} {v / units:.0f}" for k, v in ops.most_common(22)))
