"""Summarise an .ncu-rep: key metrics + top SASS lines by stall samples and exec count."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_shared_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:70s} {vals[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot_s = sum(int(r[i_s] or 0) for r in data) or 1
tot_e = sum(int(r[i_e] or 0) for r in data)
print(f"total stall samples {tot_s}, executed warp instructions {tot_e}")
base = int(data[0][0], 16)
ranked = sorted(data, key=lambda r: -int(r[i_s] or 0))[:top]
for r in sorted(ranked, key=lambda r: int(r[0], 16)):
    print(f"{int(r[0],16)-base:6x} exec {int(r[i_e] or 0):>10} stall {int(r[i_s] or 0):>6} ({100*int(r[i_s] or 0)/tot_s:4.1f}%)  {r[i_src].strip()[:80]}")
