"""Summarise an ncu --set full capture into profiles/<name>.md and record the kernel's
DRAM traffic per launch in profiles/traffic.json (read by bench.py's roofline.traffic).

    python tools/ncu_report.py gpurun_out/prof.ncu-rep profiles/r01_sweep_cfg2.md cfg1 [alg_bytes]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("smsp__inst_executed_op_shared_atom.sum", "shared atomics (warp instr)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    rep, md, key = sys.argv[1], sys.argv[2], sys.argv[3]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
    h, u, v = raw(rep)
    get = {n: (v[i], u[i]) for i, n in enumerate(h)}
    name = get.get("Kernel Name", ("?", ""))[0]
    lines = [f"# ncu --set full: `{name}`", "", f"source capture: `{os.path.basename(rep)}` (config key `{key}`)", "",
             "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in get:
            lines.append(f"| {label} (`{k}`) | {get[k][0]} {get[k][1]} |")
    stalls = sorted(((n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(val or 0)) for n, val in
                     ((n, get[n][0]) for n in get if n.startswith("smsp__pcsamp_warps_issue_stalled_")
                      and not n.endswith("not_issued"))), key=lambda t: -t[1])
    tot = sum(s for _, s in stalls) or 1.0
    lines += ["", "Warp stall samples (top 8):", "", "| reason | share |", "|---|---|"]
    lines += [f"| {n} | {100 * s / tot:.1f}% |" for n, s in stalls[:8]]
    dr = float(get.get("dram__bytes_read.sum", ("0", ""))[0] or 0)
    dw = float(get.get("dram__bytes_write.sum", ("0", ""))[0] or 0)
    unit_r = get.get("dram__bytes_read.sum", ("", "byte"))[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = dr * scale.get(unit_r, 1) + dw * scale.get(get.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
    lines += ["", f"DRAM traffic per launch: {traffic / 1e9:.4f} GB"]
    if alg:
        lines.append(f"algorithmic bytes per launch: {alg / 1e9:.4f} GB (traffic / algorithmic = {traffic / alg:.3f})")
    open(md, "w").write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(md), "traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[key] = {"kernel": name, "dram_bytes_per_launch": traffic, "source": os.path.basename(md)}
    json.dump(d, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
