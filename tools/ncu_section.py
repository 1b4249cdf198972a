"""Rewrite one config's section of profiles/<round>/ncu_summary.md from an
ncu --set full raw-page CSV export.
    python tools/ncu_section.py <summary.md> <config> <raw.csv>"""
import csv
import re
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM cycles", "sm__cycles_elapsed.avg"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe active %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tensor-core SMEM operand wavefronts", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum"),
    ("LSU shared-memory wavefronts % of peak",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("FMA pipe cycles active %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("FMA pipe %", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("registers/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def section(cfg, raw):
    rows = list(csv.reader(open(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    col = {n: i for i, n in enumerate(h)}
    out = [f"### {cfg}", "", f"kernel: `{v[col['Kernel Name']][:120]}`", "", "| metric | value |", "|---|---|"]
    traffic = 0.0
    for label, m in METRICS:
        if m in col:
            out.append(f"| {label} (`{m}`) | {v[col[m]]} {u[col[m]]} |")
            if m.startswith("dram__bytes_"):
                traffic += float(v[col[m]]) * SCALE.get(u[col[m]], 1)
    out += ["", f"traffic (read+write) per launch: {traffic:.3e} B", ""]
    return "\n".join(out) + "\n"


def main():
    path, cfg, raw = sys.argv[1:4]
    text = open(path).read()
    new = section(cfg, raw)
    pat = re.compile(rf"### {re.escape(cfg)}\n.*?(?=\n### |\Z)", re.S)
    text = pat.sub(new.rstrip("\n"), text) if pat.search(text) else text.rstrip("\n") + "\n\n" + new
    open(path, "w").write(text)


if __name__ == "__main__":
    main()
