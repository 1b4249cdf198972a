"""Summarise `ncu --set full` reports as markdown tables (run where ncu is).

    python tools/ncu_summary.py gpurun_out/prof_bonds.ncu-rep [...] > summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM cycles", "sm__cycles_elapsed.avg"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe active %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tensor-core SMEM operand wavefronts", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum"),
    ("LSU shared-memory wavefronts % of peak", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("FMA pipe cycles active %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("registers/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]


def summarise(rep: str) -> str:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    out = []
    for rec in data:
        col = dict(zip(head, rec))
        unit = dict(zip(head, units))
        out.append(f"### {rep.rsplit('/', 1)[-1]}\n\nkernel: `{col.get('Kernel Name', '?')}`\n")
        out.append("| metric | value |\n|---|---|")
        for name, m in METRICS:
            if m in col:
                out.append(f"| {name} (`{m}`) | {col[m]} {unit.get(m, '')} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n".join(summarise(r) for r in sys.argv[1:]))
