"""Summarise an ncu report into the numbers DESIGN.md / bench.py cite.

    python profiles/summarize.py <report.ncu-rep> [name]  -> prints markdown, updates profiles/traffic.json
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "tensor-core SMEM operand wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "LSU shared-memory wavefronts % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    rep = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else Path(rep).stem
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"### {name}\n\nkernel: `{kname[:120]}`\n\n| metric | value |\n|---|---|")
    got = {}
    for key, label in KEYS:
        if key in hdr:
            i = hdr.index(key)
            got[key] = (vals[i], units[i])
            print(f"| {label} (`{key}`) | {vals[i]} {units[i]} |")
    tr = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = got.get(k, ("0", "byte"))
        tr += float(v.replace(",", "")) * UNIT.get(u, 1.0)
    tj = Path(__file__).resolve().parent / "traffic.json"
    d = json.loads(tj.read_text()) if tj.exists() else {}
    d[name] = {"dram_bytes_per_launch": tr, "report": Path(rep).name}
    tj.write_text(json.dumps(d, indent=1) + "\n")
    print(f"\ntraffic (read+write) per launch: {tr:.4g} B")


if __name__ == "__main__":
    main()
