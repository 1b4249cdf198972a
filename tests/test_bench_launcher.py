"""bench.py plumbing on CPU: the self-spawning multi-rank launcher (gloo),
the parity report and the CPU-baseline restatement."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2407_18352_b200 import workloads  # noqa: E402


def test_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "bonds",
                          "--launcher-selftest"], env=env, capture_output=True, text=True, timeout=180)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["ms_per_step"] == 2.0  # max over ranks of rank + 1
    (a0, a1), (b0, b1) = line["shards"]
    assert a0 == 0 and a1 == b0 and b1 == line["rows"]


def test_parity_report_on_oracle_output():
    for name, n in [("options", 2000), ("bonds", 300), ("miniweather", 40 * 130)]:
        wl = workloads.make(name, n)
        _, _, _, to = wl.functors()
        out = wl.arrays[to.array].copy()
        rows = wl.elements // bench._inner_rows(wl)
        bench._oracle_rows(wl, 0, rows, out)
        p = bench.parity(wl, out, rows, band=64)
        assert p["bitwise"] and p["max_abs"] == 0.0 and p["pass"], (name, p)
        out_bad = out.copy()
        out_bad.reshape(-1)[np.flatnonzero(out_bad.reshape(-1))[:1]] += 1.0
        assert not bench.parity(wl, out_bad, rows, band=64)["bitwise"]


def test_cpu_reference_times_row_work_only():
    bench.CPU_SAMPLE["options"] = 4096
    ref = bench.CpuReference("options", 2)
    v, n, wall = ref.run()
    ref.close()
    assert n == 4096 and v > 0 and wall > 0
