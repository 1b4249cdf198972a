"""Benchmark: ml(infer) region elements/s (fused gather + infer + scatter).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

One step = one `Runtime.invoke_region` over the config's whole sweep with the
application arrays resident in HBM.  Weak scaling: every rank (one process
per GPU, torchrun) owns an independent shard of `elements` sweep points, no
collective on the data path; value = N*elements / max-over-ranks time.

`e2e` repeats the step through the same public API with the application
arrays in pinned HOST memory (H2D of the inputs and D2H of the outputs inside
the timed region).  `roofline` uses the fused kernel's CUDA-event duration
measured on its stream inside the timed loop.  `--impl reference` times the
CPU restatement of the reference path (oracle/, numpy, same algorithm as the
reference's _run_surrogate) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DEFAULT_CONFIG = "bonds"  # BASELINE.json configs[1]: the headline single-GPU workload
METRIC = "ml(infer) region elements/sec"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
# FP32 CUDA-core peak (no FMA credit: the exact path issues FMUL+FADD):
# 148 SMs x 128 lanes x 1.965 GHz = 37.2 Tinstr/s -> 37.2 TFLOP/s of mul+add.
FP32_NOFMA_TFLOPS_AT_MAX = 148 * 128 * 1.965e9 / 1e12


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------- CPU (port) --

def _cpu_worker(args):
    name, r0, r1 = args
    from oracle import oracle
    from paper_2407_18352_b200 import workloads
    from paper_2407_18352_b200.directives import parse_directive
    wl = workloads.make(name, _cpu_sample_elems(name))
    fi, fo, ti, to = wl.functors()
    arrs = wl.arrays
    src = arrs[ti.array]
    dst = arrs[to.array].copy()
    # the worker's block of axis-0 sweep rows
    s0 = ti.slices[0]
    lo, hi = s0.start + r0 * s0.step, s0.start + r1 * s0.step
    sub = lambda t: parse_directive(  # noqa: E731
        f"map(to: f({t.array}[{lo}:{hi}:{s0.step}" + "".join(f", {s}" for s in t.slices[1:]) + "]))").targets[0]
    st = lambda a: tuple(int(np.prod(a.shape[k + 1:])) for k in range(a.ndim))  # noqa: E731
    t0 = time.perf_counter()
    if name == "particlefilter":
        # the reference expresses the CNN as patch functor + infer + numpy pool
        # + infer; cnn_forward restates exactly that
        x = oracle.gather(fi, sub(ti), src.reshape(-1), src.shape, st(src)).reshape(r1 - r0, -1)
        y, _ = oracle.cnn_forward(wl.layers, x, (1, 128, 128))
        oracle.scatter(fo, sub(to), y, dst.reshape(-1), dst.shape, st(dst))
    else:
        oracle.region([(fi, sub(ti), src.reshape(-1), src.shape, st(src))],
                      [(fo, sub(to), dst.reshape(-1), dst.shape, st(dst))], wl.layers)
    return time.perf_counter() - t0, (r1 - r0) * _inner_rows(wl)


def _inner_rows(wl):
    _, _, ti, _ = wl.functors()
    return int(np.prod([s.count for s in ti.slices[1:]])) if len(ti.slices) > 1 else 1


# CPU sample per config (first sweep rows): a few seconds of reference-path
# work over all host cores; full size for C1 and C5
CPU_SAMPLE = {"options": 1_000_000, "bonds": 262_144, "minibude": 16_384, "miniweather": 4094 * 2046,
              "particlefilter": 2_048}


def _cpu_sample_elems(name):
    n = CPU_SAMPLE[name]
    if name == "miniweather":
        return n
    return n


def cpu_reference(name: str, procs: int):
    """Time the numpy restatement of the reference path (gather -> infer ->
    scatter, runtime.py:308-370) over a bounded sample split across `procs`
    worker processes."""
    import multiprocessing as mp
    from paper_2407_18352_b200 import workloads
    wl = workloads.make(name, _cpu_sample_elems(name))
    _, _, ti, _ = wl.functors()
    rows0 = ti.slices[0].count
    per = -(-rows0 // procs)
    jobs = [(name, r, min(r + per, rows0)) for r in range(0, rows0, per)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(jobs)) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    elems = sum(n for _, n in res)
    return elems / wall, elems, wall


# ------------------------------------------------------------------ GPU arm --

def run_ours(args, rank, world, local):
    import torch
    import paper_2407_18352_b200 as sm
    from paper_2407_18352_b200 import _native, workloads

    _native.lib()
    dev = torch.device("cuda", local)
    wl = workloads.make(args.config, args.elements, seed_offset=rank)
    spec = wl.spec
    wl.to_device(dev)
    tmp = tempfile.mkdtemp(prefix="smlrt_bench_")
    sm.save_model(wl.model, tmp)
    rt = sm.Runtime(device=dev)
    h = rt.register_region(wl.descriptor(tmp))
    for _ in range(args.warmup):
        rt.invoke_region(h)
    torch.cuda.synchronize()

    in_bytes = sum(wl.arrays[k].nbytes for k in wl.arrays if k in (wl.functors()[2].array,))
    flush = None
    if in_bytes < 2 * 126 * 2**20:
        flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)

    rt.kernel_events.clear()
    step_events = []
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rt.invoke_region(h)
            e1.record()
            step_events.append((e0, e1))
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    launches = _native.launch_count() - launches0
    barrier(world)
    ms_steps = sum(a.elapsed_time(b) for a, b in step_events)
    # kernel-only time for the roofline: CUDA events on the launch stream
    # around the native region call alone (a separate loop, same flushing)
    rt.time_kernels = True
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        rt.invoke_region(h)
    torch.cuda.synchronize()
    rt.time_kernels = False
    ms_kernel = [a.elapsed_time(b) for a, b in rt.kernel_events]
    ms_total = max_over_ranks(ms_steps, world)
    ms_per_step = ms_total / args.steps
    value = world * wl.elements / (ms_per_step / 1e3)

    # kernel roofline: achieved = algorithmic work per launch / CUDA-event time
    # of the fused launch; the binding bound is the larger fraction
    #
    pk, pk_src = peaks()
    k_ms = statistics.mean(ms_kernel)
    hbm_gbs = wl.elements * spec.bytes_per_elem / (k_ms / 1e3) / 1e9
    tflops = wl.elements * spec.flops_per_elem / (k_ms / 1e3) / 1e12
    if spec.precision == "bf16":
        # burst figure for a kernel timed alone; the sustained (power-capped)
        # one for a long step (the wide C3 path runs ~100 ms per step)
        if k_ms > 20.0 and "bf16_tflops_sustained" in pk:
            cpeak, cname = pk["bf16_tflops_sustained"], f"bf16_tflops_sustained ({pk_src}, long step)"
        else:
            cpeak, cname = pk["bf16_tflops"], f"bf16_tflops ({pk_src}, burst)"
    else:
        cpeak, cname = FP32_NOFMA_TFLOPS_AT_MAX, "FP32 CUDA-core mul+add issue rate at 1965 MHz (no FMA: exact path)"
    f_hbm, f_cmp = hbm_gbs / pk["hbm_gbs"], tflops / cpeak
    if f_hbm >= f_cmp:
        roof = {"bound": "hbm", "unit": "GB/s", "achieved": round(hbm_gbs, 1), "peak": pk["hbm_gbs"],
                "frac": round(f_hbm, 4), "peak_source": f"hbm_gbs ({pk_src})"}
    else:
        roof = {"bound": "tensor" if spec.precision == "bf16" else "fp32", "unit": "TFLOP/s",
                "achieved": round(tflops, 2), "peak": round(cpeak, 1), "frac": round(f_cmp, 4),
                "peak_source": cname}
    tj = ROOT / "profiles" / "traffic.json"
    traffic = None
    if tj.exists():
        t = json.loads(tj.read_text()).get(spec.name)
        traffic = t and t.get("dram_bytes_per_region")
        if traffic and wl.elements != spec.elements:
            traffic = traffic * wl.elements / spec.elements
    roof.update({"traffic": traffic, "traffic_unit": "DRAM read+write bytes per region call (ncu --set full, profiles/traffic.json)",
                 "alg_bytes_per_launch": wl.elements * spec.bytes_per_elem, "kernel_ms": round(k_ms, 4), "hbm_frac": round(f_hbm, 4),
                 "compute_frac": round(f_cmp, 4), "flops_per_elem": spec.flops_per_elem,
                 "bytes_per_elem": spec.bytes_per_elem})

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hw = workloads.make(args.config, args.elements, seed_offset=rank)
        hw.to_device(pinned_host=True)
        rt2 = sm.Runtime(device=dev)
        h2 = rt2.register_region(hw.descriptor(tmp, name=spec.name + "_host"))
        rt2.invoke_region(h2)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 5))
        for _ in range(e2e_steps):
            rt2.invoke_region(h2)
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world) / e2e_steps
        fi, fo, ti, to = hw.functors()
        h2d = hw.arrays[ti.array].nbytes
        from paper_2407_18352_b200.runtime import _covers
        pout = rt2._plans[spec.name + "_host"][2]
        if not _covers(pout, rt2._staging.device_view(hw.buffers[to.array], dev)):
            h2d += hw.arrays[to.array].nbytes
        d2h = hw.arrays[to.array].nbytes + 4
        e2e = {"value": round(world * hw.elements / e2e_s, 1), "unit": "elements/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(e2e_s * 1e3, 3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        procs = len(os.sched_getaffinity(0))
        v, n, wall = cpu_reference(args.config, procs)
        cpu = {"value": round(v, 1), "unit": "elements/s", "cores": procs, "kind": "port",
               "sample": f"{n} of {wl.elements} elements (first sweep rows), numpy restatement of the"
                         f" reference _run_surrogate path in {procs} processes, {wall:.1f} s"}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "elements/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if spec.precision == "bf16" else "f32",
        "data": "synthetic (seeded uniform/bump arrays, random-init weights)",
        "config": {"workload": spec.name, "elements_per_gpu": wl.elements, "model": "-".join(map(str, spec.dims)),
                   "precision": spec.precision, "directives": [spec.in_functor, spec.out_functor],
                   "parallelism": f"dp{world} (sweep shards, no collective)",
                   "l2": "flushed between steps" if flush is not None else "inputs larger than L2"},
        "roofline": roof, "e2e": e2e, "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "wall_s": round(t_wall, 3),
    }
    if rank == 0:
        print(json.dumps(line))


def run_reference(args, rank, world):
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0))
    from paper_2407_18352_b200 import workloads
    spec = workloads.CONFIGS[args.config]
    vals = []
    for _ in range(args.warmup):
        cpu_reference(args.config, procs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, n, wall = cpu_reference(args.config, procs)
        vals.append(v)
    total = time.perf_counter() - t0
    value = statistics.mean(vals)
    sample = (f"{n} of {spec.elements} elements per step, numpy restatement of the reference"
              f" _run_surrogate path (oracle/oracle.py) in {procs} processes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": spec.name, "model": "-".join(map(str, spec.dims))},
        "cpu_baseline": {"value": round(value, 1), "unit": "elements/s", "cores": procs,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 1), "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--elements", type=int, default=None, help="override the sweep size (testing)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup(args)
    run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
