"""Benchmark: ml(infer) region elements/s (fused gather + infer + scatter).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME]
                    [--scaling weak|strong] [--impl ours|reference]
                    [--no-per-config] [--no-e2e] [--no-cpu]

One step = one `Runtime.invoke_region` over the config's whole sweep with the
application arrays resident in HBM.  The headline line is BASELINE.json's
metric on the largest single-GPU config, C3 MiniBUDE (6-1024-512-256-1 over
67,108,864 poses, bf16 tcgen05); `per_config` in the same line carries the
value, kernel time, roofline, e2e and parity of all five frozen configs
(SURVEY.md section 8(d)).

Multi-GPU: one process per GPU.  Under torchrun the
ranks come from the environment; `--gpus N` without WORLD_SIZE spawns the N
ranks itself (127.0.0.1 rendezvous).  `--scaling weak` (default): every rank
owns an independent dataset of `elements` sweep points, no collective on the
data path.  `--scaling strong`: one dataset, rank r processes its block of
sweep rows (`Runtime(shard=(r, N))`).  MiniWeather at N > 1 always runs the
row-slab stepper (`halo.py`): one grouped NCCL halo exchange + the region per
step over the global 4096 x 2048 grid (strong).  value = elements all ranks
processed / max-over-ranks device time.

`e2e` repeats the step through the same public API with the application
arrays in pinned HOST memory (H2D of the inputs and D2H of the outputs inside
the timed region).  `roofline` uses the fused kernel's CUDA-event duration
measured on its launch stream inside the bench.  `parity` compares the GPU
output with the CPU oracle (C / numpy restatement of the reference path) on
the CPU-baseline sample rows (all rows for C1 and C5).  `--impl reference`
times the CPU restatement of the reference path on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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

ALL_CONFIGS = ["options", "options_bf16", "bonds", "minibude", "particlefilter", "particlefilter_bf16",
               "miniweather", "miniweather_bf16"]
DEFAULT_CONFIG = "minibude"  # the largest single-GPU config (BASELINE.json configs[2])
METRIC = "ml(infer) region elements/sec"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

# CPU baseline samples (first sweep rows): all-cores
# variant / as-shipped one-process variant
CPU_SAMPLE = {"options": 1_000_000, "options_bf16": 1_000_000, "bonds": 262_144, "minibude": 16_384, "particlefilter": 2_048,
              "particlefilter_bf16": 2_048,
              "miniweather": 4094 * 2046, "miniweather_bf16": 4094 * 2046}
CPU_SAMPLE_1P = {"options": 250_000, "options_bf16": 250_000, "bonds": 16_384, "minibude": 1_024, "particlefilter": 256,
                 "particlefilter_bf16": 256,
                 "miniweather": 512 * 2046, "miniweather_bf16": 512 * 2046}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return PEAKS_FALLBACK, "fallback"


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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
            self._stop.wait(0.1)

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


# ------------------------------------------------------------ ranks / launch --

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` without torchrun: run N copies of this script as ranks 0..N-1
    (one per GPU, 127.0.0.1 rendezvous); rank 0 prints the line."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:], env=env))
    return max(p.wait() for p in procs)


# SMLRT_BENCH_SHARED_GPU=1 (diagnostic): every rank on cuda:0 with gloo
# collectives -- exercises the N > 1 code paths (weak/strong shards, the
# MiniWeather slab stepper, max-over-ranks timing) on a one-GPU box; never a
# scaling number
SHARED_GPU = os.environ.get("SMLRT_BENCH_SHARED_GPU") == "1"


def dist_setup(backend="nccl"):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU and backend == "nccl":
        backend, local = "gloo", 0
        torch.cuda.set_device(0)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            # NCCL's init log (communicator size, transports) goes to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    on_dev = device is not None and dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=device if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------- CPU (port) --

_CPU_WL = None  # the sample workload, generated before the pool forks (not timed)


def _sub_target(t, r0, r1):
    """Rows [r0, r1) of sweep axis 0 of a map target, as a new target."""
    from paper_2407_18352_b200.directives import parse_directive
    s0 = t.slices[0]
    lo, hi = s0.start + r0 * s0.step, s0.start + r1 * s0.step
    txt = f"map(to: f({t.array}[{lo}:{hi}:{s0.step}" + "".join(f", {s}" for s in t.slices[1:]) + "]))"
    return parse_directive(txt).targets[0]


def _strides(a):
    return tuple(int(np.prod(a.shape[k + 1:])) for k in range(a.ndim))


def _inner_rows(wl):
    _, _, ti, _ = wl.functors()
    return int(np.prod([s.count for s in ti.slices[1:]])) if len(ti.slices) > 1 else 1


def _oracle_rows(wl, r0, r1, out=None):
    """Reference path (gather -> infer -> scatter, runtime.py:308-370) over
    sweep rows [r0, r1) of `wl` with the numpy oracle; returns the elements
    processed.  The CNN is the reference's patch functor + infer + pool +
    infer composition."""
    from oracle import oracle
    fi, fo, ti, to = wl.functors()
    src = wl.arrays[ti.array]
    dst = out if out is not None else wl.arrays[to.array].copy()
    if wl.spec.cnn:
        x = oracle.gather(fi, _sub_target(ti, r0, r1), src.reshape(-1), src.shape, _strides(src))
        y, _ = oracle.cnn_forward(wl.layers, x.reshape(r1 - r0, -1), (1, 128, 128))
        oracle.scatter(fo, _sub_target(to, r0, r1), y, dst.reshape(-1), dst.shape, _strides(dst))
    else:
        oracle.region([(fi, _sub_target(ti, r0, r1), src.reshape(-1), src.shape, _strides(src))],
                      [(fo, _sub_target(to, r0, r1), dst.reshape(-1), dst.shape, _strides(dst))], wl.layers)
    return (r1 - r0) * _inner_rows(wl)


def _cpu_job(rng):
    r0, r1 = rng
    return _oracle_rows(_CPU_WL, r0, r1)


class CpuReference:
    """The reference path restated on the host (oracle/, numpy): P worker
    processes forked once over the pre-generated sample, each on a disjoint
    block of sweep rows; `run()` times only the row work (pool map), not the
    fork or the data generation."""

    def __init__(self, name: str, procs: int, sample: int | None = None):
        global _CPU_WL
        import multiprocessing as mp
        from paper_2407_18352_b200 import workloads
        _CPU_WL = workloads.make(name, sample or CPU_SAMPLE[name])
        self.wl = _CPU_WL
        _, _, ti, _ = self.wl.functors()
        rows0 = ti.slices[0].count
        self.rows0 = rows0
        self.procs = procs
        per = -(-rows0 // procs)
        self.jobs = [(r, min(r + per, rows0)) for r in range(0, rows0, per)]
        self.pool = mp.get_context("fork").Pool(len(self.jobs)) if procs > 1 else None
        if self.pool is not None:
            self.pool.map(_warm, range(len(self.jobs)))

    def run(self):
        t0 = time.perf_counter()
        if self.pool is None:
            n = _oracle_rows(self.wl, 0, self.rows0)
        else:
            n = sum(self.pool.map(_cpu_job, self.jobs))
        wall = time.perf_counter() - t0
        return n / wall, n, wall

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def _warm(_):
    """Imports and first-call setup in each worker (one sweep row), untimed."""
    _oracle_rows(_CPU_WL, 0, 1)
    return os.getpid()


def cpu_baseline(name: str, total_elems: int):
    """Both CPU variants of BASELINE.md section 3, timed on this host."""
    procs = len(os.sched_getaffinity(0))
    ref = CpuReference(name, procs)
    ref.run()  # warm-up: first-touch page faults of the forked workers
    v_all, n_all, w_all = ref.run()
    ref.close()
    one = CpuReference(name, 1, CPU_SAMPLE_1P[name])
    one.run()
    v_one, n_one, w_one = one.run()
    return {"value": round(v_all, 1), "unit": "elements/s", "cores": procs, "kind": "port",
            "cpu": cpu_model(),
            "sample": f"{n_all} of {total_elems} elements (first sweep rows), numpy restatement of the"
                      f" reference _run_surrogate path in {procs} forked processes, {w_all:.2f} s"
                      " (fork and data generation excluded)",
            "one_process": {"value": round(v_one, 1), "cores": 1, "elements": n_one, "wall_s": round(w_one, 2),
                            "note": "as shipped: the reference runs in one process, no BLAS"}}


# ------------------------------------------------------------------ parity --

def parity(wl, out_host, rows: int, band: int = 512):
    """GPU output vs the CPU oracle on sweep rows [0, rows): the GPU's output
    array is read back through the out functor (numpy oracle gather) and
    compared with the oracle's forward pass on the same gathered inputs
    (C restatement of models.py:188-224 for dense models, the reference
    composition for the CNN).  fp32-exact configs must be bitwise; bf16
    within max-abs <= 2e-2 max|ref| and RMSE/RMS <= 1e-2."""
    from oracle import c_oracle, oracle
    fi, fo, ti, to = wl.functors()
    src = wl.arrays[ti.array]
    got_all, ref_all = [], []
    for r0 in range(0, rows, band):
        r1 = min(rows, r0 + band)
        x = oracle.gather(fi, _sub_target(ti, r0, r1), src.reshape(-1), src.shape, _strides(src))
        x = x.reshape(-1, fi.feature_count)
        if wl.spec.cnn:
            y, _ = oracle.cnn_forward(wl.layers, x, (1, 128, 128))
        else:
            y, _ = c_oracle.mlp_f32(wl.layers, x)
        g = oracle.gather(fo, _sub_target(to, r0, r1), out_host.reshape(-1), out_host.shape, _strides(out_host))
        got_all.append(g.reshape(-1, fo.feature_count).astype(np.float64))
        ref_all.append(y.astype(np.float64))
    got, ref = np.concatenate(got_all), np.concatenate(ref_all)
    d = np.abs(got - ref)
    scale = float(np.abs(ref).max()) or 1.0
    rms = float(np.sqrt(np.mean(ref ** 2))) or 1.0
    sig = np.abs(ref) >= 1e-3 * scale
    exact = wl.spec.precision != "bf16"
    res = {
        "vs": "CPU oracle (C/numpy restatement of models.py:188-224, pinned to reference goldens)",
        "rows_checked": int(rows), "elements_checked": int(got.size),
        "max_abs": float(d.max()), "max_rel": float((d[sig] / np.abs(ref[sig])).max()) if sig.any() else 0.0,
        "norm_max_abs": float(d.max() / scale), "rmse_rel": float(np.sqrt(np.mean(d ** 2)) / rms),
        "bitwise": bool(np.array_equal(got.view(np.uint64), ref.view(np.uint64))),
    }
    if exact:
        res["tolerance"] = "bitwise (fp32-exact path)"
        res["pass"] = res["bitwise"]
    else:
        res["tolerance"] = "max_abs <= 2e-2*max|ref| and rmse_rel <= 1e-2 (bf16 path)"
        res["pass"] = res["norm_max_abs"] <= 2e-2 and res["rmse_rel"] <= 1e-2
    return res


# ------------------------------------------------------------------ GPU arm --

def roofline(spec, elems, k_ms, pk, pk_src, fp32_peak):
    """achieved = algorithmic work of one launch / its CUDA-event time; the
    binding bound is the larger fraction."""
    hbm_gbs = elems * spec.bytes_per_elem / (k_ms / 1e3) / 1e9
    tflops = elems * spec.flops_per_elem / (k_ms / 1e3) / 1e12
    if spec.precision == "bf16":
        if k_ms > 20.0 and "bf16_tflops_sustained" in pk:
            cpeak, cname = pk["bf16_tflops_sustained"], f"bf16_tflops_sustained ({pk_src}, long launch)"
        else:
            cpeak, cname = pk["bf16_tflops"], f"bf16_tflops ({pk_src}, burst)"
    else:
        cpeak, cname = fp32_peak / 1e12, ("FP32 packed mul.f32x2 + fma.f32x2(p,1,acc) (the exact kernels'"
                                          " ordered mul-then-add), measured live by smlrt_fp32_peak")
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
        if traffic and elems != spec.elements:
            traffic = traffic * elems / spec.elements
    roof.update({"traffic": traffic,
                 "traffic_unit": "DRAM read+write bytes per region call (ncu --set full, profiles/traffic.json)",
                 "alg_bytes_per_launch": elems * spec.bytes_per_elem, "kernel_ms": round(k_ms, 4),
                 "hbm_frac": round(f_hbm, 4), "compute_frac": round(f_cmp, 4),
                 "flops_per_elem": spec.flops_per_elem, "bytes_per_elem": spec.bytes_per_elem})
    return roof


def _flush_buffer(wl, dev):
    import torch
    _, _, ti, _ = wl.functors()
    if wl.arrays[ti.array].nbytes < 2 * 126 * 2**20:
        return torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)
    return None


def measure(name, args, rank, world, local, dev, headline, pk, pk_src, fp32_peak, tmp):
    import torch
    import paper_2407_18352_b200 as sm
    from paper_2407_18352_b200 import _native, workloads

    if name == "miniweather" and world > 1:
        return measure_halo(args, rank, world, local, dev, headline, pk, pk_src, fp32_peak, tmp)
    strong = args.scaling == "strong" and world > 1
    elements = args.elements if (args.elements and name == args.config) else None
    wl = workloads.make(name, elements, seed_offset=0 if strong else rank)
    spec = wl.spec
    wl.to_device(dev)
    mdir = os.path.join(tmp, name)
    sm.save_model(wl.model, mdir)
    shard = (rank, world) if strong else None
    rt = sm.Runtime(device=dev, shard=shard)
    h = rt.register_region(wl.descriptor(mdir))
    rows0 = wl.elements // _inner_rows(wl)
    from paper_2407_18352_b200.runtime import _shard_rows
    for _ in range(args.warmup):
        rt.invoke_region(h)
    torch.cuda.synchronize()
    flush = _flush_buffer(wl, dev)
    steps = args.steps if headline else min(args.steps, 10)

    step_events = []
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    clk = ClockSampler(local) if headline else None
    if clk:
        clk.__enter__()
    t_wall = time.perf_counter()
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rt.invoke_region(h)
        e1.record()
        step_events.append((e0, e1))
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if clk:
        clk.__exit__(None, None, None)
    launches = _native.launch_count() - launches0
    barrier(world)
    ms_steps = sum(a.elapsed_time(b) for a, b in step_events)
    # kernel-only time for the roofline: CUDA events on the launch stream
    # around the native region call alone (a separate loop, same flushing)
    rt.time_kernels = True
    rt.kernel_events.clear()
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        rt.invoke_region(h)
    torch.cuda.synchronize()
    rt.time_kernels = False
    k_ms = statistics.mean(rt.kernel_times())
    ms_per_step = max_over_ranks(ms_steps, world, dev) / steps
    total_elems = wl.elements if strong else world * wl.elements
    my_elems = wl.elements
    if strong:
        r0, r1 = _shard_rows(rows0, shard)
        my_elems = (r1 - r0) * (wl.elements // rows0)
    res = {"workload": spec.name, "value": round(total_elems / (ms_per_step / 1e3), 1),
           "ms_per_step": round(ms_per_step, 4), "elements": total_elems,
           "elements_per_gpu": my_elems, "model": "-".join(map(str, spec.dims)),
           "precision": spec.precision, "directives": [spec.in_functor, spec.out_functor],
           "l2": "flushed between steps (512 MiB write)" if flush is not None else "inputs larger than L2",
           "gpu_launches": launches, "steps": steps, "wall_s": round(t_wall, 3),
           "roofline": roofline(spec, my_elems, k_ms, pk, pk_src, fp32_peak)}
    if clk:
        res["clocks"] = clk.summary()

    if rank == 0 and not args.no_parity:
        _, _, _, to = wl.functors()
        out_host = wl.buffers[to.array].to_numpy()
        n = rows0 if name in ("options", "options_bf16", "miniweather", "miniweather_bf16") \
            else min(rows0, CPU_SAMPLE[name])
        if strong:
            n = min(n, _shard_rows(rows0, shard)[1])
        res["parity"] = parity(wl, out_host, n)

    if not args.no_e2e:
        res["e2e"] = e2e(wl, args, rank, world, dev, mdir, shard)
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline(name, wl.elements)
    del rt, wl
    torch.cuda.empty_cache()
    return res


def e2e(wl, args, rank, world, dev, mdir, shard):
    """The same metric through the public API with pinned host arrays: every
    step copies the inputs host->device and the outputs device->host."""
    import torch
    import paper_2407_18352_b200 as sm
    from paper_2407_18352_b200 import workloads
    mw = wl.spec.name.startswith("miniweather")
    hw = workloads.make(wl.spec.name, wl.elements if not mw else None, seed_offset=0 if shard else rank)
    if mw and wl.elements != wl.spec.elements:
        hw = workloads.make(wl.spec.name, wl.elements, seed_offset=0 if shard else rank)
    hw.to_device(pinned_host=True)
    rt2 = sm.Runtime(device=dev, shard=shard)
    h2 = rt2.register_region(hw.descriptor(mdir, name=wl.spec.name + "_host"))
    rt2.invoke_region(h2)
    torch.cuda.synchronize()
    barrier(world)
    e2e_steps = max(1, min(args.steps, 5))
    b0 = (rt2._staging.h2d_bytes, rt2._staging.d2h_bytes)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        rt2.invoke_region(h2)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, dev) / e2e_steps
    # bytes the runtime actually moved per step (whole arrays, row ranges or
    # window boxes), counted by its staging layer; + the 4-B status word
    h2d = (rt2._staging.h2d_bytes - b0[0]) // e2e_steps
    d2h = (rt2._staging.d2h_bytes - b0[1]) // e2e_steps + 4
    total = hw.elements if shard else world * hw.elements
    out = {"value": round(total / e2e_s, 1), "unit": "elements/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": round(e2e_s * 1e3, 3), "steps": e2e_steps,
           "path": "Runtime.invoke_region on pinned host ArrayBuffers (chunked H2D/kernel/D2H overlap"
                   " where the plan allows)"}
    del rt2, hw
    return out


def measure_halo(args, rank, world, local, dev, headline, pk, pk_src, fp32_peak, tmp):
    """C5 sharded across ranks: row slabs of the global grid, one grouped
    halo exchange (NCCL) + the ml(infer) region per step (halo.py,
    SURVEY.md section 8(e))."""
    import torch
    import paper_2407_18352_b200 as sm
    from paper_2407_18352_b200 import _native, halo, workloads
    wl = workloads.make("miniweather")
    spec = wl.spec
    mdir = os.path.join(tmp, "miniweather")
    sm.save_model(wl.model, mdir)
    state = wl.arrays["state"]
    slab = halo.Slab.from_global(state, world, rank, dev)
    rt = sm.Runtime(device=dev)
    stepper = halo.SlabStepper(slab, mdir, runtime=rt, exchange=halo.HaloExchange())
    for _ in range(args.warmup):
        stepper.step()
    torch.cuda.synchronize()
    steps = args.steps if headline else min(args.steps, 10)
    launches0 = _native.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    ev = []
    t_wall = time.perf_counter()
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        stepper.step()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    launches = _native.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms_per_step = max_over_ranks(ms, world, dev) / steps
    rt.time_kernels = True
    rt.kernel_events.clear()
    for _ in range(steps):
        stepper.step()
    torch.cuda.synchronize()
    rt.time_kernels = False
    k_ms = statistics.mean(rt.kernel_times())
    my_elems = slab.rows * (state.shape[2] - 2)
    res = {"workload": spec.name, "value": round(wl.elements / (ms_per_step / 1e3), 1),
           "ms_per_step": round(ms_per_step, 4), "elements": wl.elements, "elements_per_gpu": my_elems,
           "model": "-".join(map(str, spec.dims)), "precision": spec.precision,
           "directives": [halo.HALO_FUNCTOR, halo.PTS_FUNCTOR], "scaling": "strong",
           "parallelism": f"row slabs x{world}, grouped NCCL halo exchange (+-1 row) per step",
           "l2": "slab state resident (step = exchange + region)", "gpu_launches": launches,
           "steps": steps, "wall_s": round(t_wall, 3),
           "roofline": roofline(spec, my_elems, k_ms, pk, pk_src, fp32_peak)}
    if not args.no_parity:
        # one step from a fresh copy of the initial field on every rank (the
        # exchange is collective); rank 0's slab interior vs the unsharded oracle
        from oracle import oracle
        fresh = halo.Slab.from_global(state, world, rank, dev)
        st2 = halo.SlabStepper(fresh, mdir, runtime=rt, exchange=halo.HaloExchange(), name="mw_parity")
        st2.step()
    if rank == 0 and not args.no_parity:
        got = st2.interior()
        fi, fo, ti, to = wl.functors()
        want = state.copy()
        oracle.region([(fi, ti, state.reshape(-1), state.shape, _strides(state))],
                      [(fo, to, want.reshape(-1), want.shape, _strides(want))], wl.layers)
        ref = want[:, fresh.g0:fresh.g1, :]
        res["parity"] = {"vs": "CPU oracle region over the global grid (one step, rank 0's slab)",
                         "rows_checked": int(fresh.rows), "bitwise": bool(np.array_equal(got, ref)),
                         "max_abs": float(np.abs(got.astype(np.float64) - ref).max()),
                         "tolerance": "bitwise (fp32-exact path)"}
        res["parity"]["pass"] = res["parity"]["bitwise"]
    barrier(world)
    del stepper, rt
    torch.cuda.empty_cache()
    return res


def run_ours(args, rank, world, local):
    import torch
    from paper_2407_18352_b200 import _native

    _native.lib()
    dev = torch.device("cuda", local)
    pk, pk_src = peaks()
    fp32 = {m: _native.fp32_peak(m) for m in (0, 1, 2)}
    tmp = tempfile.mkdtemp(prefix="smlrt_bench_")
    names = [args.config] + ([c for c in ALL_CONFIGS if c != args.config] if not args.no_per_config else [])
    results = {}
    for name in names:
        results[name] = measure(name, args, rank, world, local, dev, name == args.config, pk, pk_src, fp32[2], tmp)
    head = results[args.config]
    spec_dtype = "bf16" if head["precision"] == "bf16" else "f32"
    scaling = head.get("scaling", "strong" if (args.scaling == "strong" and world > 1) else "weak")
    line = {
        "metric": METRIC, "value": head["value"], "unit": "elements/s", "n_gpus": world,
        "steps": head["steps"], "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": spec_dtype, "data": "synthetic (seeded uniform/bump arrays, random-init weights)",
        "config": {"workload": head["workload"], "elements": head["elements"],
                   "elements_per_gpu": head["elements_per_gpu"], "model": head["model"],
                   "precision": head["precision"], "directives": head["directives"],
                   "parallelism": head.get("parallelism", f"dp{world} ({scaling} sweep shards, no collective)"),
                   "l2": head["l2"]},
        "roofline": head["roofline"], "e2e": head.get("e2e"), "cpu_baseline": head.get("cpu_baseline"),
        "parity": head.get("parity"),
        "gpu_launches": head["gpu_launches"], "clocks": head.get("clocks"), "wall_s": head["wall_s"],
        "fp32_peak_tflops": {"ffma": round(fp32[0] / 1e12, 2), "fmul_fadd": round(fp32[1] / 1e12, 2),
                             "packed_mul_fma1": round(fp32[2] / 1e12, 2)},
        "per_config": {k: {kk: v[kk] for kk in ("value", "ms_per_step", "elements", "elements_per_gpu",
                                                 "model", "precision", "roofline", "e2e", "parity",
                                                 "cpu_baseline", "gpu_launches", "scaling")
                           if kk in v} for k, v in results.items()},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """The reference's CPU path (numpy restatement, all host cores) on the
    headline config; under torchrun only rank 0 runs it."""
    if rank != 0:
        return
    from paper_2407_18352_b200 import workloads
    procs = len(os.sched_getaffinity(0))
    spec = workloads.CONFIGS[args.config]
    ref = CpuReference(args.config, procs)
    for _ in range(args.warmup):
        ref.run()
    vals, walls = [], []
    for _ in range(args.steps):
        v, n, wall = ref.run()
        vals.append(v)
        walls.append(wall)
    ref.close()
    value = statistics.median(vals)
    sample = (f"{n} of {spec.elements} elements per step (first sweep rows), numpy restatement of the"
              f" reference _run_surrogate path (oracle/oracle.py) in {procs} forked processes"
              " (fork and data generation excluded)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(walls), 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": spec.name, "elements": spec.elements, "model": "-".join(map(str, spec.dims)),
                   "precision": "fp32 (reference numpy path)", "directives": [spec.in_functor, spec.out_functor]},
        "cpu_baseline": {"value": round(value, 1), "unit": "elements/s", "cores": procs, "kind": "port",
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 1), "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def launcher_selftest(args):
    """CPU check of the multi-rank plumbing (gloo): rendezvous, each rank's
    strong-scaling row block, max-over-ranks timing, one line from rank 0."""
    from paper_2407_18352_b200 import workloads
    from paper_2407_18352_b200.runtime import _shard_rows
    rank, world, _ = dist_setup("gloo")
    spec = workloads.CONFIGS[args.config]
    rows = spec.elements
    r0, r1 = _shard_rows(rows, (rank, world))
    import torch
    import torch.distributed as dist
    t = torch.tensor([r0, r1], dtype=torch.int64)
    got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, t)
    ms = max_over_ranks(float(rank + 1), world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "ms_per_step": ms,
                          "shards": [g.tolist() for g in got], "rows": rows}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=ALL_CONFIGS)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--elements", type=int, default=None, help="override the headline sweep size (testing)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-per-config", action="store_true", help="headline config only")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--launcher-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if args.launcher_selftest:
        launcher_selftest(args)
        return
    if args.impl == "reference":
        run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = dist_setup()
    run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
