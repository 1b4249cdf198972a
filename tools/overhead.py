"""Fixed per-invoke cost of Runtime.invoke_region and the price of
commit="checked", measured on the GPU.

    python tools/overhead.py   -> one JSON line per measurement
"""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_18352_b200 as sm  # noqa: E402
from paper_2407_18352_b200 import workloads  # noqa: E402


def timed(rt, h, n=200):
    for _ in range(10):
        rt.invoke_region(h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        rt.invoke_region(h)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    torch.cuda.set_device(0)
    tmp = tempfile.mkdtemp()
    # fixed cost: a 1-row options region (the kernel itself is ~3 us)
    for rows in (1, 1000):
        wl = workloads.make("options", rows)
        wl.to_device()
        sm.save_model(wl.model, os.path.join(tmp, "o"))
        for graphs in (True, False):
            rt = sm.Runtime(graphs=graphs)
            h = rt.register_region(wl.descriptor(os.path.join(tmp, "o")))
            us = timed(rt, h)
            # the native prepared call alone (no Python dispatch above it)
            call = rt._fast["options"][1]
            stream = torch.cuda.current_stream().cuda_stream
            t0 = time.perf_counter()
            for _ in range(200):
                call(stream)
            native_us = (time.perf_counter() - t0) / 200 * 1e6
            print(json.dumps({"what": "invoke_region wall", "rows": rows, "graphs": graphs,
                              "us_per_call": round(us, 1), "native_prepared_us": round(native_us, 1)}), flush=True)
            if rows == 1 and graphs and os.environ.get("PROFILE"):
                import cProfile
                import pstats
                pr = cProfile.Profile()
                pr.enable()
                for _ in range(200):
                    rt.invoke_region(h)
                pr.disable()
                pstats.Stats(pr).sort_stats("tottime").print_stats(12)
            del rt
    if os.environ.get("ONLY_FIXED"):
        return
    # checked vs fused commit per config (step time, CUDA events)
    for name in ("options", "bonds", "minibude", "particlefilter", "miniweather"):
        wl = workloads.make(name)
        wl.to_device()
        sm.save_model(wl.model, os.path.join(tmp, name))
        res = {}
        for commit in ("fused", "checked"):
            rt = sm.Runtime(commit=commit)
            h = rt.register_region(wl.descriptor(os.path.join(tmp, name)))
            for _ in range(3):
                rt.invoke_region(h)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps = 5 if name == "minibude" else 20
            e0.record()
            for _ in range(steps):
                rt.invoke_region(h)
            e1.record()
            torch.cuda.synchronize()
            res[commit] = round(e0.elapsed_time(e1) / steps, 4)
            del rt
        print(json.dumps({"what": "commit cost (ms per step)", "config": name, **res,
                          "checked_over_fused": round(res["checked"] / res["fused"], 4)}), flush=True)
        del wl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
