"""A/B of the Runtime's chunked host path vs whole-array staging (e2e ms per call)."""
import sys
import tempfile
import time

import torch

import paper_2407_18352_b200 as sm
from paper_2407_18352_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "options"
wl = workloads.make(cfg)
wl.to_device(pinned_host=True)
with tempfile.TemporaryDirectory() as d:
    sm.save_model(wl.model, d + "/m")
    for mode in ("chunked", "whole", "chunked", "whole"):
        with sm.Runtime() as rt:
            if mode == "whole":
                rt.STREAM_MIN_BYTES = 1 << 62
            h = rt.register_region(wl.descriptor(d + "/m"))
            rt.invoke_region(h)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                rt.invoke_region(h)
            torch.cuda.synchronize()
            print(cfg, mode, f"{(time.perf_counter() - t0) / 10 * 1e3:.3f} ms", "chunked" if rt._side else "whole")
