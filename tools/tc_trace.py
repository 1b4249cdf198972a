"""Pipeline trace of the fused tcgen05 bonds kernel (debug build only).

    make -C paper_2407_18352_b200/csrc trace
    SMLRT_B200_LIB=paper_2407_18352_b200/libsmlrt_b200_trace.so python tools/tc_trace.py

Prints, for CTA 0, per-tile clock64 deltas of each role's events relative to
the L1 MMA issue of that tile, and the steady-state period."""
import ctypes as C
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_18352_b200 as sm  # noqa: E402
from paper_2407_18352_b200 import _native, workloads  # noqa: E402

EV = {0: "L1 issue", 9: "mma sees XFULL", 1: "L2 issue", 11: "mma sees A2FULL", 2: "epi1 L1FULL", 3: "A2EMPTY|A2F q3p1",
      4: "epi1 drained|A2F q1p1", 5: "epi1 A2FULL", 10: "A2FULL q2p0", 6: "epi2 L2FULL", 7: "epi2 done", 8: "loader XFULL",
      12: "epi1 L1bFULL", 13: "L1 committed", 14: "L1a issued", 15: "L2b issue"}
COLS = tuple(int(c) for c in os.environ.get("TRACE_COLS", "8,9,0,2,3,4,5,11,1,6,7").split(","))

n = int(os.environ.get("N", 148 * 128 * 64 * 2))
wl = workloads.make("bonds", n)
wl.to_device()
with tempfile.TemporaryDirectory() as d:
    sm.save_model(wl.model, d + "/m")
    with sm.Runtime() as rt:
        h = rt.register_region(wl.descriptor(d + "/m"))
        rt.invoke_region(h)
        rt.invoke_region(h)
import torch  # noqa: E402
torch.cuda.synchronize()
lib = _native.lib()
TT = 1024
buf = (C.c_ulonglong * (2 * TT * 16))()
assert lib.smlrt_tc_trace_dump(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, TT, 16).astype(np.int64)
for cta in (0, 1):
    tr = t[cta]
    base = tr[0, 0] if tr[0, 0] else tr[0, 2]
    print(f"== CTA {cta} (cycles from tile-0 L1 issue)")
    print("tile " + " ".join(f"{EV[e][:13]:>13}" for e in COLS))
    for it in range(0, 24):
        print(f"{it:4d} " + " ".join(f"{(tr[it, e] - base) if tr[it, e] else -1:13d}" for e in COLS))
    for lo, hi in ((8, 60), (200, 260), (600, 660), (820, 880)):
        for e in (0, 1, 7):
            col = tr[lo:hi, e]
            col = col[col > 0]
            if len(col) > 2:
                print(f"tiles {lo}-{hi} period({EV[e]}): {np.median(np.diff(col)):.0f} cycles")
        if tr[hi, 15] > tr[lo, 15] > 0:
            print(f"tiles {lo}-{hi}: SM clock {(tr[hi, 0] - tr[lo, 0]) / (tr[hi, 15] - tr[lo, 15]) * 1e3:.0f} MHz, "
                  f"{(tr[hi, 15] - tr[lo, 15]) / (hi - lo):.0f} ns per tile")
