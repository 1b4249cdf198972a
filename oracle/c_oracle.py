"""ctypes wrapper of oracle/build/liboracle.so (ORACLE -- test infrastructure).

`mlp_f32` runs the C restatement of models.py:188-224 over row blocks on a
thread pool (ctypes drops the GIL for the duration of each call)."""

from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "build" / "liboracle.so"
_ACT = {"identity": 0, "relu": 1, "tanh": 2}
_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(_LIB))
        _lib.oracle_mlp_f32.restype = C.c_int
        _lib.oracle_mlp_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def available() -> bool:
    return _LIB.exists()


def mlp_f32(layers, x, threads: int | None = None):
    """layers: [(W [out,in] f32, b [out] f32, act)] -> (y f32 [rows, G], finite)."""
    L = lib()
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows = x.shape[0]
    ws = [np.ascontiguousarray(w, np.float32) for w, _, _ in layers]
    bs = [np.ascontiguousarray(b, np.float32) for _, b, _ in layers]
    dims = np.array([x.shape[1]] + [w.shape[0] for w in ws], dtype=np.int32)
    acts = np.array([_ACT[a] for _, _, a in layers], dtype=np.int32)
    wp = (C.c_void_p * len(ws))(*[w.ctypes.data for w in ws])
    bp = (C.c_void_p * len(bs))(*[b.ctypes.data for b in bs])
    y = np.empty((rows, int(dims[-1])), dtype=np.float32)
    threads = threads or len(os.sched_getaffinity(0))
    step = max(1, -(-rows // threads))

    def run(r0):
        n = min(step, rows - r0)
        return L.oracle_mlp_f32(x[r0:].ctypes.data, n, len(ws), dims.ctypes.data,
                                acts.ctypes.data, wp, bp, y[r0:].ctypes.data)

    with ThreadPoolExecutor(threads) as ex:
        bad = list(ex.map(run, range(0, rows, step)))
    return y, not any(bad)
