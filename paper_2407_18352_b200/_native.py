"""ctypes binding of libsmlrt_b200.so (the C-ABI in include/smlrt_b200.h).

This is the only module that touches the native library.  It loads the
in-tree shared object built by `__graft_entry__.build()`; if the library is
missing, every data-path call raises immediately -- there is no Python or CPU
fallback for the region path.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Sequence

from .errors import from_status

MAX_SWEEP = 6
MAX_FEAT = 6
LIB_PATH = Path(__file__).resolve().parent / "libsmlrt_b200.so"

TO, FROM = 0, 1
FP32_EXACT, BF16 = 0, 1
COMMIT_FUSED, COMMIT_CHECKED, FORCE_UNFUSED, SYNC_STATUS = 0, 1, 2, 4
ACT = {"identity": 0, "relu": 1, "tanh": 2}


class View(C.Structure):
    _fields_ = [
        ("array", C.c_int32),
        ("n_feat", C.c_int32),
        ("base", C.c_int64),
        ("sweep_stride", C.c_int64 * MAX_SWEEP),
        ("feat_count", C.c_int64 * MAX_FEAT),
        ("feat_stride", C.c_int64 * MAX_FEAT),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int64),
        ("n_cols", C.c_int32),
        ("n_views", C.c_int32),
        ("n_arrays", C.c_int32),
        ("uniform", C.c_int32),
        ("dense_rows", C.c_int32),
        ("injective", C.c_int32),
        ("row_pitch", C.c_int64),
    ]


class Layer(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("in_", C.c_int32),
        ("out", C.c_int32),
        ("activation", C.c_int32),
        ("kernel", C.c_int32),
        ("stride", C.c_int32),
        ("in_channels", C.c_int32),
        ("in_h", C.c_int32),
        ("in_w", C.c_int32),
        ("weights", C.c_void_p),
        ("bias", C.c_void_p),
    ]


KIND = {"dense": 0, "conv2d": 1, "maxpool2d": 2}


_P = C.c_void_p
_I = C.c_int
_I32 = C.c_int32
_I64 = C.c_int64

# name -> (restype, argtypes); every symbol include/smlrt_b200.h declares
SIGNATURES = {
    "smlrt_version": (C.c_char_p, []),
    "smlrt_last_error": (C.c_char_p, []),
    "smlrt_launch_count": (C.c_ulonglong, []),
    "smlrt_plan_create": (_I, [C.POINTER(View), _I, _I, C.POINTER(_I64), _I, C.POINTER(_I64), _I,
                               C.POINTER(_P)]),
    "smlrt_plan_info": (_I, [_P, C.POINTER(PlanInfo)]),
    "smlrt_plan_row_ranges": (_I, [_P, _I64, _I64, C.POINTER(_I64), _I32, C.POINTER(_I32), C.POINTER(_I32)]),
    "smlrt_plan_destroy": (_I, [_P]),
    "smlrt_model_upload": (_I, [C.POINTER(Layer), _I, _I, _I, C.POINTER(_P)]),
    "smlrt_model_free": (_I, [_P]),
    "smlrt_model_path": (_I, [_P, _I32, C.POINTER(_I32)]),
    "smlrt_gather": (_I, [_P, C.POINTER(_P), C.POINTER(_I32), _P, _I32, _I64, _I64, _P]),
    "smlrt_scatter": (_I, [_P, _P, _I32, C.POINTER(_P), C.POINTER(_I32), _I64, _I64, _P]),
    "smlrt_infer": (_I, [_P, _P, _I32, _I64, _P, _I32, _P, _P]),
    "smlrt_region_workspace": (_I, [_P, _P, _P, _I64, _I32, C.POINTER(C.c_size_t)]),
    "smlrt_region_infer": (_I, [_P, C.POINTER(_P), C.POINTER(_I32), _P, C.POINTER(_P),
                                C.POINTER(_I32), _P, _I64, _I64, _I32, _P, _P, _P]),
    "smlrt_region_prepare": (_I, [_P, C.POINTER(_P), C.POINTER(_I32), _P, C.POINTER(_P), C.POINTER(_I32), _P,
                                  _I64, _I64, _I32, _P, _I32, C.POINTER(_P)]),
    "smlrt_region_run": (_I, [_P, _P]),
    "smlrt_region_run_timed": (_I, [_P, _P, C.POINTER(C.c_float)]),
    "smlrt_region_graphed": (_I, [_P, C.POINTER(_I32)]),
    "smlrt_region_release": (_I, [_P]),
    "smlrt_collect_async": (_I, [_P, C.c_size_t, _P, _P, _P]),
    "smlrt_collect_wait": (_I, [_P]),
    "smlrt_copy_box_async": (_I, [_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _P]),
    "smlrt_tc_selftest": (_I, [_I, _I, _P, _P, _P]),
    "smlrt_tc_selftest_ts": (_I, [_I, _I, _P, _P, _P]),
    "smlrt_fp32_peak": (_I, [_I32, C.POINTER(C.c_double)]),
}

_lib = None
_load_error = None


def _load():
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise _load_error
    path = os.environ.get("SMLRT_B200_LIB", str(LIB_PATH))
    try:
        lib = C.CDLL(path)
    except OSError as e:
        _load_error = RuntimeError(
            f"libsmlrt_b200.so not loadable ({e}); run `python -c 'import __graft_entry__ as g;"
            " g.build()'` -- the region path has no CPU fallback")
        raise _load_error from None
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _load()


def loaded() -> bool:
    return _lib is not None


def _check(rc: int):
    if rc != 0:
        msg = _lib.smlrt_last_error().decode(errors="replace")
        raise from_status(rc, msg)


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


def version() -> str:
    return lib().smlrt_version().decode()


def launch_count() -> int:
    """Kernels this library has launched since load (bench instrumentation)."""
    return int(lib().smlrt_launch_count())


# ------------------------------------------------------------------ plans --

def plan_create(flat_views, sweep: Sequence[int], direction: str, array_numel: Sequence[int]):
    """flat_views: [(array_index, MemoryView)] -> (handle, n_rows, n_cols)."""
    L = lib()
    n_sweep = len(sweep)
    if n_sweep > MAX_SWEEP:
        from .errors import ArityMismatchError
        raise ArityMismatchError(f"{n_sweep} sweep axes exceed the native limit of {MAX_SWEEP}")
    vs = (View * len(flat_views))()
    for i, (a, v) in enumerate(flat_views):
        feat_shape = v.shape[v.n_sweep:]
        feat_strides = v.strides[v.n_sweep:]
        if len(feat_shape) > MAX_FEAT:
            raise ValueError(f"view with {len(feat_shape)} feature axes exceeds {MAX_FEAT}")
        vs[i].array = a
        vs[i].n_feat = len(feat_shape)
        vs[i].base = v.base_offset
        for k in range(n_sweep):
            vs[i].sweep_stride[k] = v.strides[k]
        for k, (n, s) in enumerate(zip(feat_shape, feat_strides)):
            vs[i].feat_count[k] = n
            vs[i].feat_stride[k] = s
    h = C.c_void_p()
    _check(L.smlrt_plan_create(vs, len(flat_views), n_sweep, _arr(_I64, sweep),
                               TO if direction == "to" else FROM,
                               _arr(_I64, array_numel), len(array_numel), C.byref(h)))
    info = PlanInfo()
    _check(L.smlrt_plan_info(h, C.byref(info)))
    return h, int(info.n_rows), int(info.n_cols)


def plan_info(handle) -> dict:
    info = PlanInfo()
    _check(lib().smlrt_plan_info(handle, C.byref(info)))
    return {k: getattr(info, k) for k, _ in PlanInfo._fields_}


def plan_row_ranges(handle, r0: int, r1: int, max_ranges: int = 16):
    """[(lo, hi), ...] element ranges rows [r0, r1) touch, and whether they are
    exact; None when the plan is not uniform 1-D or needs > max_ranges."""
    buf = (_I64 * (2 * max_ranges))()
    n, exact = _I32(0), _I32(0)
    rc = lib().smlrt_plan_row_ranges(handle, r0, r1, buf, max_ranges, C.byref(n), C.byref(exact))
    if rc == 10:  # SMLRT_E_UNSUPPORTED
        return None
    _check(rc)
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)], bool(exact.value)


def plan_destroy(handle):
    if _lib is not None and handle:
        _lib.smlrt_plan_destroy(handle)


# ----------------------------------------------------------------- models --

def model_upload(layers, precision: int, device: int):
    """layers: [(kind, W, b, act, params)] from Model.native_layers() (or the
    legacy dense triples (W, b, act))."""
    L = lib()
    arr = (Layer * len(layers))()
    keep = []
    width = None
    for i, spec in enumerate(layers):
        if len(spec) == 3:
            spec = ("dense", spec[0], spec[1], spec[2], {})
        kind, w, b, act, prm = spec
        arr[i].kind = KIND[kind]
        arr[i].activation = ACT[act]
        if kind == "dense":
            arr[i].in_, arr[i].out = w.shape[1], w.shape[0]
        else:
            c, h, wd, k = prm["in_channels"], prm["in_h"], prm["in_w"], prm["kernel"]
            arr[i].kernel, arr[i].stride = k, prm["stride"]
            arr[i].in_channels, arr[i].in_h, arr[i].in_w = c, h, wd
            oc = w.shape[0] if kind == "conv2d" else c
            arr[i].in_, arr[i].out = c * h * wd, oc * (h // k) * (wd // k)
        if w is not None:
            keep += [w, b]
            arr[i].weights = w.ctypes.data
            arr[i].bias = b.ctypes.data
    h = C.c_void_p()
    _check(L.smlrt_model_upload(arr, len(layers), precision, device, C.byref(h)))
    return h


def model_free(handle):
    if _lib is not None and handle:
        _lib.smlrt_model_free(handle)


def model_path(handle, n_in_cols: int = 0) -> int:
    p = C.c_int32()
    _check(lib().smlrt_model_path(handle, n_in_cols, C.byref(p)))
    return int(p.value)


# ------------------------------------------------------------ data paths --

def gather(plan, ptrs, dtypes, out_ptr, out_dtype, r0, r1, stream):
    _check(lib().smlrt_gather(plan, _arr(_P, ptrs), _arr(_I32, dtypes), out_ptr, out_dtype,
                              r0, r1, stream))


def scatter(plan, in_ptr, in_dtype, ptrs, dtypes, r0, r1, stream):
    _check(lib().smlrt_scatter(plan, in_ptr, in_dtype, _arr(_P, ptrs), _arr(_I32, dtypes),
                               r0, r1, stream))


def infer(model, x_ptr, x_dtype, rows, y_ptr, y_dtype, stream, status_ptr):
    _check(lib().smlrt_infer(model, x_ptr, x_dtype, rows, y_ptr, y_dtype, stream, status_ptr))


def region_infer(pin, in_ptrs, in_dts, pout, out_ptrs, out_dts, model, r0, r1, flags,
                 workspace, stream, status_ptr):
    _check(lib().smlrt_region_infer(pin, _arr(_P, in_ptrs), _arr(_I32, in_dts), pout,
                                    _arr(_P, out_ptrs), _arr(_I32, out_dts), model, r0, r1,
                                    flags, workspace, stream, status_ptr))


class PreparedRegion:
    """A native prepared region (smlrt_region_prepare): the steady-state
    invoke_region of a device-resident region, replayed as one CUDA graph.
    `keep` holds the objects owning the plan/model handles alive."""

    def __init__(self, pin, in_ptrs, in_dts, pout, out_ptrs, out_dts, model, r0, r1, flags, status_ptr,
                 *keep, graph: bool = True):
        self._keep = keep
        self.handle = None
        h = _P()
        _check(lib().smlrt_region_prepare(pin, _arr(_P, in_ptrs), _arr(_I32, in_dts), pout, _arr(_P, out_ptrs),
                                          _arr(_I32, out_dts), model, r0, r1, flags, status_ptr, int(graph),
                                          C.byref(h)))
        self.handle = h
        self._run = lib().smlrt_region_run

    @property
    def graphed(self) -> bool:
        g = _I32(0)
        _check(lib().smlrt_region_graphed(self.handle, C.byref(g)))
        return bool(g.value)

    def __call__(self, stream, timing: list | None = None) -> int:
        """1 if the output was non-finite, else 0 (other errors raise).
        `timing`: a list that receives the launches' device time in ms."""
        if timing is not None:
            ms = C.c_float(0.0)
            rc = lib().smlrt_region_run_timed(self.handle, stream, C.byref(ms))
            timing.append(float(ms.value))
        else:
            rc = self._run(self.handle, stream)
        if rc == 0:
            return 0
        if rc == 7:  # SMLRT_E_NONFINITE
            return 1
        _check(rc)

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be gone
            if h is not None and _lib is not None:
                _lib.smlrt_region_release(h)
                self.handle = None
        except Exception:
            pass


def prepare_region(pin, in_ptrs, in_dts, pout, out_ptrs, out_dts, model, r0, r1, flags, status_ptr, *keep,
                   graph: bool = True) -> PreparedRegion:
    return PreparedRegion(pin, in_ptrs, in_dts, pout, out_ptrs, out_dts, model, r0, r1, flags, status_ptr,
                          *keep, graph=graph)


def region_workspace(pin, pout, model, rows, flags) -> int:
    n = C.c_size_t()
    _check(lib().smlrt_region_workspace(pin, pout, model, rows, flags, C.byref(n)))
    return int(n.value)


def collect_async(dev_ptr, nbytes, host_ptr, side_stream, after_event):
    _check(lib().smlrt_collect_async(dev_ptr, nbytes, host_ptr, side_stream, after_event))


def collect_wait(side_stream):
    _check(lib().smlrt_collect_wait(side_stream))


def copy_box_async(dst_ptr, src_ptr, elem_size, box, direction, stream):
    """box = (offset, width, height, depth, pitch, slice) in elements."""
    off, w, h, d, pitch, sl = box
    _check(lib().smlrt_copy_box_async(dst_ptr, src_ptr, elem_size, off, w, h, d, pitch, sl, direction, stream))


def tc_selftest(A, B, tmem_a: bool = False):
    """D = A @ B.T on one CTA through tcgen05 (A [128,K], B [N,K] float32);
    tmem_a stages A in tensor memory (TS form) instead of shared memory."""
    import numpy as np
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    D = np.zeros((128, B.shape[0]), np.float32)
    fn = lib().smlrt_tc_selftest_ts if tmem_a else lib().smlrt_tc_selftest
    _check(fn(A.shape[1], B.shape[0], A.ctypes.data, B.ctypes.data, D.ctypes.data))
    return D


def fp32_peak(mode: int) -> float:
    """Measured FP32 flop/s of the current device: 0 FFMA, 1 FMUL+FADD,
    2 packed f32x2 mul then fma(p, 1, acc) (the exact kernels' mix)."""
    v = C.c_double()
    _check(lib().smlrt_fp32_peak(mode, C.byref(v)))
    return float(v.value)
