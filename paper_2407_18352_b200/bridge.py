"""Application memory <-> dense tensors, device-resident.

Geometry (steps 1-3 of the reference's Fig. 4 pipeline) is integer
bookkeeping and stays on the host: `extract_symbolic_shape`,
`resolve_symbolic_shape` and `wrap_tensors` reproduce
`/root/reference/pkg/src/smlrt/bridge.py:190-344` result for result (same
descriptors, same `MemoryView` base/shape/strides, same eager bounds errors).

The copying steps do not run here.  `wrap_tensors` output is flattened into a
*plan* (one `smlrt_view_t` per RHS view, `include/smlrt_b200.h`) that the
native library validates once (flat bounds, and for the reverse direction
injectivity) and caches; `concretize_to` / `scatter_from` / `gather_batch`
then launch the sm_100a gather / scatter kernels through the C-ABI.  There is
no host fallback: an `ArrayBuffer` must live on a CUDA device, and every data
movement goes through `libsmlrt_b200.so`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native
from .directives import FunctorDecl, MapTarget, SliceDim
from .errors import (
    ArityMismatchError,
    FeatureMismatchError,
    NonInjectiveScatterError,
    OutOfBoundsError,
    ShapeMismatchError,
)

__all__ = [
    "ArrayBuffer", "Tensor", "MemoryView", "SliceDescriptor", "ResolvedSlice",
    "extract_symbolic_shape", "resolve_symbolic_shape", "wrap_tensors",
    "compose_tensor", "concretize_to", "scatter_from", "gather_batch",
    "expected_tensor_shape", "Plan", "build_plan", "PLAN_CACHE",
]

_TORCH = {"f32": torch.float32, "f64": torch.float64}
_NP = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8")}
DTYPE_CODE = {"f32": 0, "f64": 1}


def dtype_name(dt) -> str:
    if dt in (torch.float32, np.dtype("<f4"), np.float32):
        return "f32"
    if dt in (torch.float64, np.dtype("<f8"), np.float64):
        return "f64"
    raise ValueError(f"unsupported dtype {dt} (expected f32 or f64)")


def np_dtype(name: str) -> np.dtype:
    try:
        return _NP[name]
    except KeyError:
        raise ValueError(f"unsupported dtype {name!r} (expected f32 or f64)") from None


def _default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


# ---------------------------------------------------------------------------
# Memory spaces (bridge.py:76-167)
# ---------------------------------------------------------------------------

class ArrayBuffer:
    """Application array: flat storage + logical shape + element strides.

    `data` is a 1-D torch tensor.  For the region path it lives in HBM; a
    host (CPU) buffer is accepted by the Runtime, which stages it through the
    device (the end-to-end path), but never computed on by the CPU.
    """

    __slots__ = ("data", "shape", "strides", "_version")

    def __init__(self, data, shape: Sequence[int], strides: Sequence[int]):
        if isinstance(data, np.ndarray):
            data = torch.from_numpy(np.ascontiguousarray(data))
        if not isinstance(data, torch.Tensor):
            raise TypeError("ArrayBuffer storage must be a torch tensor or numpy array")
        self.shape = tuple(int(s) for s in shape)
        self.strides = tuple(int(s) for s in strides)
        if data.dim() != 1:
            raise ValueError("ArrayBuffer storage must be flat")
        if not data.is_contiguous():
            raise ValueError("ArrayBuffer storage must be a dense 1-D tensor")
        dtype_name(data.dtype)
        if len(self.shape) != len(self.strides):
            raise ValueError("shape and strides must have equal rank")
        if any(s < 1 for s in self.shape):
            raise ValueError(f"non-positive extent in shape {self.shape}")
        if any(s < 1 for s in self.strides):
            raise ValueError(f"non-positive stride in {self.strides}")
        span = 1 + sum((n - 1) * s for n, s in zip(self.shape, self.strides))
        if span > data.numel():
            raise ValueError(
                f"shape {self.shape} with strides {self.strides} needs {span}"
                f" elements, storage has {data.numel()}")
        self.data = data
        self._version = 0

    # constructors ---------------------------------------------------------
    @classmethod
    def from_torch(cls, t: torch.Tensor) -> "ArrayBuffer":
        """Wrap a contiguous tensor without copying (row-major strides)."""
        if not t.is_contiguous():
            raise ValueError("from_torch needs a contiguous tensor; pass strides explicitly")
        strides = tuple(t.stride()) if t.dim() else ()
        return cls(t.reshape(-1), tuple(t.shape), strides)

    @classmethod
    def from_numpy(cls, arr: np.ndarray, device=None) -> "ArrayBuffer":
        """Upload a host array to HBM (row-major).  Unlike the reference this
        copies: application arrays of the B200 runtime are device-resident."""
        arr = np.ascontiguousarray(arr)
        dt = dtype_name(arr.dtype)
        dev = torch.device(device) if device is not None else _default_device()
        t = torch.from_numpy(arr.reshape(-1).astype(np_dtype(dt), copy=False)).to(dev)
        strides = tuple(s // arr.itemsize for s in arr.strides)
        return cls(t, tuple(arr.shape), strides)

    @classmethod
    def zeros(cls, shape: Sequence[int], dtype: str = "f64", device=None) -> "ArrayBuffer":
        dev = torch.device(device) if device is not None else _default_device()
        n = int(np.prod(shape)) if len(shape) else 1
        t = torch.zeros(n, dtype=_TORCH[dtype], device=dev)
        strides = tuple(int(np.prod(shape[k + 1:])) for k in range(len(shape)))
        return cls(t, tuple(shape), strides)

    # accessors ---------------------------------------------------------------
    @property
    def dtype(self) -> str:
        return dtype_name(self.data.dtype)

    @property
    def device(self) -> torch.device:
        return self.data.device

    @property
    def is_device(self) -> bool:
        return self.data.is_cuda

    def view(self) -> torch.Tensor:
        """Strided torch view (no copy) shaped like the logical array."""
        return torch.as_strided(self.data, self.shape, self.strides)

    def to_numpy(self) -> np.ndarray:
        """Host copy of the logical array."""
        return self.view().detach().cpu().numpy()

    def __eq__(self, other):
        return (isinstance(other, ArrayBuffer) and self.data is other.data
                and self.shape == other.shape and self.strides == other.strides)

    def __hash__(self):
        return id(self.data)

    def __repr__(self):
        return f"ArrayBuffer({self.dtype}, shape={self.shape}, strides={self.strides}, {self.device})"


class Tensor:
    """Dense row-major tensor (torch storage, normally in HBM)."""

    __slots__ = ("data",)

    def __init__(self, data):
        if isinstance(data, np.ndarray):
            data = torch.from_numpy(np.ascontiguousarray(data))
        dtype_name(data.dtype)
        self.data = data.contiguous()

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.data.shape)

    @property
    def dtype(self) -> str:
        return dtype_name(self.data.dtype)

    def to_numpy(self) -> np.ndarray:
        return self.data.detach().cpu().numpy()


@dataclass(frozen=True)
class MemoryView:
    """Zero-copy strided window: shape (sweep..., feature...), element strides."""

    source: ArrayBuffer
    base_offset: int
    shape: tuple[int, ...]
    strides: tuple[int, ...]
    n_sweep: int

    def as_torch(self) -> torch.Tensor:
        return torch.as_strided(self.source.data, self.shape, self.strides, self.base_offset)


# ---------------------------------------------------------------------------
# Step 1: symbolic shape extraction (bridge.py:174-224)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SliceDescriptor:
    offset_per_dim: tuple[int, ...]
    elem_count_per_dim: tuple[int, ...]
    step_per_dim: tuple[int, ...]
    symbol_per_dim: tuple[Optional[int], ...]


def _describe(dim: SliceDim, sym_index: dict[str, int]):
    """(offset, count, step, sweep axis | None) of one RHS slice dim."""
    axis = sym_index[dim.symbol] if dim.symbol is not None else None
    if dim.is_point:
        return dim.start.offset, 1, 1, axis
    if axis is not None:
        n = -(-(dim.stop.offset - dim.start.offset) // dim.step)
        return dim.start.offset, n, dim.step, axis
    return dim.start.offset, dim.const_count(), dim.step, None


def extract_symbolic_shape(functor: FunctorDecl, target: MapTarget) -> list[SliceDescriptor]:
    sym_index = {name: k for k, name in enumerate(functor.symbols)}
    if len(target.slices) != len(sym_index):
        raise ArityMismatchError(
            f"functor {functor.name!r} sweeps {len(sym_index)} symbol(s) but the"
            f" target {target.array!r} supplies {len(target.slices)} slice(s)")
    out = []
    for s in functor.rhs:
        cols = list(zip(*[_describe(d, sym_index) for d in s.dims]))
        out.append(SliceDescriptor(*(tuple(c) for c in cols)))
    return out


# ---------------------------------------------------------------------------
# Step 2: symbolic shape resolution (bridge.py:231-281)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ResolvedSlice:
    descriptor: SliceDescriptor
    start_per_dim: tuple[int, ...]
    stop_per_dim: tuple[int, ...]
    step_per_dim: tuple[int, ...]
    sweep_shape: tuple[int, ...]
    feature_shape: tuple[int, ...]

    @property
    def feature_count(self) -> int:
        return int(np.prod(self.feature_shape))


def resolve_symbolic_shape(descriptors: Sequence[SliceDescriptor],
                           target: MapTarget) -> list[ResolvedSlice]:
    sweep = tuple(s.count for s in target.slices)
    out = []
    for d in descriptors:
        starts, stops, steps = [], [], []
        for off, axis, step, count in zip(d.offset_per_dim, d.symbol_per_dim,
                                          d.step_per_dim, d.elem_count_per_dim):
            if axis is None:
                starts.append(off)
                stops.append(off + (count - 1) * step + 1)
                steps.append(step)
            else:
                t = target.slices[axis]
                starts.append(t.start)
                stops.append(t.stop)
                steps.append(t.step)
        feats = tuple(c for c in d.elem_count_per_dim if c > 1) or (1,)
        out.append(ResolvedSlice(d, tuple(starts), tuple(stops), tuple(steps), sweep, feats))
    return out


# ---------------------------------------------------------------------------
# Step 3: tensor wrapping (bridge.py:288-344)
# ---------------------------------------------------------------------------

def wrap_tensors(resolved: Sequence[ResolvedSlice], array: ArrayBuffer) -> list[MemoryView]:
    views = []
    rank = len(array.shape)
    for r in resolved:
        d = r.descriptor
        if len(d.offset_per_dim) != rank:
            raise ArityMismatchError(
                f"RHS slice addresses {len(d.offset_per_dim)} dim(s), array has {rank}")
        n_sweep = len(r.sweep_shape)
        sweep_strides = [0] * n_sweep
        base = 0
        feat = []
        for k in range(rank):
            astride, extent = array.strides[k], array.shape[k]
            off, count = d.offset_per_dim[k], d.elem_count_per_dim[k]
            step, axis = d.step_per_dim[k], d.symbol_per_dim[k]
            if axis is None:
                first, swept = off, 0
            else:
                first = r.start_per_dim[k] + off
                swept = (r.sweep_shape[axis] - 1) * r.step_per_dim[k]
                sweep_strides[axis] += astride * r.step_per_dim[k]
            last = first + swept + (count - 1) * step
            if first < 0 or last >= extent:
                raise OutOfBoundsError(
                    f"slice sweeps indices {first}..{last} on array dim {k}"
                    f" of extent {extent}")
            base += first * astride
            if count > 1:
                feat.append((count, astride * step))
        fshape = tuple(c for c, _ in feat) or (1,)
        fstrides = tuple(s for _, s in feat) or (1,)
        views.append(MemoryView(array, base, r.sweep_shape + fshape,
                                tuple(sweep_strides) + fstrides, n_sweep))
    return views


def expected_tensor_shape(functor: FunctorDecl, target: MapTarget) -> tuple[int, ...]:
    return tuple(s.count for s in target.slices) + functor.feature_sizes


# ---------------------------------------------------------------------------
# Plans: wrap_tensors output flattened for the native library
# ---------------------------------------------------------------------------

class _NativePlan:
    """Owns one native plan handle; shared by every Plan with the same geometry."""

    __slots__ = ("handle", "n_rows", "n_cols", "__weakref__")

    def __init__(self, handle, n_rows, n_cols):
        self.handle = handle
        self.n_rows = n_rows
        self.n_cols = n_cols

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be gone
            if h is not None and _native.loaded():
                _native.plan_destroy(h)
                self.handle = None
        except Exception:
            pass


class _PlanCache:
    """Process-wide cache of validated native plans, keyed by geometry only
    (per view: array index, base offset, shape, element strides; the sweep,
    the direction and every array's element count).  A native plan holds no
    pointers -- they are passed per call -- so any Runtime, and the library
    entry points `concretize_to` / `scatter_from`, reuse one plan (its bounds
    and injectivity proof included) for every array with that geometry.  The
    closest reference analogue is the realpath-keyed model cache shared by a
    Runtime's regions (`runtime.py:185-197`); bounded LRU."""

    def __init__(self, capacity: int = 512):
        import collections
        import threading
        self.capacity = capacity
        self._d = collections.OrderedDict()
        self._lock = threading.Lock()
        self.hits = 0
        self.misses = 0

    def get(self, key):
        with self._lock:
            hit = self._d.get(key)
            if hit is not None:
                self._d.move_to_end(key)
                self.hits += 1
            return hit

    def put(self, key, plan: _NativePlan):
        with self._lock:
            self.misses += 1
            self._d[key] = plan
            self._d.move_to_end(key)
            while len(self._d) > self.capacity:
                self._d.popitem(last=False)

    def clear(self):
        with self._lock:
            self._d.clear()

    def __len__(self):
        return len(self._d)


PLAN_CACHE = _PlanCache()


class Plan:
    """Validated native plan over one or more maps, bound to its arrays.

    `arrays` lists the distinct ArrayBuffers the views address, in the order
    the native call receives their pointers; `n_cols` is the dense feature
    width; `n_rows` the flattened sweep size.  The native handle comes from
    the process-wide PLAN_CACHE.
    """

    def __init__(self, native, arrays, n_rows, n_cols, sweep, direction, views=()):
        self._native_plan = native
        self.handle = native.handle
        self.views = list(views)  # [(array index, MemoryView)]
        self.arrays = arrays
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.sweep = sweep
        self.direction = direction

    def ptrs_and_dtypes(self):
        return ([a.data.data_ptr() for a in self.arrays],
                [DTYPE_CODE[a.dtype] for a in self.arrays])


def build_plan(view_groups: Sequence[Sequence[MemoryView]], direction: str) -> Plan:
    """Flatten the views of several maps (concatenated on the feature axis,
    in order) into one native plan.  direction: "to" (gather) | "from" (scatter).
    Validation (bounds; injectivity for "from") runs once per geometry."""
    arrays: list[ArrayBuffer] = []
    index: dict[int, int] = {}
    flat = []
    sweep = None
    for views in view_groups:
        for v in views:
            s = v.shape[: v.n_sweep]
            if sweep is None:
                sweep = s
            elif s != sweep:
                raise ShapeMismatchError(f"maps disagree on the sweep shape: {s} vs {sweep}")
            key = id(v.source.data)
            if key not in index:
                index[key] = len(arrays)
                arrays.append(v.source)
            flat.append((index[key], v))
    numel = tuple(a.data.numel() for a in arrays)
    key = (direction, tuple(sweep) if sweep is not None else None, numel,
           tuple((a, v.base_offset, tuple(v.shape), tuple(v.strides), v.n_sweep) for a, v in flat))
    native = PLAN_CACHE.get(key)
    if native is None:
        handle, n_rows, n_cols = _native.plan_create(flat, sweep, direction, list(numel))
        native = _NativePlan(handle, n_rows, n_cols)
        PLAN_CACHE.put(key, native)
    return Plan(native, arrays, native.n_rows, native.n_cols, sweep, direction, flat)


def _views_for(functor: FunctorDecl, target: MapTarget, array: ArrayBuffer):
    return wrap_tensors(resolve_symbolic_shape(extract_symbolic_shape(functor, target), target), array)


def _check_features(views: Sequence[MemoryView], functor: FunctorDecl):
    """compose_tensor's checks (bridge.py:359-372)."""
    sweep = views[0].shape[: views[0].n_sweep]
    dt = views[0].source.dtype
    for v in views:
        if v.shape[: v.n_sweep] != sweep:
            raise ShapeMismatchError("RHS views disagree on the sweep shape")
        if v.source.dtype != dt:
            raise ShapeMismatchError("RHS views disagree on dtype")
    total = sum(int(np.prod(v.shape[v.n_sweep:])) for v in views)
    if total != functor.feature_count:
        raise FeatureMismatchError(
            f"RHS slices supply {total} feature element(s), LHS of"
            f" {functor.name!r} declares {functor.feature_count}")
    return sweep


def _require_device(array: ArrayBuffer):
    if not array.is_device:
        raise ValueError("the B200 bridge operates on device-resident ArrayBuffers"
                         " (ArrayBuffer.from_numpy uploads to HBM)")


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# ---------------------------------------------------------------------------
# Step 4 and the two directions (bridge.py:351-462)
# ---------------------------------------------------------------------------

def compose_tensor(views: Sequence[MemoryView], functor: FunctorDecl) -> Tensor:
    if not views:
        raise ValueError("nothing to compose")
    sweep = _check_features(views, functor)
    for v in views:
        _require_device(v.source)
    plan = build_plan([views], "to")
    dev = views[0].source.device
    out = torch.empty((plan.n_rows, plan.n_cols), dtype=views[0].source.data.dtype, device=dev)
    ptrs, dts = plan.ptrs_and_dtypes()
    _native.gather(plan.handle, ptrs, dts, out.data_ptr(), DTYPE_CODE[views[0].source.dtype],
                   0, plan.n_rows, _stream_ptr(dev))
    return Tensor(out.reshape(tuple(sweep) + functor.feature_sizes))


def concretize_to(functor: FunctorDecl, target: MapTarget, array: ArrayBuffer) -> Tensor:
    """Application memory -> fresh dense tensor in HBM (the array is not written)."""
    return compose_tensor(_views_for(functor, target, array), functor)


def check_scatter_functor(functor: FunctorDecl):
    """scatter_from's functor-level checks, in the reference order (bridge.py:416-427)."""
    for s in functor.rhs:
        for d in s.dims:
            if not d.is_point:
                raise NonInjectiveScatterError(
                    f"RHS range slice {d} in functor {functor.name!r} gives"
                    " tensor elements more than one destination")
    if len(functor.rhs) != functor.feature_count:
        raise FeatureMismatchError(
            f"scatter functor {functor.name!r} has {len(functor.rhs)} point"
            f" slice(s) but declares {functor.feature_count} feature(s)")


def scatter_from(functor: FunctorDecl, target: MapTarget, tensor: Tensor,
                 array: ArrayBuffer) -> None:
    """Dense tensor -> exactly the mapped elements of `array`, in place.
    Injectivity is proven (or refuted) once at plan time, before any write."""
    check_scatter_functor(functor)
    want = expected_tensor_shape(functor, target)
    if tensor.shape != want:
        raise ShapeMismatchError(f"tensor shape {tensor.shape} does not match mapping shape {want}")
    _require_device(array)
    views = _views_for(functor, target, array)
    plan = build_plan([views], "from")
    src = tensor.data
    if src.device != array.device:
        src = src.to(array.device)
    src = src.contiguous()
    ptrs, dts = plan.ptrs_and_dtypes()
    _native.scatter(plan.handle, src.data_ptr(), DTYPE_CODE[tensor.dtype], ptrs, dts,
                    0, plan.n_rows, _stream_ptr(array.device))


def gather_batch(functor: FunctorDecl, target: MapTarget, array: ArrayBuffer):
    """Concretize and flatten to (batch, features)."""
    t = concretize_to(functor, target, array)
    n_sweep = len(target.slices)
    batch = int(np.prod(t.shape[:n_sweep], dtype=np.int64)) if n_sweep else 1
    return t, t.data.reshape(batch, -1)
