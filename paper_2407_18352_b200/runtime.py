"""Execution control: the reference's Runtime API over the B200 data path.

Same registry, dispatch, caches, outcome/stats records and error classes as
`/root/reference/pkg/src/smlrt/runtime.py:129-398`.  What changes is the body
of the two data paths:

* `_run_surrogate` (runtime.py:308-370) validates the maps on the host, looks
  up (or compiles once) the gather and scatter plans, and issues ONE native
  call, `smlrt_region_infer`: gather -> forward pass -> scatter fused in a
  single sm_100a kernel (fp32-exact CUDA-core or bf16 tcgen05 by model
  precision).  The only device->host traffic is the 4-byte status word.
* `_run_collect` (runtime.py:279-306) gathers the inputs with the native
  gather kernel into HBM, copies the dense tile to pinned host memory on a
  side stream (`smlrt_collect_async`), runs the accurate callback, gathers the
  outputs the same way and appends the record to the SRDB store.

Application arrays normally live in HBM.  A host-resident ArrayBuffer is
staged through a cached device mirror (H2D before, D2H of written outputs
after): that is the end-to-end path the bench times with host buffers.

Sharding: `Runtime(shard=(rank, world))` restricts every invocation to the
rank's contiguous block of flattened sweep rows (axis 0 blocks for row-major
sweeps); there is no collective on the inference path.

A Runtime instance belongs to one thread of control (runtime.py:22).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field, replace
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _native, srdb
from .bridge import (
    ArrayBuffer,
    DTYPE_CODE,
    Plan,
    Tensor,
    _check_features,
    _views_for,
    build_plan,
    check_scatter_functor,
    expected_tensor_shape,
)
from .directives import FunctorDecl, MapTarget, MlDirective
from .errors import (
    DeviceError,
    DuplicateRegionError,
    InvalidScheduleError,
    MissingClauseError,
    MissingPredicateError,
    ModelLoadError,
    ModelShapeMismatchError,
    NonFiniteOutputError,
    ShapeMismatchError,
    UnknownRegionError,
)
from .models import Model, device_model, load_model

__all__ = ["BoundMap", "RegionDescriptor", "RegionOutcome", "RegionStats", "Runtime",
           "interleave_predicate"]

ACCURATE = "accurate"
SURROGATE = "surrogate"


@dataclass
class BoundMap:
    functor: FunctorDecl
    target: MapTarget
    array: ArrayBuffer


@dataclass
class RegionDescriptor:
    name: str
    accurate_fn: Callable[[], None]
    ml: MlDirective
    in_maps: list = field(default_factory=list)
    out_maps: list = field(default_factory=list)
    inout_maps: list = field(default_factory=list)
    env: dict = field(default_factory=dict)


@dataclass
class RegionOutcome:
    """elapsed_region_ns: the executed body (accurate callback, or the fused
    surrogate launch through its completion).  On the fused path map_to covers
    host validation + plan lookup and map_from the status check; the device
    work of gather and scatter is inside the infer interval."""

    path_taken: str
    elapsed_region_ns: int
    elapsed_map_to_ns: int = 0
    elapsed_map_from_ns: int = 0
    elapsed_infer_ns: int = 0
    record_index: Optional[int] = None


@dataclass
class RegionStats:
    invocations: int = 0
    accurate_calls: int = 0
    surrogate_calls: int = 0
    records: int = 0
    model_loads: int = 0
    map_to_ns: int = 0
    map_from_ns: int = 0
    infer_ns: int = 0
    accurate_ns: int = 0


def interleave_predicate(step: int, n_accurate: int, n_surrogate: int) -> bool:
    """True on the surrogate part of a repeating n_accurate:n_surrogate schedule."""
    if n_accurate < 0 or n_surrogate < 0:
        raise InvalidScheduleError("interleave counts must be non-negative")
    period = n_accurate + n_surrogate
    if period == 0:
        raise InvalidScheduleError("interleave schedule needs a non-zero period")
    return (step % period) >= n_accurate


def _resolve_refs(refs: Sequence[str], maps: Sequence[BoundMap], clause: str):
    names = {}
    for m in maps:
        if m.target.array in names:
            raise MissingClauseError(f"array {m.target.array!r} bound twice in {clause} maps")
        names[m.target.array] = m
    for r in refs:
        if r not in names:
            raise MissingClauseError(f"ml {clause}({r}) has no matching bound map")


def _ns_since(t0: int) -> int:
    return max(time.perf_counter_ns() - t0, 1)


def _shard_rows(n_rows: int, shard, inner: int = 1) -> tuple[int, int]:
    """Flattened sweep rows [r0, r1) of a shard: sweep axis 0 split into
    contiguous blocks; `inner` = product of the other sweep
    extents, so a shard of a 2-D sweep is whole rows of the grid."""
    if shard is None:
        return 0, n_rows
    rank, world = shard
    a0 = n_rows // inner
    per = -(-a0 // world)
    return min(rank * per, a0) * inner, min((rank + 1) * per, a0) * inner


def _inner_of(plan) -> int:
    """product of the sweep extents after axis 0 (1 for a 1-D sweep)"""
    return int(np.prod(plan.sweep[1:], dtype=np.int64)) if plan.sweep is not None and len(plan.sweep) > 1 else 1


def gather_rows_to_root(local: torch.Tensor, n_rows: int, shard, root: int = 0, group=None, inner: int = 1):
    """Concatenate every rank's block of sweep rows (`_shard_rows` order) on
    `root`: the collect snapshots of a sharded region go to the one rank that
    holds the SRDB writer lock (srdb.py:116-126), SURVEY.md 8(e).  `local` is
    this rank's [r1 - r0, F] tile; blocks are padded to the largest so one
    collective (NCCL send/recv under torch.distributed.gather) moves them.
    Returns the [n_rows, F] tensor on root, None elsewhere."""
    import torch.distributed as dist
    rank, world = shard
    per = -(-(n_rows // inner) // world) * inner  # the largest block (_shard_rows)
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        local = local.cpu()  # gloo gathers host tensors (NCCL moves device tensors directly)
    buf = local
    if local.shape[0] != per:
        buf = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == root else None
    dist.gather(buf.contiguous(), parts, dst=root, group=group)
    if rank != root:
        return None
    return torch.cat(parts)[:n_rows]


class _Staging:
    """Device mirrors of host-resident ArrayBuffers (the e2e path)."""

    def __init__(self):
        self._mirror: dict[int, tuple[torch.Tensor, ArrayBuffer]] = {}
        self.h2d_bytes = 0  # host<->device bytes moved by the e2e path (instrumentation)
        self.d2h_bytes = 0

    def device_view(self, a: ArrayBuffer, device: torch.device) -> ArrayBuffer:
        if a.is_device:
            return a
        key = id(a.data)
        hit = self._mirror.get(key)
        if hit is None or hit[0].numel() != a.data.numel() or hit[0].dtype != a.data.dtype:
            t = torch.empty(a.data.numel(), dtype=a.data.dtype, device=device)
            hit = (t, ArrayBuffer(t, a.shape, a.strides))
            self._mirror[key] = hit
        return hit[1]

    def upload(self, a: ArrayBuffer, dev_a: ArrayBuffer):
        if dev_a is not a:
            dev_a.data.copy_(a.data, non_blocking=a.data.is_pinned())
            self.h2d_bytes += a.data.numel() * a.data.element_size()

    def download(self, a: ArrayBuffer, dev_a: ArrayBuffer):
        if dev_a is not a:
            a.data.copy_(dev_a.data, non_blocking=a.data.is_pinned())
            self.d2h_bytes += a.data.numel() * a.data.element_size()


class Runtime:
    """Registry of annotated regions plus model, plan and database caches.

    precision: override every model's precision ("fp32" exact | "bf16").
    commit:    "fused" (outputs written from the kernel epilogue) or "checked"
               (staged; nothing written if the output is non-finite, the
               reference's error-before-write order, runtime.py:341-344).
    shard:     (rank, world) row block processed by this instance.
    graphs:    replay the launches of a repeated device-resident region as
               one CUDA graph (smlrt_region_prepare); default on,
               SMLRT_GRAPHS=0 turns it off.
    collect_root: with `shard` and an initialised torch.distributed group,
               ml(collect) snapshots each rank's rows and gathers them on
               this rank, the single SRDB writer (srdb.py:116-126).
    """

    def __init__(self, precision: Optional[str] = None, commit: str = "fused",
                 shard: Optional[tuple[int, int]] = None, device=None, graphs: Optional[bool] = None,
                 collect_root: int = 0):
        if commit not in ("fused", "checked"):
            raise ValueError("commit must be 'fused' or 'checked'")
        self._regions: dict[str, RegionDescriptor] = {}
        self._stats: dict[str, RegionStats] = {}
        self._models: dict[str, Model] = {}
        self._dbs: dict[str, srdb.SrdbDatabase] = {}
        self._plans: dict[str, tuple] = {}
        self._staging = _Staging()
        self._side = None  # (host->device, device->host) streams of the chunked host path
        self._collect_side = None  # device->host stream of the collect snapshots
        self._pinned_bufs: dict = {}  # (region, direction) -> reused pinned host buffer
        self._fast: dict = {}  # region -> (key, prepared native call) of device-resident regions
        self.precision = precision
        self.commit = commit
        self.shard = shard
        self.graphs = graphs if graphs is not None else os.environ.get("SMLRT_GRAPHS", "1") != "0"
        self.collect_root = collect_root
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else None)
        self._status = None
        # bench/profiling hook: device time of each region's launches (CUDA
        # events on their stream; kernel_times() reads them as ms)
        self.time_kernels = False
        self.kernel_events: list = []
        self._realpaths: dict = {}  # model path -> realpath (the model cache key, runtime.py:186)

    # -- registration ---------------------------------------------------------

    def register_region(self, desc: RegionDescriptor) -> str:
        ml = desc.ml
        if ml.mode in ("infer", "predicated") and not ml.model_path:
            raise MissingClauseError(f"ml({ml.mode}) region without a model path")
        if ml.mode in ("collect", "predicated") and not ml.db_path:
            raise MissingClauseError(f"ml({ml.mode}) region without a db path")
        _resolve_refs(ml.in_refs, desc.in_maps, "in")
        _resolve_refs(ml.out_refs, desc.out_maps, "out")
        _resolve_refs(ml.inout_refs, desc.inout_maps, "inout")
        prev = self._regions.get(desc.name)
        if prev is not None:
            if prev != desc:
                raise DuplicateRegionError(
                    f"region {desc.name!r} already registered with a different descriptor")
            return desc.name
        self._regions[desc.name] = desc
        self._stats[desc.name] = RegionStats()
        return desc.name

    def _region(self, handle: str) -> RegionDescriptor:
        try:
            return self._regions[handle]
        except KeyError:
            raise UnknownRegionError(f"no region registered as {handle!r}") from None

    # -- caches ---------------------------------------------------------------

    def _model_for(self, desc: RegionDescriptor) -> Model:
        key = self._realpaths.get(desc.ml.model_path)
        if key is None:
            key = self._realpaths[desc.ml.model_path] = os.path.realpath(desc.ml.model_path)
        m = self._models.get(key)
        if m is None:
            try:
                m = load_model(desc.ml.model_path)
            except Exception as e:
                raise ModelLoadError(f"cannot load model {desc.ml.model_path!r}: {e}") from e
            self._models[key] = m
            self._stats[desc.name].model_loads += 1
        return m

    def _db_for(self, desc: RegionDescriptor) -> srdb.SrdbDatabase:
        path = desc.ml.db_path
        db = self._dbs.get(path)
        if db is None:
            exists = os.path.exists(os.path.join(path, srdb.MANIFEST_NAME))
            db = srdb.open_db(path, "append" if exists else "create")
            self._dbs[path] = db
        return db

    def unload_models(self):
        """Drop cached models; the next inference reloads from disk."""
        self._fast.clear()
        self._models.clear()
        self._realpaths.clear()

    def close(self):
        for db in self._dbs.values():
            db.close()
        self._dbs.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _status_word(self) -> torch.Tensor:
        if self._status is None:
            self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        return self._status

    # -- invocation -----------------------------------------------------------

    def invoke_region(self, handle: str, predicate_value: Optional[bool] = None,
                      if_value: Optional[bool] = None) -> RegionOutcome:
        desc = self._region(handle)
        st = self._stats[handle]
        st.invocations += 1
        ml = desc.ml
        if ml.if_cond is not None:
            if if_value is None:
                raise MissingPredicateError(
                    f"region {handle!r} has an if({ml.if_cond}) clause; pass if_value on every invocation")
            if not if_value:
                return self._run_plain_accurate(desc, st)
        if ml.mode == "collect":
            surrogate = False
        elif ml.mode == "infer":
            surrogate = True
        else:
            if predicate_value is None:
                raise MissingPredicateError(
                    f"region {handle!r} is predicated ({ml.predicate}); pass predicate_value on every invocation")
            surrogate = bool(predicate_value)
        return self._run_surrogate(desc, st) if surrogate else self._run_collect(desc, st)

    # -- paths ----------------------------------------------------------------

    def _sync(self):
        if self.device is not None:
            torch.cuda.current_stream(self.device).synchronize()

    def _run_plain_accurate(self, desc, st) -> RegionOutcome:
        self._sync()
        t0 = time.perf_counter_ns()
        desc.accurate_fn()
        self._sync()
        dt = _ns_since(t0)
        st.accurate_calls += 1
        st.accurate_ns += dt
        return RegionOutcome(path_taken=ACCURATE, elapsed_region_ns=dt)

    def _device_maps(self, maps):
        out = []
        for m in maps:
            if m.array.is_device:
                out.append(m)
            else:
                if self.device is None:
                    raise RuntimeError("no CUDA device: the B200 runtime has no CPU data path")
                out.append(BoundMap(m.functor, m.target,
                                    self._staging.device_view(m.array, self.device)))
        return out

    def _gather_dense(self, maps, rows=None) -> Tensor:
        """_combined_tensor (runtime.py:379-398) on the device; `rows` = (r0, r1)
        restricts it to a block of the flattened sweep ([r1 - r0, F])."""
        if not maps:
            raise MissingClauseError("region has no maps for this direction")
        groups, sweep = [], None
        for m in maps:
            views = _views_for(m.functor, m.target, m.array)
            s = _check_features(views, m.functor)
            if sweep is None:
                sweep = s
            elif s != sweep:
                raise ShapeMismatchError(f"map over {m.target.array!r} sweeps {s}, expected {sweep}")
            groups.append(views)
        dt = "f64" if any(m.array.dtype == "f64" for m in maps) else "f32"
        plan = build_plan(groups, "to")
        r0, r1 = rows if rows is not None else (0, plan.n_rows)
        out = torch.empty((r1 - r0, plan.n_cols), device=self.device,
                          dtype=torch.float32 if dt == "f32" else torch.float64)
        ptrs, dts = plan.ptrs_and_dtypes()
        _native.gather(plan.handle, ptrs, dts, out.data_ptr(), DTYPE_CODE[dt], r0, r1,
                       torch.cuda.current_stream(self.device).cuda_stream)
        if rows is not None:
            return Tensor(out)
        return Tensor(out.reshape(tuple(sweep) + (plan.n_cols,)))

    def _pinned(self, key, shape, dtype) -> torch.Tensor:
        """Pinned host staging buffer of the collect path, reused across calls
        (one per region direction; page-locking is the expensive part of a
        host allocation).  The SRDB append consumes it synchronously, so the
        next call may overwrite it."""
        buf = self._pinned_bufs.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape) or buf.dtype != dtype:
            buf = torch.empty(shape, dtype=dtype, pin_memory=True)
            self._pinned_bufs[key] = buf
        return buf

    def _snapshot(self, maps, key=None):
        """Gather on the compute stream, copy to pinned host memory on a side stream."""
        t = self._gather_dense(maps)
        host = self._pinned(key, t.data.shape, t.data.dtype) if key is not None else \
            torch.empty(t.data.shape, dtype=t.data.dtype, pin_memory=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        side = self._side_stream()
        _native.collect_async(t.data.data_ptr(), t.data.numel() * t.data.element_size(),
                              host.data_ptr(), side.cuda_stream, ev.cuda_event)
        return host, t

    def _side_stream(self):
        s = self._collect_side
        if s is None:
            s = self._collect_side = torch.cuda.Stream(self.device)
        return s

    def _collect_sharded(self) -> bool:
        if self.shard is None or self.shard[1] <= 1:
            return False
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()

    def _run_collect_sharded(self, desc, st) -> RegionOutcome:
        """ml(collect) of a sharded region: each rank snapshots its block of
        sweep rows, the blocks meet on the writer rank (gather_rows_to_root),
        which appends the one record; every rank returns its index."""
        import torch.distributed as dist
        in_maps = self._device_maps(desc.in_maps + desc.inout_maps)
        out_maps = self._device_maps(desc.out_maps + desc.inout_maps)
        rank, world = self.shard
        t0 = time.perf_counter_ns()
        for m, d in zip(desc.in_maps + desc.inout_maps, in_maps):
            self._staging.upload(m.array, d.array)
        n_rows = self._plans_rows(in_maps)
        sweep = self._sweep_of(in_maps)
        inner = int(np.prod(sweep[1:], dtype=np.int64)) if len(sweep) > 1 else 1
        rows = _shard_rows(n_rows, self.shard, inner)
        x_loc = self._gather_dense(in_maps, rows=rows).data
        self._sync()
        map_to = _ns_since(t0)
        t0 = time.perf_counter_ns()
        desc.accurate_fn()
        self._sync()
        region_ns = _ns_since(t0)
        t0 = time.perf_counter_ns()
        for m, d in zip(desc.out_maps + desc.inout_maps, out_maps):
            self._staging.upload(m.array, d.array)
        y_loc = self._gather_dense(out_maps, rows=rows).data
        x_all = gather_rows_to_root(x_loc, n_rows, self.shard, root=self.collect_root, inner=inner)
        y_all = gather_rows_to_root(y_loc, n_rows, self.shard, root=self.collect_root, inner=inner)
        index = -1
        if rank == self.collect_root:
            xs = self._full_shape(in_maps, x_all)
            ys = self._full_shape(out_maps, y_all)
            x_host = self._pinned((desc.name, "in"), xs.shape, xs.dtype)
            y_host = self._pinned((desc.name, "out"), ys.shape, ys.dtype)
            x_host.copy_(xs)
            y_host.copy_(ys)
            index = self._db_for(desc).append_record(desc.name, x_host.numpy(), y_host.numpy(), region_ns)
        idx = torch.tensor([index], dtype=torch.int64, device=self.device)
        dist.broadcast(idx, src=self.collect_root)
        map_from = _ns_since(t0)
        st.accurate_calls += 1
        st.accurate_ns += region_ns
        st.map_to_ns += map_to
        st.map_from_ns += map_from
        st.records += 1
        return RegionOutcome(path_taken=ACCURATE, elapsed_region_ns=region_ns,
                             elapsed_map_to_ns=map_to, elapsed_map_from_ns=map_from,
                             record_index=int(idx.item()))

    @staticmethod
    def _sweep_of(maps):
        m = maps[0]
        views = _views_for(m.functor, m.target, m.array)
        return tuple(views[0].shape[: views[0].n_sweep])

    def _plans_rows(self, maps) -> int:
        return int(np.prod(self._sweep_of(maps), dtype=np.int64))

    def _full_shape(self, maps, flat: torch.Tensor) -> torch.Tensor:
        return flat.reshape(self._sweep_of(maps) + (flat.shape[-1],))

    def _run_collect(self, desc, st) -> RegionOutcome:
        if self._collect_sharded():
            return self._run_collect_sharded(desc, st)
        in_maps = self._device_maps(desc.in_maps + desc.inout_maps)
        out_maps = self._device_maps(desc.out_maps + desc.inout_maps)
        t0 = time.perf_counter_ns()
        for m, d in zip(desc.in_maps + desc.inout_maps, in_maps):
            self._staging.upload(m.array, d.array)
        x_host, x_dev = self._snapshot(in_maps, (desc.name, "in"))
        self._sync()
        map_to = _ns_since(t0)

        t0 = time.perf_counter_ns()
        desc.accurate_fn()
        self._sync()
        region_ns = _ns_since(t0)

        t0 = time.perf_counter_ns()
        for m, d in zip(desc.out_maps + desc.inout_maps, out_maps):
            self._staging.upload(m.array, d.array)
        y_host, y_dev = self._snapshot(out_maps, (desc.name, "out"))
        _native.collect_wait(self._side_stream().cuda_stream)
        map_from = _ns_since(t0)

        index = self._db_for(desc).append_record(desc.name, x_host.numpy(), y_host.numpy(),
                                                 region_ns)
        st.accurate_calls += 1
        st.accurate_ns += region_ns
        st.map_to_ns += map_to
        st.map_from_ns += map_from
        st.records += 1
        return RegionOutcome(path_taken=ACCURATE, elapsed_region_ns=region_ns,
                             elapsed_map_to_ns=map_to, elapsed_map_from_ns=map_from,
                             record_index=index)

    def _plans_for(self, desc, in_maps, out_maps):
        key = tuple((id(m.array.data), m.array.shape, m.array.strides, m.array.dtype,
                     id(m.functor), m.target) for m in in_maps + out_maps)
        hit = self._plans.get(desc.name)
        if hit is not None and hit[0] == key:
            return hit[1], hit[2], hit[3]
        # in-maps: gather_batch per map in order (runtime.py:312-324)
        groups, batch_rows = [], None
        for m in in_maps:
            views = _views_for(m.functor, m.target, m.array)
            sweep = _check_features(views, m.functor)
            rows = int(np.prod(sweep, dtype=np.int64))
            if batch_rows is None:
                batch_rows = rows
            elif rows != batch_rows:
                raise ShapeMismatchError("input maps disagree on the sweep/batch size")
            groups.append(views)
        pin = build_plan(groups, "to") if _same_sweeps(groups) else _flat_plan(groups, "to")
        # out-maps: shape checks (runtime.py:344-352) then scatter_from's checks
        ogroups = []
        for m in out_maps:
            shape = expected_tensor_shape(m.functor, m.target)
            rows = int(np.prod(shape[: len(m.target.slices)], dtype=np.int64))
            if rows != batch_rows:
                raise ModelShapeMismatchError(
                    f"output map over {m.target.array!r} sweeps {rows} entries, batch holds {batch_rows}")
            check_scatter_functor(m.functor)
            ogroups.append(_views_for(m.functor, m.target, m.array))
        pout = build_plan(ogroups, "from") if _same_sweeps(ogroups) else _flat_plan(ogroups, "from")
        self._plans[desc.name] = (key, pin, pout, batch_rows)
        return pin, pout, batch_rows

    def _fast_key(self, desc, model):
        """What a prepared call depends on: the bound arrays' storage and
        geometry, the functors/targets, the model object and the runtime's
        settings.  Equal keys -> the cached native arguments are still valid."""
        maps = desc.in_maps + desc.out_maps + desc.inout_maps
        return (id(model), self.precision, self.commit, self.shard,
                tuple((id(m.array.data), m.array.data.data_ptr(), m.array.data.dtype, m.array.shape,
                       m.array.strides, id(m.functor), id(m.target)) for m in maps))

    def _run_surrogate(self, desc, st) -> RegionOutcome:
        model = self._model_for(desc)
        if self.device is None:
            raise RuntimeError("no CUDA device: the B200 runtime has no CPU data path")
        fast = self._fast.get(desc.name)
        if fast is not None and fast[0] == self._fast_key(desc, model):
            return self._run_prepared(fast[1], st)
        host_in = desc.in_maps + desc.inout_maps
        host_out = desc.out_maps + desc.inout_maps
        t0 = time.perf_counter_ns()
        in_maps = self._device_maps(host_in)
        out_maps = self._device_maps(host_out)
        pin, pout, rows = self._plans_for(desc, in_maps, out_maps)
        if pin.n_cols != model.input_features:
            raise ModelShapeMismatchError(
                f"region {desc.name!r} gathers {pin.n_cols} features, model expects {model.input_features}")
        out_counts = sum(m.functor.feature_count for m in out_maps)
        if out_counts != model.output_features:
            raise ModelShapeMismatchError(
                f"region {desc.name!r} scatters {out_counts} features, model emits {model.output_features}")
        handle = device_model(model, self.device, self.precision)
        chunks = self._stream_chunks(desc, host_in, host_out, pin, pout, rows)
        if chunks is not None:
            return self._run_streamed(st, host_in[0], in_maps[0], host_out[0], out_maps[0], pin, pout, chunks,
                                      handle, _ns_since(t0))
        # an output array sharing storage with an input array (inout maps, or
        # in/out maps over one buffer): outputs are staged and scattered after
        # every row has been gathered -- the reference's gather-all / infer /
        # scatter order (runtime.py:315-357) -- instead of written from the
        # fused epilogue while other rows may still be reading
        staged = self.commit == "checked" or _shares_storage(pin, pout)
        for m, d in zip(host_in, in_maps):
            self._staging.upload(m.array, d.array)
        # a host output's device mirror is downloaded whole afterwards, so it
        # must hold the host's values wherever this call may not write: skip
        # the upload only when the scatter surely writes every element (no
        # shard, and no checked/staged commit that writes nothing on error)
        skip_ok = self.shard is None and not staged
        for m, d in zip(host_out, out_maps):
            if not m.array.is_device and not (skip_ok and _covers(pout, d.array)):
                self._staging.upload(m.array, d.array)
        r0, r1 = _shard_rows(rows, self.shard, _inner_of(pin))
        status = self._status_word()
        stream = torch.cuda.current_stream(self.device)
        map_to = _ns_since(t0)

        t0 = time.perf_counter_ns()
        iptr, idt = pin.ptrs_and_dtypes()
        optr, odt = pout.ptrs_and_dtypes()
        flags = _native.COMMIT_CHECKED if staged else _native.COMMIT_FUSED
        # device-resident outputs: status reset, launch, status read-back and
        # the stream sync happen inside one native call (SMLRT_SYNC_STATUS)
        sync_native = all(m.array.is_device for m in host_out)
        if sync_native:
            flags |= _native.SYNC_STATUS
            # device-resident region: later calls with the same arrays, model
            # and settings replay a prepared native call (a CUDA graph of
            # this call's launches) with these arguments
            if all(m.array.is_device for m in host_in):
                try:
                    self._fast[desc.name] = (self._fast_key(desc, model), _native.prepare_region(
                        pin.handle, iptr, idt, pout.handle, optr, odt, handle, r0, r1, flags, status.data_ptr(),
                        pin, pout, model, graph=self.graphs))
                except DeviceError:
                    self._fast.pop(desc.name, None)  # no prepared call: every call takes this path
        else:
            status.zero_()
        if self.time_kernels:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(stream)
        bad = 0
        try:
            _native.region_infer(pin.handle, iptr, idt, pout.handle, optr, odt, handle, r0, r1,
                                 flags, None, stream.cuda_stream, status.data_ptr())
        except NonFiniteOutputError:
            bad = 1
        if self.time_kernels:
            ev[1].record(stream)
            self.kernel_events.append(ev)
        if not sync_native:
            for m, d in zip(host_out, out_maps):
                self._staging.download(m.array, d.array)
            bad = int(status.item())  # synchronises the stream
        infer_ns = _ns_since(t0)

        t0 = time.perf_counter_ns()
        if bad:
            raise NonFiniteOutputError("forward pass produced NaN/inf")
        map_from = _ns_since(t0)
        st.surrogate_calls += 1
        st.map_to_ns += map_to
        st.map_from_ns += map_from
        st.infer_ns += infer_ns
        return RegionOutcome(path_taken=SURROGATE, elapsed_region_ns=infer_ns,
                             elapsed_map_to_ns=map_to, elapsed_map_from_ns=map_from,
                             elapsed_infer_ns=infer_ns)

    def _run_prepared(self, call, st) -> RegionOutcome:
        """The steady-state surrogate call: one native call (status reset,
        graph launch, status read-back, stream sync) with cached arguments."""
        t0 = time.perf_counter_ns()
        if self.time_kernels:
            ms = []
            bad = call(torch._C._cuda_getCurrentRawStream(self.device.index), ms)
            self.kernel_events.append(ms[0])
        else:
            bad = call(torch._C._cuda_getCurrentRawStream(self.device.index))
        infer_ns = _ns_since(t0)
        if bad:
            raise NonFiniteOutputError("forward pass produced NaN/inf")
        st.surrogate_calls += 1
        st.infer_ns += infer_ns
        return RegionOutcome(path_taken=SURROGATE, elapsed_region_ns=infer_ns, elapsed_infer_ns=infer_ns)

    # host-resident (pinned) input and output over uniform 1-D plans (AoS rows
    # or SoA columns): the row range is cut into chunks whose host->device
    # copies (the element ranges the chunk's rows touch, smlrt_plan_row_ranges),
    # kernel and device->host copies run on three streams, so the PCIe
    # transfers overlap the kernel and each other
    # (below ~64 MB the per-chunk host overhead outweighs the overlap: options
    # 20 MB, 0.64 ms staged whole vs 0.74 ms in 8 chunks)
    STREAM_MIN_BYTES = 64 << 20
    STREAM_CHUNK_BYTES = 16 << 20  # minimum input bytes per chunk; at most STREAM_CHUNKS chunks
    STREAM_CHUNKS = 16

    def _stream_chunks(self, desc, host_in, host_out, pin, pout, rows):
        """The chunk schedule of the chunked host path -- [(a, b, in_ranges,
        out_ranges)] -- or None when the call does not qualify.  Every chunk's
        element ranges are computed before anything is launched: a plan whose
        whole-range intervals merge (e.g. SoA columns) may still need more
        ranges per chunk than plan_row_ranges allows, and then the call takes
        the whole-array path instead of failing half-way."""
        if self.time_kernels or self.commit != "fused" or desc.inout_maps:
            return None
        if len(host_in) != 1 or len(host_out) != 1:
            return None
        r0, r1 = _shard_rows(rows, self.shard, _inner_of(pin))
        if r1 <= r0:
            return None
        if _shares_storage(pin, pout):
            return None
        for m, plan in ((host_in[0], pin), (host_out[0], pout)):
            if m.array.is_device or not m.array.data.is_pinned() or len(plan.arrays) != 1:
                return None
        in_bytes = (r1 - r0) * pin.n_cols * host_in[0].array.data.element_size()
        if in_bytes < self.STREAM_MIN_BYTES:
            return None
        row_bytes = pin.n_cols * host_in[0].array.data.element_size()
        step = max(-(-self.STREAM_CHUNK_BYTES // row_bytes), -(-(r1 - r0) // self.STREAM_CHUNKS))
        if len(pin.sweep) == 2:
            return self._band_chunks(pin, pout, r0, r1, step)
        box = _window_box(pin)
        chunks = []
        for a in range(r0, r1, step):
            b = min(r1, a + step)
            ri = _native.plan_row_ranges(pin.handle, a, b)
            ro = _native.plan_row_ranges(pout.handle, a, b)
            if ro is None or not ro[1]:
                return None
            if box is not None and (ri is None or not ri[1]):
                # a window functor: the chunk's windows as one strided box
                # (exactly the window bytes, where merged ranges copy the gaps)
                off, w, h, pitch, slice_ = box
                chunks.append((a, b, ("box", (off + a * slice_, w, h, b - a, pitch, slice_)), ro[0]))
                continue
            if ri is None:
                return None
            # gaps inside an input's ranges are copied too: allow at most 2x the touched elements
            if sum(hi - lo for lo, hi in ri[0]) > 2 * (b - a) * pin.n_cols:
                return None
            chunks.append((a, b, ri[0], ro[0]))
        return chunks

    def _band_chunks(self, pin, pout, r0, r1, step):
        """2-D sweeps (a halo stencil over grid rows): chunks are bands of whole
        sweep rows; each band's input (its rows plus the halo) and output (the
        band's interior) are strided 3-D boxes, copied exactly."""
        bi, bo = _sweep_box(pin), _sweep_box(pout)
        if bi is None or bo is None or tuple(pout.sweep) != tuple(pin.sweep):
            return None
        nj = pin.sweep[1]
        if r0 % nj or (r1 % nj and r1 != pin.n_rows):
            return None
        rows_per = max(1, step // nj)
        chunks = []
        for ia in range(r0 // nj, -(-r1 // nj), rows_per):
            ib = min(-(-r1 // nj), ia + rows_per)
            boxes = []
            for (off, w, h, d, pitch, slice_, s0) in (bi, bo):
                boxes.append(("box", (off + ia * s0, w, h + (ib - ia) - 1, d, pitch, slice_)))
            chunks.append((ia * nj, min(r1, ib * nj), boxes[0], [boxes[1]]))
        return chunks

    def _run_streamed(self, st, hin_map, din_map, hout_map, dout_map, pin, pout, chunks, handle, map_to):
        t0 = time.perf_counter_ns()
        cs = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
        up, down = self._side
        status = self._status_word()
        status.zero_()
        hin, din = hin_map.array.data.view(-1), din_map.array.data.view(-1)
        hout, dout = hout_map.array.data.view(-1), dout_map.array.data.view(-1)
        iptr, idt = pin.ptrs_and_dtypes()
        optr, odt = pout.ptrs_and_dtypes()
        up.wait_stream(cs)      # the mirrors may still be read/written by earlier work
        down.wait_stream(cs)
        for a, b, in_ranges, out_ranges in chunks:
            with torch.cuda.stream(up):
                if in_ranges and in_ranges[0] == "box":
                    bx = in_ranges[1]
                    _native.copy_box_async(din.data_ptr(), hin.data_ptr(), hin.element_size(), bx, 0,
                                           up.cuda_stream)
                    self._staging.h2d_bytes += bx[1] * bx[2] * bx[3] * hin.element_size()
                else:
                    for lo, hi in in_ranges:
                        din[lo:hi].copy_(hin[lo:hi], non_blocking=True)
                        self._staging.h2d_bytes += (hi - lo) * hin.element_size()
            cs.wait_stream(up)
            _native.region_infer(pin.handle, iptr, idt, pout.handle, optr, odt, handle, a, b,
                                 _native.COMMIT_FUSED, None, cs.cuda_stream, status.data_ptr())
            down.wait_stream(cs)
            with torch.cuda.stream(down):
                for rng in out_ranges:
                    if rng[0] == "box":
                        bx = rng[1]
                        _native.copy_box_async(hout.data_ptr(), dout.data_ptr(), hout.element_size(), bx, 1,
                                               down.cuda_stream)
                        self._staging.d2h_bytes += bx[1] * bx[2] * bx[3] * hout.element_size()
                        continue
                    lo, hi = rng
                    hout[lo:hi].copy_(dout[lo:hi], non_blocking=True)
                    self._staging.d2h_bytes += (hi - lo) * hout.element_size()
        cs.wait_stream(down)
        bad = int(status.item())  # synchronises the stream
        infer_ns = _ns_since(t0)
        if bad:
            raise NonFiniteOutputError("forward pass produced NaN/inf")
        st.surrogate_calls += 1
        st.map_to_ns += map_to
        st.infer_ns += infer_ns
        return RegionOutcome(path_taken=SURROGATE, elapsed_region_ns=infer_ns,
                             elapsed_map_to_ns=map_to, elapsed_map_from_ns=0,
                             elapsed_infer_ns=infer_ns)

    def kernel_times(self) -> list:
        """ms per timed region call (time_kernels): the prepared call measures
        its own launches; the first call's events are read here."""
        torch.cuda.synchronize(self.device)
        return [e if isinstance(e, float) else e[0].elapsed_time(e[1]) for e in self.kernel_events]

    def stats(self, handle: str) -> RegionStats:
        self._region(handle)
        return replace(self._stats[handle])


def _window_box(plan: Plan):
    """(offset, width, height, pitch, slice) of a window functor's in-plan --
    one view, one sweep axis, a [height, width] window of rows `pitch`
    elements apart, consecutive sweep rows `slice` elements apart (a multiple
    of pitch) -- or None."""
    if len(plan.views) != 1:
        return None
    _, v = plan.views[0]
    if v.n_sweep != 1 or len(v.shape) != 3:
        return None
    slice_, pitch, one = v.strides
    h, w = v.shape[1], v.shape[2]
    if one != 1 or pitch < w or slice_ <= 0 or slice_ % pitch or slice_ < pitch * h:
        return None
    if v.base_offset % pitch + w > pitch:
        return None
    return v.base_offset, w, h, pitch, slice_


def _sweep_box(plan: Plan):
    """The elements a 2-D sweep plan touches as a 3-D box per sweep row, or
    None: sweep strides (s0, 1) and either one view whose feature axes are
    (planes, rows, columns) with strides (slice, s0, 1) -- the halo in-functor
    -- or point views whose bases step by a constant multiple of s0 -- one per
    output plane.  Returns (offset of sweep row 0, width, height of one sweep
    row, depth, pitch, slice, s0): band [ia, ib) spans height + ib - ia - 1
    rows from offset + ia*s0."""
    views = [v for _, v in plan.views]
    if not views or any(v.n_sweep != 2 for v in views):
        return None
    s0 = views[0].strides[0]
    if any(v.strides[:2] != (s0, 1) for v in views) or s0 <= 0:
        return None
    nj = views[0].shape[1]
    if len(views) == 1 and len(views[0].shape) == 5:
        v = views[0]
        d, h, w = v.shape[2:]
        slice_, pitch, one = v.strides[2:]
        if pitch != s0 or one != 1 or slice_ % s0 or slice_ < s0 * h:
            return None
        off, width, height, depth = v.base_offset, nj + w - 1, h, d
    elif all(int(np.prod(v.shape[2:])) == 1 for v in views):
        bases = [v.base_offset for v in views]
        slice_ = bases[1] - bases[0] if len(bases) > 1 else s0 * (1 << 20)
        if any(b1 - b0 != slice_ for b0, b1 in zip(bases, bases[1:])) or slice_ <= 0 or slice_ % s0:
            return None
        off, width, height, depth = bases[0], nj, 1, len(bases)
    else:
        return None
    if off % s0 + width > s0:
        return None
    return off, width, height, depth, s0, slice_, s0


def _same_sweeps(groups) -> bool:
    sweeps = {g[0].shape[: g[0].n_sweep] for g in groups}
    return len(sweeps) == 1


def _flat_plan(groups, direction):
    """Maps with equal row counts but different sweep shapes: re-express each
    view over a 1-D sweep when its sweep strides allow it (row-major
    collapsible), else refuse."""
    from .bridge import MemoryView
    flat = []
    for views in groups:
        fv = []
        for v in views:
            sweep, strides = v.shape[: v.n_sweep], v.strides[: v.n_sweep]
            for k in range(len(sweep) - 1):
                if strides[k] != strides[k + 1] * sweep[k + 1]:
                    raise ShapeMismatchError(
                        "maps with different sweep shapes need row-major collapsible strides")
            n = int(np.prod(sweep))
            fv.append(MemoryView(v.source, v.base_offset, (n,) + v.shape[v.n_sweep:],
                                 (strides[-1],) + v.strides[v.n_sweep:], 1))
        flat.append(fv)
    return build_plan(flat, direction)


def _shares_storage(pin: Plan, pout: Plan) -> bool:
    """True when an element the out plan writes may be an element the in plan
    reads (in device memory).  Arrays that do not overlap at all, or whose
    touched address intervals do not overlap, are independent; over one
    buffer, views whose sweep strides share a pitch P and whose touched
    offsets mod P are disjoint (e.g. an AoS record's input fields and a
    separate output field) are independent too.  Anything else counts as
    shared (conservative: the call is staged)."""
    def span(a):
        t = a.data
        lo = t.data_ptr()
        return lo, lo + t.numel() * t.element_size()

    def touched(plan, k):
        a = plan.arrays[k]
        es = a.data.element_size()
        base = a.data.data_ptr()
        out = []
        for idx, v in plan.views:
            if idx != k:
                continue
            hi = v.base_offset + sum((n - 1) * st for n, st in zip(v.shape, v.strides))
            out.append((v, base + v.base_offset * es, base + (hi + 1) * es))
        return out

    def residues(v, pitch, limit=4096):
        feat_n, feat_s = v.shape[v.n_sweep:], v.strides[v.n_sweep:]
        if int(np.prod(feat_n)) > limit:
            return None
        offs = {v.base_offset % pitch}
        for n, st in zip(feat_n, feat_s):
            offs = {(o + i * st) % pitch for o in offs for i in range(n)}
        return offs

    for ko, ao in enumerate(pout.arrays):
        olo, ohi = span(ao)
        for ki, ai in enumerate(pin.arrays):
            ilo, ihi = span(ai)
            if not (olo < ihi and ilo < ohi):
                continue
            tin, tout = touched(pin, ki), touched(pout, ko)
            if not any(a0 < b1 and b0 < a1 for _, a0, a1 in tin for _, b0, b1 in tout):
                continue
            if ai.data.data_ptr() != ao.data.data_ptr() or ai.data.element_size() != ao.data.element_size():
                return True
            pitch = 0
            for v, _, _ in tin + tout:
                for n, st in zip(v.shape[: v.n_sweep], v.strides[: v.n_sweep]):
                    if n > 1:
                        pitch = int(np.gcd(pitch, st))
            if pitch <= 1:
                return True
            rin, rout = set(), set()
            for v, _, _ in tin:
                r = residues(v, pitch)
                if r is None:
                    return True
                rin |= r
            for v, _, _ in tout:
                r = residues(v, pitch)
                if r is None:
                    return True
                rout |= r
            if rin & rout:
                return True
    return False


def _covers(plan: Plan, array: ArrayBuffer) -> bool:
    """True when the scatter writes every element of `array` (no upload needed)."""
    if plan.direction != "from" or len(plan.arrays) != 1:
        return False
    info = _native.plan_info(plan.handle)
    return bool(info["dense_rows"]) and info["row_pitch"] == plan.n_cols and \
        plan.n_rows * plan.n_cols == array.data.numel()
