"""The C-ABI library loads and exports every entry point include/smlrt_b200.h
declares; the plan compiler (pure host code) validates without a GPU."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2407_18352_b200 import _native, errors
from paper_2407_18352_b200.bridge import ArrayBuffer, MemoryView, build_plan, _views_for
from paper_2407_18352_b200.directives import ConcreteSlice, MapTarget, parse_functor_decl

HEADER = Path(__file__).resolve().parents[1] / "include" / "smlrt_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(smlrt_[a-z_]+)\s*\(", text)) - {"smlrt_view_t"})


def test_every_declared_symbol_is_exported_and_bound():
    lib = _native.lib()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
        assert n in _native.SIGNATURES, n
    assert "sm_100a" in _native.version()


def cpu_array(shape, dtype=np.float32):
    return ArrayBuffer.from_numpy(np.zeros(shape, dtype), device="cpu")


def plan(ftxt, slices, shape, direction):
    f = parse_functor_decl(ftxt)
    t = MapTarget("a", tuple(ConcreteSlice(*s) for s in slices))
    return build_plan([_views_for(f, t, cpu_array(shape))], direction)


def test_plan_column_table_and_flags():
    p = plan("f: [k, 0:5] = ([k, 0:5])", [(0, 1000)], (1000, 5), "to")
    info = _native.plan_info(p.handle)
    assert (p.n_rows, p.n_cols) == (1000, 5)
    assert info["uniform"] and info["dense_rows"] and info["row_pitch"] == 5
    p = plan("f: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2])", [(1, 3), (1, 3)], (4, 4), "to")
    info = _native.plan_info(p.handle)
    assert (p.n_rows, p.n_cols) == (4, 5) and info["uniform"] and not info["dense_rows"]


def test_plan_injectivity_proofs():
    # MiniWeather output: 4 planes, interior sweep -> proven analytically
    p = plan("f: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j])",
             [(1, 63), (1, 31)], (4, 64, 32), "from")
    assert _native.plan_info(p.handle)["injective"]
    # strides (2,3) over extents (3,2) are injective but not mixed-radix: bitmap path
    arr = cpu_array((64,))
    v = MemoryView(arr, 0, (3, 2, 1), (2, 3, 1), 2)
    p = build_plan([[v]], "from")
    assert _native.plan_info(p.handle)["injective"]
    # overlapping destinations
    with pytest.raises(errors.NonInjectiveScatterError):
        plan("f: [i, 0:2] = ([i], [i+1])", [(1, 4)], (8,), "from")
    with pytest.raises(errors.NonInjectiveScatterError):
        plan("f: [i, j, 0:1] = ([i, 0])", [(0, 2), (0, 3)], (4, 4), "from")
    v = MemoryView(arr, 0, (4, 3, 1), (2, 3, 1), 2)  # 2*3 == 3*2 collide
    with pytest.raises(errors.NonInjectiveScatterError):
        build_plan([[v]], "from")


def test_plan_flat_bounds():
    arr = cpu_array((10,))
    with pytest.raises(errors.OutOfBoundsError):
        build_plan([[MemoryView(arr, 5, (3, 1), (3, 1), 1)]], "to")
    with pytest.raises(errors.OutOfBoundsError):
        build_plan([[MemoryView(arr, -1, (3, 1), (1, 1), 1)]], "to")


def test_rows_limit_and_invalid_args():
    lib = _native.lib()
    import ctypes as C
    h = C.c_void_p()
    rc = lib.smlrt_plan_create(None, 0, 1, None, 0, None, 0, C.byref(h))
    assert rc == 9 and b"empty" in lib.smlrt_last_error()


def test_plan_row_ranges():
    """smlrt_plan_row_ranges: the element ranges a row block touches (the
    chunked host path copies exactly these)."""
    # AoS rows: one merged, exact range
    p = plan("f: [k, 0:5] = ([k, 0:5])", [(0, 1000)], (1000, 5), "to")
    assert _native.plan_row_ranges(p.handle, 10, 20) == ([(50, 100)], True)
    # SoA columns: one exact range per feature
    p = plan("f: [k, 0:6] = ([0:6, k])", [(0, 1000)], (6, 1000), "to")
    rr, exact = _native.plan_row_ranges(p.handle, 100, 300)
    assert exact and rr == [(c * 1000 + 100, c * 1000 + 300) for c in range(6)]
    # SoA with a sub-slice of the sweep (offset base)
    p = plan("f: [k, 0:2] = ([0:2, k])", [(5, 900)], (2, 1000), "to")
    assert _native.plan_row_ranges(p.handle, 0, 10) == ([(5, 15), (1005, 1015)], True)
    # strided columns of AoS records: merged span with gaps -> not exact
    p = plan("f: [k, 0:2] = ([k, 0], [k, 3])", [(0, 1000)], (1000, 5), "to")
    assert _native.plan_row_ranges(p.handle, 2, 4) == ([(10, 19)], False)
    # too many ranges, or a 2-D sweep: unsupported -> None
    p = plan("f: [k, 0:6] = ([0:6, k])", [(0, 1000)], (6, 1000), "to")
    assert _native.plan_row_ranges(p.handle, 0, 10, max_ranges=4) is None
    p = plan("f: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2])", [(1, 3), (1, 3)], (4, 4), "to")
    assert _native.plan_row_ranges(p.handle, 0, 2) is None
    p = plan("f: [k, 0:5] = ([k, 0:5])", [(0, 10)], (10, 5), "to")
    with pytest.raises(ValueError):
        _native.plan_row_ranges(p.handle, 5, 11)


def test_plan_cache_shared_by_geometry():
    """One native plan per geometry, process-wide: two arrays (two Runtimes'
    bindings) with the same shape reuse the validated handle; another
    geometry or direction gets its own."""
    from paper_2407_18352_b200.bridge import PLAN_CACHE
    f = parse_functor_decl("f: [k, 0:5] = ([k, 0:5])")
    t = MapTarget("a", (ConcreteSlice(0, 700),))
    p1 = build_plan([_views_for(f, t, cpu_array((700, 5)))], "to")
    hits = PLAN_CACHE.hits
    a2 = cpu_array((700, 5))
    p2 = build_plan([_views_for(f, t, a2)], "to")
    assert PLAN_CACHE.hits == hits + 1
    assert p2.handle.value == p1.handle.value and p2.arrays[0] is a2
    p3 = build_plan([_views_for(f, t, cpu_array((701, 5)))], "to")  # other extent
    assert p3.handle.value != p1.handle.value
    g = parse_functor_decl("g: [k, 0:1] = ([k, 0])")
    p4 = build_plan([_views_for(g, t, cpu_array((700, 5)))], "from")
    assert p4.handle.value not in (p1.handle.value, p3.handle.value)
    # errors are not cached: the same bad geometry raises every time
    bad = MemoryView(cpu_array((64,)), 0, (4, 3, 1), (2, 3, 1), 2)
    for _ in range(2):
        with pytest.raises(errors.NonInjectiveScatterError):
            build_plan([[bad]], "from")
