"""Host-side plan geometry (extract -> resolve -> wrap) against the reference's
published values (tests/test_bridge.py:58-132) and error classes (golden)."""

import numpy as np
import pytest
import torch

from goldens import functor, meta, target
from paper_2407_18352_b200 import errors
from paper_2407_18352_b200.bridge import (ArrayBuffer, check_scatter_functor, extract_symbolic_shape,
                                          resolve_symbolic_shape, wrap_tensors, _check_features)
from paper_2407_18352_b200.directives import ConcreteSlice, MapTarget, parse_functor_decl, parse_tensor_map

IF = "ifnctr: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2])"


def grid44():
    return ArrayBuffer.from_numpy(np.arange(16, dtype=np.float32).reshape(4, 4), device="cpu")


def test_extraction_offsets():
    f = parse_functor_decl(IF)
    t = parse_tensor_map("map(to: ifnctr(t[1:N-1, 1:M-1]))", {"N": 4, "M": 4}).targets[0]
    d = extract_symbolic_shape(f, t)
    assert d[0].offset_per_dim == (-1, 0) and d[0].elem_count_per_dim == (1, 1)
    assert d[1].offset_per_dim == (1, 0) and d[2].offset_per_dim == (0, -1)
    assert d[2].elem_count_per_dim == (1, 3)
    with pytest.raises(errors.ArityMismatchError):
        extract_symbolic_shape(f, MapTarget("t", (ConcreteSlice(1, 3),)))


def test_resolution_and_view_geometry():
    f = parse_functor_decl(IF)
    t = parse_tensor_map("map(to: ifnctr(t[1:N-1, 1:M-1]))", {"N": 16, "M": 16}).targets[0]
    r = resolve_symbolic_shape(extract_symbolic_shape(f, t), t)
    assert all(x.sweep_shape == (14, 14) for x in r)
    assert [x.feature_shape for x in r] == [(1,), (1,), (3,)]
    t4 = parse_tensor_map("map(to: ifnctr(t[1:N-1, 1:M-1]))", {"N": 4, "M": 4}).targets[0]
    views = wrap_tensors(resolve_symbolic_shape(extract_symbolic_shape(f, t4), t4), grid44())
    assert (views[0].base_offset, views[0].shape, views[0].strides) == (1, (2, 2, 1), (4, 1, 1))
    assert (views[2].base_offset, views[2].shape, views[2].strides) == (4, (2, 2, 3), (4, 1, 1))
    # the zero-copy view reads the worked-example values
    vals = torch.cat([v.as_torch().reshape(2, 2, -1) for v in views], -1)
    assert vals[0, 0].tolist() == [1, 9, 4, 5, 6] and vals[1, 1].tolist() == [6, 14, 9, 10, 11]


def test_golden_error_classes_host_side():
    for c in meta()["errors"]:
        f, t = functor(c["functor"]), target(c["target"])
        arr = ArrayBuffer.from_numpy(np.zeros(c["shape"], np.float32), device="cpu")
        want = getattr(errors, c["error"]) if c["error"] else None

        def run():
            if c["op"] == "scatter":
                check_scatter_functor(f)
            views = wrap_tensors(resolve_symbolic_shape(extract_symbolic_shape(f, t), t), arr)
            if c["op"] == "concretize":
                _check_features(views, f)
            return views

        if want is None:
            run()
        elif want is errors.NonInjectiveScatterError and all(
                d.is_point for s in f.rhs for d in s.dims):
            run()  # duplicate destinations are found by the native plan compiler
        else:
            with pytest.raises(want):
                run()


def test_array_buffer_validation():
    with pytest.raises(ValueError):
        ArrayBuffer(torch.zeros(5), (2, 3), (3, 1))
    with pytest.raises(ValueError):
        ArrayBuffer(torch.zeros(6, dtype=torch.int32), (2, 3), (3, 1))
    b = ArrayBuffer(torch.arange(16, dtype=torch.float64), (4, 4), (1, 4))  # column-major
    assert b.view()[1, 0].item() == 1.0 and b.view()[0, 1].item() == 4.0
