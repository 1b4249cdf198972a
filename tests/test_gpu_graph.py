"""Prepared regions replayed as CUDA graphs (smlrt_region_prepare/run): the
steady-state invoke_region of a device-resident region is one graph launch.
Replays must be bitwise the direct launches, report NaN/inf like them (fused
and checked commits), count their kernels, and follow input changes (the
graph holds pointers, not values)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from paper_2407_18352_b200 import _native, workloads
from paper_2407_18352_b200.errors import NonFiniteOutputError

pytestmark = pytest.mark.gpu

CASES = [("options", 5001), ("bonds", 3001), ("minibude", 2000), ("particlefilter", 40),
         ("particlefilter_bf16", 300), ("miniweather", 40 * 130)]


def _run(name, n, tmp_path, graphs, commit="fused", calls=3):
    wl = workloads.make(name, n)
    wl.to_device()
    sm.save_model(wl.model, tmp_path / name)
    _, _, _, to = wl.functors()
    with sm.Runtime(graphs=graphs, commit=commit) as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / name)))
        rt.invoke_region(h)  # first call: validation + prepare (capture)
        prepared = rt._fast[wl.spec.name][1]
        assert prepared.graphed == graphs
        n0 = _native.launch_count()
        for _ in range(calls):
            wl.buffers[to.array].data.zero_()
            rt.invoke_region(h)
        launches = _native.launch_count() - n0
    return wl, wl.buffers[to.array].to_numpy(), launches


@pytest.mark.parametrize("name,n", CASES)
def test_graph_replay_bitwise_direct(cuda, tmp_path, name, n):
    _, direct, l_direct = _run(name, n, tmp_path / "d", graphs=False)
    _, graphed, l_graph = _run(name, n, tmp_path / "g", graphs=True)
    assert graphed.tobytes() == direct.tobytes()
    assert l_graph == l_direct > 0  # every replay counts the graph's kernels


@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_graph_replay_nonfinite_and_input_changes(cuda, tmp_path, commit):
    wl = workloads.make("options", 3000)
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    recs, price = wl.buffers["recs"], wl.buffers["price"]
    with sm.Runtime(commit=commit) as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        rt.invoke_region(h)
        assert rt._fast["options"][1].graphed
        first = price.to_numpy().copy()
        # new input values, same storage: the replay reads them
        recs.data.mul_(0.5)
        rt.invoke_region(h)
        second = price.to_numpy().copy()
        assert not np.array_equal(first, second)
        recs.data.mul_(2.0)
        rt.invoke_region(h)
        assert price.to_numpy().tobytes() == first.tobytes()
        # a NaN input raises from the replay; checked commits write nothing
        recs.data[5] = float("nan")
        price.data.fill_(7.0)
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(h)
        if commit == "checked":
            assert (price.to_numpy() == 7.0).all()
        # and the status resets: the next clean replay succeeds
        recs.data[5] = 100.0
        rt.invoke_region(h)
        assert np.isfinite(price.to_numpy()).all()


def test_graph_kernel_timing(cuda, tmp_path):
    wl = workloads.make("bonds", 100_000)
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        rt.time_kernels = True
        for _ in range(3):
            rt.invoke_region(h)
        ts = rt.kernel_times()
    assert len(ts) == 3 and all(0.0 < t < 1000.0 for t in ts)
