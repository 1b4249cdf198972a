"""Runtime semantics (the reference's tests/test_runtime.py behaviours) on
device-resident arrays."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from paper_2407_18352_b200.errors import (DuplicateRegionError, MissingClauseError,
                                          MissingPredicateError, ModelLoadError,
                                          ModelShapeMismatchError, NonFiniteOutputError,
                                          UnknownRegionError)

pytestmark = pytest.mark.gpu

IF = sm.parse_directive("functor(ifnctr: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2]))")
OF = sm.parse_directive("functor(ofnctr: [i, j, 0:1] = ([i, j]))")
ENV = {"N": 6, "M": 6}
TO = sm.parse_directive("map(to: ifnctr(t[1:N-1, 1:M-1]))", ENV).targets[0]
FROM = sm.parse_directive("map(from: ofnctr(tnew[1:N-1, 1:M-1]))", ENV).targets[0]


def field(seed=0, n=6):
    return np.random.default_rng(seed).uniform(0, 1, size=(n, n)).astype(np.float32)


def jacobi_ref(f):
    c = np.float32(0.25)
    return f[:-2, 1:-1] * c + f[2:, 1:-1] * c + f[1:-1, :-2] * c + f[1:-1, 2:] * c


def make_region(mode, db=None, model=None, if_cond=None, name="stencil"):
    t = sm.ArrayBuffer.from_numpy(field())
    tnew = sm.ArrayBuffer.from_numpy(field())
    calls = []

    def accurate():
        calls.append(1)
        f, g = t.view(), tnew.view()
        c = 0.25
        g[1:-1, 1:-1] = f[:-2, 1:-1] * c + f[2:, 1:-1] * c + f[1:-1, :-2] * c + f[1:-1, 2:] * c

    clauses = [f"ml({mode})", "in(t)", "out(tnew)"]
    if db:
        clauses.append(f'db("{db}")')
    if model:
        clauses.append(f'model("{model}")')
    if if_cond:
        clauses.append(f"if({if_cond})")
    desc = sm.RegionDescriptor(name=name, accurate_fn=accurate, ml=sm.parse_ml_clause(" ".join(clauses)),
                               in_maps=[sm.BoundMap(IF, TO, t)], out_maps=[sm.BoundMap(OF, FROM, tnew)],
                               env=dict(ENV))
    return desc, t, tnew, calls


@pytest.fixture
def jdir(tmp_path):
    sm.save_model(sm.jacobi_model(0.25), tmp_path / "jm")
    return str(tmp_path / "jm")


def test_registration(cuda, tmp_path, jdir):
    desc, *_ = make_region("infer", model=jdir)
    rt = sm.Runtime()
    h = rt.register_region(desc)
    assert rt.register_region(desc) == h
    other, *_ = make_region("infer", model=jdir)
    with pytest.raises(DuplicateRegionError):
        rt.register_region(other)
    with pytest.raises(UnknownRegionError):
        rt.invoke_region("ghost")
    bad, *_ = make_region("infer", model=jdir, name="x")
    bad.in_maps = []
    with pytest.raises(MissingClauseError):
        rt.register_region(bad)


def test_lazy_model_load(cuda, tmp_path):
    desc, *_ = make_region("infer", model=str(tmp_path / "missing"))
    rt = sm.Runtime()
    h = rt.register_region(desc)
    with pytest.raises(ModelLoadError):
        rt.invoke_region(h)


def test_surrogate_replaces_accurate_and_border_untouched(cuda, jdir):
    desc, t, tnew, calls = make_region("infer", model=jdir)
    before, sentinel = t.to_numpy(), tnew.to_numpy()
    with sm.Runtime() as rt:
        out = rt.invoke_region(rt.register_region(desc))
    assert out.path_taken == "surrogate" and calls == [] and out.elapsed_infer_ns > 0
    after = tnew.to_numpy()
    assert np.array_equal(after[1:-1, 1:-1], jacobi_ref(before))  # bitwise: same op order
    for sl in (np.s_[0, :], np.s_[-1, :], np.s_[:, 0], np.s_[:, -1]):
        assert np.array_equal(after[sl], sentinel[sl])


def test_model_shape_mismatch_and_cache(cuda, tmp_path, jdir):
    bad = sm.Model(4, 1, [sm.DenseLayer(np.zeros((1, 4), np.float32), np.zeros(1, np.float32), "identity")])
    sm.save_model(bad, tmp_path / "bad")
    desc, *_ = make_region("infer", model=str(tmp_path / "bad"))
    with sm.Runtime() as rt:
        with pytest.raises(ModelShapeMismatchError):
            rt.invoke_region(rt.register_region(desc))
    desc, *_ = make_region("infer", model=jdir)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        rt.invoke_region(h)
        rt.invoke_region(h)
        assert rt.stats(h).model_loads == 1
        rt.unload_models()
        rt.invoke_region(h)
        assert rt.stats(h).model_loads == 2


def test_collect_records_bitwise(cuda, tmp_path):
    desc, t, tnew, calls = make_region("collect", db=tmp_path / "db")
    snaps = []
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        for _ in range(5):
            snaps.append(sm.concretize_to(IF, TO, t).to_numpy())
            out = rt.invoke_region(h)
            t.view().copy_(tnew.view())
        assert rt.stats(h).records == 5 and out.record_index == 4
    with sm.open_db(tmp_path / "db", "read") as db:
        recs = db.read_records("stencil")
    for r, s in zip(recs, snaps):
        assert np.array_equal(r.inputs.to_numpy(), s) and r.elapsed_ns > 0
    assert recs[0].outputs.shape == (4, 4, 1)


def test_predicated_and_if_gate(cuda, tmp_path, jdir):
    desc, _, _, calls = make_region("predicated:host", db=tmp_path / "db", model=jdir)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        paths = [rt.invoke_region(h, predicate_value=v).path_taken for v in [False, False, True, False, True]]
        st = rt.stats(h)
        with pytest.raises(MissingPredicateError):
            rt.invoke_region(h)
    assert paths == ["accurate", "accurate", "surrogate", "accurate", "surrogate"]
    assert st.records == 3 and st.surrogate_calls == 2 and len(calls) == 3
    desc, _, _, calls = make_region("infer", model=jdir, if_cond="enabled", name="gated")
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        assert rt.invoke_region(h, if_value=False).path_taken == "accurate"
        assert rt.invoke_region(h, if_value=True).path_taken == "surrogate"
        assert calls == [1]


def test_inout_snapshot_collect(cuda, tmp_path):
    state = sm.ArrayBuffer.from_numpy(np.arange(8, dtype=np.float64))
    f = sm.parse_directive("functor(f: [k, 0:1] = ([k]))")
    t = sm.parse_directive("map(to: f(state[0:8]))").targets[0]

    def double():
        state.view().mul_(2)

    desc = sm.RegionDescriptor(name="inplace", accurate_fn=double,
                               ml=sm.parse_ml_clause(f'ml(collect) inout(state) db("{tmp_path / "db"}")'),
                               inout_maps=[sm.BoundMap(f, t, state)])
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    with sm.open_db(tmp_path / "db", "read") as db:
        rec = db.read_records("inplace", 0, 1)[0]
    assert np.array_equal(rec.inputs.to_numpy()[:, 0], np.arange(8))
    assert np.array_equal(rec.outputs.to_numpy()[:, 0], 2 * np.arange(8))


def test_inout_infer_snapshot_semantics(cuda, tmp_path):
    """in == out buffer: every output computed from the pre-call state."""
    sm.save_model(sm.Model(1, 1, [sm.DenseLayer(np.array([[2.0]], np.float32), np.array([1.0], np.float32),
                                                "identity")]), tmp_path / "m")
    data = np.arange(1000, dtype=np.float32)
    state = sm.ArrayBuffer.from_numpy(data)
    f = sm.parse_directive("functor(f: [k, 0:1] = ([k]))")
    t = sm.parse_directive("map(to: f(state[0:1000]))").targets[0]
    desc = sm.RegionDescriptor(name="io", accurate_fn=lambda: None,
                               ml=sm.parse_ml_clause(f'ml(infer) inout(state) model("{tmp_path / "m"}")'),
                               inout_maps=[sm.BoundMap(f, t, state)])
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    assert np.array_equal(state.to_numpy(), data * 2 + 1)


def test_nonfinite_checked_commit_leaves_outputs(cuda, tmp_path):
    sm.save_model(sm.Model(5, 1, [sm.DenseLayer(np.full((1, 5), 1e38, np.float32), np.zeros(1, np.float32),
                                                "identity")]), tmp_path / "big")
    for commit in ("checked", "fused"):
        desc, t, tnew, _ = make_region("infer", model=str(tmp_path / "big"), name=commit)
        t.view().fill_(10.0)
        before = tnew.to_numpy()
        with sm.Runtime(commit=commit) as rt:
            with pytest.raises(NonFiniteOutputError):
                rt.invoke_region(rt.register_region(desc))
        if commit == "checked":
            assert np.array_equal(tnew.to_numpy(), before)


def test_host_buffers_end_to_end(cuda, jdir):
    """Host-resident ArrayBuffers are staged through HBM (the e2e path)."""
    f0 = field(3)
    t = sm.ArrayBuffer(torch.from_numpy(f0.reshape(-1).copy()).pin_memory(), (6, 6), (6, 1))
    tnew = sm.ArrayBuffer(torch.from_numpy(f0.reshape(-1).copy()), (6, 6), (6, 1))
    desc = sm.RegionDescriptor(name="host", accurate_fn=lambda: None,
                               ml=sm.parse_ml_clause(f'ml(infer) in(t) out(tnew) model("{jdir}")'),
                               in_maps=[sm.BoundMap(IF, TO, t)], out_maps=[sm.BoundMap(OF, FROM, tnew)])
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    got = tnew.data.numpy().reshape(6, 6)
    assert np.array_equal(got[1:-1, 1:-1], jacobi_ref(f0))
    assert np.array_equal(got[0], f0[0]) and np.array_equal(got[:, 0], f0[:, 0])


def test_stats_bounded_by_wall(cuda, jdir):
    import time
    desc, *_ = make_region("infer", model=jdir)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        t0 = time.perf_counter_ns()
        for _ in range(5):
            rt.invoke_region(h)
        wall = time.perf_counter_ns() - t0
        st = rt.stats(h)
    assert st.map_to_ns + st.map_from_ns + st.infer_ns <= wall and st.invocations == 5


def test_status_word_resets_between_calls(cuda, tmp_path, jdir):
    """The status word is reset per call on both native paths (one-call sync
    and the event-timed asynchronous path): a NonFinite call does not poison
    the next one, and both paths raise it."""
    sm.save_model(sm.Model(5, 1, [sm.DenseLayer(np.full((1, 5), 1e38, np.float32), np.zeros(1, np.float32),
                                                "identity")]), tmp_path / "big")
    bad, t, _, _ = make_region("infer", model=str(tmp_path / "big"), name="bad")
    t.view().fill_(10.0)
    good, _, _, _ = make_region("infer", model=jdir, name="good")
    for timed in (False, True):
        with sm.Runtime() as rt:
            rt.time_kernels = timed
            hb, hg = rt.register_region(bad), rt.register_region(good)
            with pytest.raises(NonFiniteOutputError):
                rt.invoke_region(hb)
            assert rt.invoke_region(hg).path_taken == "surrogate"
            with pytest.raises(NonFiniteOutputError):
                rt.invoke_region(hb)


def _small_chunks(rt):
    # exercise the chunked path at test sizes: no size floor, ~1 MB chunks
    rt.STREAM_MIN_BYTES = 0
    rt.STREAM_CHUNK_BYTES = 1 << 20
    return rt


@pytest.mark.parametrize("config,n,shard", [("bonds", 312345, None), ("bonds", 312345, (1, 3)),
                                            ("options", 312345, None), ("options_bf16", 312345, None),
                                            ("options_bf16", 312345, (2, 3)), ("minibude", 312345, None),
                                            ("minibude", 312345, (0, 2)), ("particlefilter", 601, None),
                                            ("miniweather", 130 * 300, None), ("miniweather_bf16", 130 * 300, None),
                                            ("miniweather", 130 * 300, (1, 3))])
def test_chunked_host_path_matches_device_path(cuda, tmp_path, config, n, shard):
    """Pinned host input/output over uniform 1-D plans (AoS rows, SoA columns,
    2-D windows) take the chunked three-stream path (H2D / kernel / D2H
    overlapped); results are bitwise those of the device-resident call,
    including a ragged last chunk."""
    from paper_2407_18352_b200 import workloads
    dev_wl = workloads.make(config, n)
    dev_wl.to_device()
    host_wl = workloads.make(config, n)
    host_wl.to_device(pinned_host=True)
    sm.save_model(dev_wl.model, tmp_path / "m")
    with _small_chunks(sm.Runtime(shard=shard)) as rt:
        rt.invoke_region(rt.register_region(dev_wl.descriptor(str(tmp_path / "m"))))
        hd = host_wl.descriptor(str(tmp_path / "m"), name="host")
        plans_before = len(rt._plans)
        rt.invoke_region(rt.register_region(hd))
        assert rt._side is not None, "chunked path not taken"
        assert len(rt._plans) == plans_before + 1
    _, _, _, to = dev_wl.functors()
    got = host_wl.buffers[to.array].data.numpy()
    want = dev_wl.buffers[to.array].data.cpu().numpy()
    assert np.array_equal(got, want)


def test_chunked_host_path_grid_bands(cuda, tmp_path):
    """A 2-D sweep (the halo stencil) streams in bands of grid rows: each
    band's input rows + halo and its output interior cross PCIe as strided
    boxes -- the border of the host output is never written."""
    from paper_2407_18352_b200 import workloads
    wl = workloads.make("miniweather", 130 * 300)
    wl.arrays["state_new"][:] = 7.0
    wl.to_device(pinned_host=True)
    sm.save_model(wl.model, tmp_path / "m")
    with _small_chunks(sm.Runtime()) as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        b0 = rt._staging.h2d_bytes, rt._staging.d2h_bytes
        rt.invoke_region(h)
        nx, nz = wl.arrays["state"].shape[1:]
        assert rt._staging.d2h_bytes - b0[1] == 4 * (nx - 2) * (nz - 2) * 4  # interiors only
        assert rt._staging.h2d_bytes - b0[0] < 1.2 * wl.arrays["state"].nbytes  # bands + 2 halo rows each
    out = wl.buffers["state_new"].data.numpy().reshape(wl.arrays["state"].shape)
    assert (out[:, 0, :] == 7.0).all() and (out[:, -1, :] == 7.0).all()
    assert (out[:, :, 0] == 7.0).all() and (out[:, :, -1] == 7.0).all()


def test_chunked_host_path_window_box(cuda, tmp_path):
    """A window functor's host input crosses PCIe as the windows only (one
    strided 3-D copy per chunk), not whole frames; outputs bitwise the
    device-resident call's."""
    from paper_2407_18352_b200 import workloads
    n = 300
    dev_wl = workloads.make("particlefilter", n)
    dev_wl.to_device()
    host_wl = workloads.make("particlefilter", n)
    host_wl.to_device(pinned_host=True)
    sm.save_model(dev_wl.model, tmp_path / "m")
    with _small_chunks(sm.Runtime()) as rt:
        rt.invoke_region(rt.register_region(dev_wl.descriptor(str(tmp_path / "m"))))
        h = rt.register_region(host_wl.descriptor(str(tmp_path / "m"), name="host"))
        b0 = rt._staging.h2d_bytes
        rt.invoke_region(h)
        assert rt._staging.h2d_bytes - b0 == n * 128 * 128 * 4  # the windows, not the 160x160 frames
    assert np.array_equal(host_wl.buffers["locs"].data.numpy(), dev_wl.buffers["locs"].data.cpu().numpy())


def test_chunked_host_path_size_floor(cuda, tmp_path):
    """Below STREAM_MIN_BYTES the host buffers are staged whole (per-chunk
    host overhead would outweigh the overlap)."""
    from paper_2407_18352_b200 import workloads
    wl = workloads.make("options", 100000)
    wl.to_device(pinned_host=True)
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
        assert rt._side is None


def test_chunked_host_path_nonfinite(cuda, tmp_path):
    from paper_2407_18352_b200 import workloads
    n = 100007
    wl = workloads.make("bonds", n)
    wl.to_device(pinned_host=True)
    fi, fo, ti, to = wl.functors()
    wl.buffers[ti.array].data[-16:] = float("inf")  # last row of the last chunk
    sm.save_model(wl.model, tmp_path / "m")
    with _small_chunks(sm.Runtime()) as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(h)
        assert rt._side is not None


@pytest.mark.parametrize("host", [False, True])
def test_in_and_out_maps_on_one_array_use_pre_call_state(cuda, jdir, host):
    """An in-map reading a halo and an out-map writing the interior of the SAME
    array: every output comes from the pre-call state (the reference gathers
    all rows before it scatters), so the fused epilogue must not write rows
    other CTAs still read -- the runtime stages such calls."""
    n = 2048  # many CTA waves: later rows' halos are written by earlier CTAs
    f0 = np.random.default_rng(7).uniform(0, 1, size=(n, n)).astype(np.float32)
    env = {"N": n, "M": n}
    to = sm.parse_directive("map(to: ifnctr(t[1:N-1, 1:M-1]))", env).targets[0]
    frm = sm.parse_directive("map(from: ofnctr(t[1:N-1, 1:M-1]))", env).targets[0]
    if host:
        t = sm.ArrayBuffer(torch.from_numpy(f0.reshape(-1).copy()).pin_memory(), (n, n), (n, 1))
    else:
        t = sm.ArrayBuffer.from_numpy(f0)
    desc = sm.RegionDescriptor(name="inplace", accurate_fn=lambda: None,
                               ml=sm.parse_ml_clause(f'ml(infer) in(t) out(t) model("{jdir}")'),
                               in_maps=[sm.BoundMap(IF, to, t)], out_maps=[sm.BoundMap(OF, frm, t)])
    with sm.Runtime() as rt:
        rt._side = None
        rt.STREAM_MIN_BYTES = 0
        rt.invoke_region(rt.register_region(desc))
        assert rt._side is None  # never the chunked host path
    got = (t.data.numpy() if host else t.to_numpy()).reshape(n, n)
    assert np.array_equal(got[1:-1, 1:-1], jacobi_ref(f0))
    assert np.array_equal(got[0], f0[0]) and np.array_equal(got[:, -1], f0[:, -1])


def test_aos_in_place_1d_not_chunked_and_exact(cuda, tmp_path):
    """One pinned AoS buffer read (fields 0-4) and written (field 5) by the
    same region: disjoint fields of a shared buffer are not 'shared storage'
    (element-level check), every other element is left untouched, the output
    matches the device-resident run."""
    from paper_2407_18352_b200 import workloads
    n = 50_000
    rng = np.random.default_rng(1)
    recs = rng.uniform(0.1, 1.0, (n, 6)).astype(np.float32)
    wl = workloads.make("options", 16)
    sm.save_model(wl.model, tmp_path / "m")
    env = {"N": n}
    fi = sm.parse_directive("functor(fi: [k, 0:5] = ([k, 0:5]))")
    fo = sm.parse_directive("functor(fo: [k, 0:1] = ([k, 5]))")
    ti = sm.parse_directive("map(to: fi(r[0:N]))", env).targets[0]
    tf = sm.parse_directive("map(from: fo(r[0:N]))", env).targets[0]
    outs = []
    for host in (False, True):
        if host:
            buf = sm.ArrayBuffer(torch.from_numpy(recs.reshape(-1).copy()).pin_memory(), (n, 6), (6, 1))
        else:
            buf = sm.ArrayBuffer.from_numpy(recs)
        desc = sm.RegionDescriptor(name="aos", accurate_fn=lambda: None,
                                   ml=sm.parse_ml_clause(f'ml(infer) in(r) out(r) model("{tmp_path / "m"}")'),
                                   in_maps=[sm.BoundMap(fi, ti, buf)], out_maps=[sm.BoundMap(fo, tf, buf)], env=env)
        with sm.Runtime() as rt:
            rt.STREAM_MIN_BYTES = 0
            rt.invoke_region(rt.register_region(desc))
            pin, pout = rt._plans["aos"][1], rt._plans["aos"][2]
            from paper_2407_18352_b200.runtime import _shares_storage
            assert not _shares_storage(pin, pout)
        outs.append(buf.data.numpy().reshape(n, 6).copy() if host else buf.to_numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0][:, :5], recs[:, :5])
    from oracle import oracle
    want, _ = oracle.infer(wl.layers, recs[:, :5])
    assert np.array_equal(outs[0][:, 5], want[:, 0])


@pytest.mark.parametrize("mode", ["shard", "checked_nan"])
def test_host_output_untouched_where_not_written(cuda, tmp_path, mode):
    """Host (pinned, non-chunked: below the size floor) output buffers: rows
    outside this rank's shard, or everything on a checked commit that hits a
    non-finite output, keep their host values (the device mirror is
    downloaded whole, so it must be uploaded first)."""
    from paper_2407_18352_b200 import workloads
    n = 10_000
    wl = workloads.make("options", n)
    wl.to_device(pinned_host=True)
    _, _, ti, to = wl.functors()
    wl.buffers[to.array].data[:] = 123.0
    if mode == "checked_nan":
        wl.buffers[ti.array].data[7] = float("nan")
    sm.save_model(wl.model, tmp_path / "m")
    rt = sm.Runtime(shard=(1, 2)) if mode == "shard" else sm.Runtime(commit="checked")
    with rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        if mode == "shard":
            rt.invoke_region(h)
        else:
            with pytest.raises(NonFiniteOutputError):
                rt.invoke_region(h)
    out = wl.buffers[to.array].data.numpy()
    if mode == "shard":
        half = (n + 1) // 2
        assert (out[:half] == 123.0).all() and not (out[half:] == 123.0).any()
    else:
        assert (out == 123.0).all()


def test_prepared_fast_path(cuda, tmp_path, jdir):
    """Steady-state calls reuse the prepared native call; a new array bound to
    the descriptor, a NaN input and unload_models all behave as on the first
    call."""
    desc, t, tnew, _ = make_region("infer", model=jdir)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        rt.invoke_region(h)
        assert "stencil" in rt._fast
        for _ in range(3):
            rt.invoke_region(h)
        assert np.array_equal(tnew.to_numpy()[1:-1, 1:-1], jacobi_ref(t.to_numpy()))
        # rebind the input to a different array
        t2 = sm.ArrayBuffer.from_numpy(field(5))
        desc.in_maps[0] = sm.BoundMap(IF, TO, t2)
        rt.invoke_region(h)
        assert np.array_equal(tnew.to_numpy()[1:-1, 1:-1], jacobi_ref(t2.to_numpy()))
        t2.data[7] = float("nan")
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(h)
        t2.data[7] = 0.5
        rt.unload_models()
        rt.invoke_region(h)
        assert rt.stats(h).model_loads == 2
        assert np.array_equal(tnew.to_numpy()[1:-1, 1:-1], jacobi_ref(t2.to_numpy()))
