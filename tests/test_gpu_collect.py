"""ml(collect) on the GPU: the reference's acceptance criterion 4
(tests/test_acceptance.py:113-144) -- 50 records of a device-resident
stencil read back bitwise equal to an independent oracle reconstruction,
positive times, consistent manifest and payload sizes -- and the records
read through a reader written from the documented format alone, as the
trainer's read_region does (trainer/src/smlrt_train/srdb_reader.py:50-82)."""

import json
from pathlib import Path

import numpy as np
import torch

import paper_2407_18352_b200 as sm
from oracle import oracle
from paper_2407_18352_b200 import stencil

import pytest

pytestmark = pytest.mark.gpu

N = 8
STEPS = 50


def jacobi_np(f):
    """the accurate step in the reference's operation order (bench/stencil.py:62-76)"""
    c = np.float32(0.25)
    g = f.copy()
    g[1:-1, 1:-1] = f[:-2, 1:-1] * c + f[2:, 1:-1] * c + f[1:-1, :-2] * c + f[1:-1, 2:] * c
    return g


def read_region(db_path, region):
    """(inputs, outputs, elapsed_ns) from manifest.json + raw LE payloads,
    validating file lengths against the manifest first."""
    man = json.loads((Path(db_path) / "manifest.json").read_text())
    assert man["version"] == 1
    info = next(r for r in man["regions"] if r["name"] == region)
    dt = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8")}[info["dtype"]]
    count = int(info["record_count"])
    out = []
    for name, shape, d in (("inputs.bin", info["input_shape"], dt), ("outputs.bin", info["output_shape"], dt),
                           ("times.bin", [], np.dtype("<u8"))):
        path = Path(db_path) / "regions" / region / name
        want = count * int(np.prod(shape, dtype=np.int64)) * d.itemsize
        assert path.stat().st_size == want, (name, path.stat().st_size, want)
        out.append(np.fromfile(path, dtype=d).reshape((count,) + tuple(shape)))
    return out


def test_criterion_4_collection_fidelity(cuda, tmp_path):
    rng = np.random.default_rng(11)
    field0 = rng.uniform(0, 1, (N, N)).astype(np.float32)
    t = torch.from_numpy(field0.copy()).to(cuda).reshape(-1)
    tnew = t.clone()
    t2, tnew2 = t.view(N, N), tnew.view(N, N)
    env = {"N": N, "M": N}
    tb, tnb = sm.ArrayBuffer(t, (N, N), (N, 1)), sm.ArrayBuffer(tnew, (N, N), (N, 1))
    ifn, ofn = sm.parse_directive(stencil.IN_FUNCTOR), sm.parse_directive(stencil.OUT_FUNCTOR)
    to_t = sm.parse_directive(stencil.MAP_TO, env).targets[0]
    from_t = sm.parse_directive(stencil.MAP_FROM, env).targets[0]
    db = tmp_path / "db"
    desc = sm.RegionDescriptor(
        name="stencil", accurate_fn=lambda: stencil.jacobi_step_(t2, tnew2),
        ml=sm.parse_directive(f'ml(collect) in(t) out(tnew) db("{db}")'),
        in_maps=[sm.BoundMap(ifn, to_t, tb)], out_maps=[sm.BoundMap(ofn, from_t, tnb)], env=env)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        for _ in range(STEPS):
            rt.invoke_region(h)
            t.copy_(tnew)
        assert rt.stats(h).records == STEPS

    # independent reconstruction: numpy trajectory + the oracle's functor gather
    states = [field0]
    for _ in range(STEPS):
        states.append(jacobi_np(states[-1]))
    st = (N, 1)
    with sm.open_db(db, "read") as d:
        assert d.info().region("stencil").record_count == STEPS
        records = d.read_records("stencil")
    ins, outs, times = read_region(db, "stencil")
    for k in range(STEPS):
        want_in = oracle.gather(ifn, to_t, states[k].reshape(-1), (N, N), st)
        want_out = oracle.gather(ofn, to_t, states[k + 1].reshape(-1), (N, N), st)
        assert records[k].inputs.to_numpy().tobytes() == want_in.tobytes()
        assert records[k].outputs.to_numpy().tobytes() == want_out.tobytes()
        assert ins[k].tobytes() == want_in.tobytes() and outs[k].tobytes() == want_out.tobytes()
        assert records[k].elapsed_ns > 0 and times[k] > 0
    assert (db / "regions" / "stencil" / "inputs.bin").stat().st_size == STEPS * 36 * 5 * 4


def test_collect_reuses_pinned_buffers(cuda, tmp_path):
    rng = np.random.default_rng(3)
    t = sm.ArrayBuffer.from_numpy(rng.uniform(0, 1, (N, N)).astype(np.float32))
    tn = sm.ArrayBuffer.from_numpy(np.zeros((N, N), np.float32))
    env = {"N": N, "M": N}
    desc = sm.RegionDescriptor(
        name="s", accurate_fn=lambda: None,
        ml=sm.parse_directive(f'ml(collect) in(t) out(tnew) db("{tmp_path / "db"}")'),
        in_maps=[sm.BoundMap(sm.parse_directive(stencil.IN_FUNCTOR), sm.parse_directive(stencil.MAP_TO, env).targets[0], t)],
        out_maps=[sm.BoundMap(sm.parse_directive(stencil.OUT_FUNCTOR),
                              sm.parse_directive(stencil.MAP_FROM, env).targets[0], tn)], env=env)
    with sm.Runtime() as rt:
        h = rt.register_region(desc)
        rt.invoke_region(h)
        bufs = {k: v.data_ptr() for k, v in rt._pinned_bufs.items()}
        rt.invoke_region(h)
        assert {k: v.data_ptr() for k, v in rt._pinned_bufs.items()} == bufs and len(bufs) == 2
