"""ml(collect) of a sharded region: every rank of
Runtime(shard=(rank, world)) snapshots its block of sweep rows and the blocks
meet on the writer rank (collect_root), which appends the one record the
unsharded runtime would -- byte for byte -- while the other ranks write
nothing.  Two processes share cuda:0 over gloo here (one GPU in the test
box); with one GPU per rank the same code gathers device tensors over NCCL."""

import os
import socket
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N = 12


def _region(sm, db, t, tnew):
    ifn = sm.parse_directive("functor(ifn: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2]))")
    ofn = sm.parse_directive("functor(ofn: [i, j, 0:1] = ([i, j]))")
    env = {"N": N, "M": N}
    to = sm.parse_directive("map(to: ifn(t[1:N-1, 1:M-1]))", env).targets[0]
    fr = sm.parse_directive("map(from: ofn(tnew[1:N-1, 1:M-1]))", env).targets[0]

    def accurate():
        f, g = t.view(), tnew.view()
        g[1:-1, 1:-1] = f[:-2, 1:-1] * 0.25 + f[2:, 1:-1] * 0.25 + f[1:-1, :-2] * 0.25 + f[1:-1, 2:] * 0.25

    return sm.RegionDescriptor(name="jac", accurate_fn=accurate,
                               ml=sm.parse_ml_clause(f'ml(collect) in(t) out(tnew) db("{db}")'),
                               in_maps=[sm.BoundMap(ifn, to, t)], out_maps=[sm.BoundMap(ofn, fr, tnew)], env=env)


def _field(seed):
    return np.random.default_rng(seed).uniform(0, 1, (N, N)).astype(np.float32)


def _worker(rank, world, port, db, q):
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import paper_2407_18352_b200 as sm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    idx = []
    with sm.Runtime(shard=(rank, world), collect_root=0) as rt:
        for step in range(3):
            t, tnew = sm.ArrayBuffer.from_numpy(_field(step)), sm.ArrayBuffer.from_numpy(_field(99))
            h = rt.register_region(_region(sm, db, t, tnew)) if step == 0 else h
            rt._regions[h] = _region(sm, db, t, tnew)
            idx.append(rt.invoke_region(h).record_index)
    q.put((rank, idx))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_collect_matches_single_writer(cuda, tmp_path):
    import paper_2407_18352_b200 as sm
    # unsharded reference records
    ref_db = str(tmp_path / "ref.srdb")
    with sm.Runtime() as rt:
        for step in range(3):
            t, tnew = sm.ArrayBuffer.from_numpy(_field(step)), sm.ArrayBuffer.from_numpy(_field(99))
            h = rt.register_region(_region(sm, ref_db, t, tnew)) if step == 0 else h
            rt._regions[h] = _region(sm, ref_db, t, tnew)
            rt.invoke_region(h)
    db = str(tmp_path / "sharded.srdb")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3  # 10 sweep rows over 3 ranks: blocks 4 / 4 / 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, db, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(res[r] == [0, 1, 2] for r in range(world))
    for name in ("inputs.bin", "outputs.bin"):
        a = (Path(ref_db) / "regions" / "jac" / name).read_bytes()
        b = (Path(db) / "regions" / "jac" / name).read_bytes()
        assert a == b and len(a) > 0, name
    import json
    m1 = json.loads((Path(ref_db) / "manifest.json").read_text())
    m2 = json.loads((Path(db) / "manifest.json").read_text())
    r1, r2 = m1["regions"][0], m2["regions"][0]
    assert (r1["input_shape"], r1["output_shape"], r1["record_count"]) == \
        (r2["input_shape"], r2["output_shape"], r2["record_count"])
