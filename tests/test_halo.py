"""Row-slab sharded MiniWeather time stepping with halo exchange (SURVEY.md
section 8(e)): T steps on world-size-2 / 3 slab decompositions reproduce the
unsharded trajectory bit for bit.

CPU tests: the slab bookkeeping and the halo exchange (gloo, two processes;
and in-process) with the CPU oracle standing in for the device region.  GPU
test: slabs stepped by the native region kernel on one B200 against the
unsharded native run and the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_18352_b200 import halo
from paper_2407_18352_b200.directives import parse_directive

NX, NZ, T = 23, 14, 4


def _field():
    from paper_2407_18352_b200 import workloads
    return np.stack([workloads._bumps(NX, NZ, k) for k in range(4)])


def _layers():
    from paper_2407_18352_b200 import workloads
    return workloads.init_weights([36, 8, 4])


def _oracle_region_fn(layers):
    """region_fn for SlabStepper: the numpy restatement of _run_surrogate on
    the slab's host tensors (test infrastructure only)."""
    from oracle import oracle
    f_in, f_out = parse_directive(halo.HALO_FUNCTOR), parse_directive(halo.PTS_FUNCTOR)

    def fn(slab):
        V, Rp2, nz = slab.cur.shape
        env = {"R": slab.rows, "NZ": nz}
        t_in = parse_directive("map(to: halo(state[1:R+1, 1:NZ-1]))", env).targets[0]
        t_out = parse_directive("map(from: pts(state_new[1:R+1, 1:NZ-1]))", env).targets[0]
        shape, st = (V, Rp2, nz), (Rp2 * nz, nz, 1)
        cur, nxt = slab.cur.numpy().reshape(-1), slab.nxt.numpy().reshape(-1)
        _, _, ok = oracle.region([(f_in, t_in, cur, shape, st)], [(f_out, t_out, nxt, shape, st)], layers)
        assert ok
    return fn


def _reference_trajectory(field, layers, steps):
    """Unsharded: one slab covering every interior row."""
    s = halo.Slab.from_global(field, 1, 0, "cpu")
    st = halo.SlabStepper(s, "", region_fn=_oracle_region_fn(layers))
    for _ in range(steps):
        st.step()
    return s.cur.numpy().copy()


def test_slab_rows_partition():
    for nx in (3, 10, 23, 4096):
        for world in (1, 2, 3, 8):
            if nx - 2 < world:
                with pytest.raises(ValueError):
                    halo.slab_rows(nx, world, 0)
                continue
            blocks = [halo.slab_rows(nx, world, r) for r in range(world)]
            assert blocks[0][0] == 1 and blocks[-1][1] == nx - 1
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_local_exchange_matches_unsharded(world):
    field, layers = _field(), _layers()
    want = _reference_trajectory(field, layers, T)
    slabs = [halo.Slab.from_global(field, world, r, "cpu") for r in range(world)]
    steppers = [halo.SlabStepper(s, "", region_fn=_oracle_region_fn(layers)) for s in slabs]
    ex = halo.LocalExchange()
    for _ in range(T):
        ex.exchange_all(slabs)
        for st in steppers:
            st.step()
    for s in slabs:
        assert np.array_equal(s.cur[:, 1:s.rows + 1].numpy(), want[:, s.g0:s.g1]), s.rank
    # the global border rows are never touched
    assert np.array_equal(slabs[0].cur[:, 0].numpy(), field[:, 0])
    assert np.array_equal(slabs[-1].cur[:, -1].numpy(), field[:, -1])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    slab = halo.Slab.from_global(_field(), world, rank, "cpu")
    st = halo.SlabStepper(slab, "", exchange=halo.HaloExchange(), region_fn=_oracle_region_fn(_layers()))
    for _ in range(T):
        st.step()
    out.put((rank, slab.g0, slab.g1, st.interior().tobytes()))
    dist.destroy_process_group()


def test_gloo_two_rank_halo_exchange_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _reference_trajectory(_field(), _layers(), T)
    for rank, g0, g1, raw in got:
        part = np.frombuffer(raw, dtype=np.float32).reshape(4, g1 - g0, NZ)
        assert np.array_equal(part, want[:, g0:g1]), rank


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3])
def test_gpu_slabs_match_oracle(cuda, tmp_path, world):
    import paper_2407_18352_b200 as sm
    field, layers = _field(), _layers()
    want = _reference_trajectory(field, layers, T)
    model = sm.Model(36, 4, [sm.DenseLayer(w, b, a) for w, b, a in layers])
    sm.save_model(model, tmp_path / "m")
    slabs = [halo.Slab.from_global(field, world, r, cuda) for r in range(world)]
    with sm.Runtime() as rt:
        steppers = [halo.SlabStepper(s, str(tmp_path / "m"), runtime=rt) for s in slabs]
        ex = halo.LocalExchange()
        for _ in range(T):
            ex.exchange_all(slabs)
            for st in steppers:
                st.step()
        for s, st in zip(slabs, steppers):
            assert np.array_equal(st.interior(), want[:, s.g0:s.g1]), s.rank


@pytest.mark.gpu
def test_gpu_two_steppers_share_a_runtime(cuda, tmp_path):
    """A second stepper over the same rank's slab (the bench's one-step parity
    check next to the timed stepper) registers its own regions: names are
    per stepper, so one Runtime holds both (a shared name would raise
    DuplicateRegionError, as the reference's registry does)."""
    import paper_2407_18352_b200 as sm
    from paper_2407_18352_b200.errors import DuplicateRegionError
    field, layers = _field(), _layers()
    want = _reference_trajectory(field, layers, 1)
    sm.save_model(sm.Model(36, 4, [sm.DenseLayer(w, b, a) for w, b, a in layers]), tmp_path / "m")
    with sm.Runtime() as rt:
        sa, sb = halo.Slab.from_global(field, 1, 0, cuda), halo.Slab.from_global(field, 1, 0, cuda)
        a = halo.SlabStepper(sa, str(tmp_path / "m"), runtime=rt)
        b = halo.SlabStepper(sb, str(tmp_path / "m"), runtime=rt, name="mw_parity")
        for st, s in ((a, sa), (b, sb)):
            st.step()
            assert np.array_equal(st.interior(), want[:, s.g0:s.g1])
        with pytest.raises(DuplicateRegionError):
            halo.SlabStepper(halo.Slab.from_global(field + 1, 1, 0, cuda), str(tmp_path / "m"), runtime=rt)
