"""Multi-process (gloo, world size 2) coverage of the sharded region path:
each rank takes its block of sweep rows exactly as Runtime(shard=(rank,world))
does, computes it (CPU oracle stands in for the device), and the gathered
shards reproduce the single-process result bit for bit; the bench's
max-over-ranks reduction is exercised too."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_18352_b200.runtime import _shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_of_a_grid_are_whole_rows():
    """A 2-D sweep shards along axis 0: every block is whole grid rows and the
    blocks tile the sweep."""
    rows0, inner = 4094, 2046
    for world in (1, 2, 3, 8):
        blocks = [_shard_rows(rows0 * inner, (r, world), inner) for r in range(world)]
        assert blocks[0][0] == 0 and blocks[-1][1] == rows0 * inner
        for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
            assert a1 == b0
        assert all(a % inner == 0 and b % inner == 0 for a, b in blocks)


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2407_18352_b200 import workloads
    wl = workloads.make("options", n)
    r0, r1 = _shard_rows(n, (rank, world))
    y, _ = oracle.infer(wl.layers, wl.arrays["recs"][r0:r1])
    # pad to equal length for all_gather
    per = -(-n // world)
    buf = torch.zeros(per, dtype=torch.float32)
    buf[: r1 - r0] = torch.from_numpy(y[:, 0])
    parts = [torch.zeros(per, dtype=torch.float32) for _ in range(world)]
    dist.all_gather(parts, buf)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = torch.cat(parts)[:n].numpy()
        out.put((full.tobytes(), float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 4096])
def test_two_rank_shards_reassemble_bitwise(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    full_bytes, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle
    from paper_2407_18352_b200 import workloads
    wl = workloads.make("options", n)
    want, _ = oracle.infer(wl.layers, wl.arrays["recs"])
    assert full_bytes == want[:, 0].tobytes()
    assert mx == 2.0


def test_shard_rows_partition():
    for n in (1, 7, 128, 1000, 16_777_216):
        for world in (1, 2, 3, 4, 8):
            blocks = [_shard_rows(n, (r, world)) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1


def _gather_worker(rank, world, port, n, out, inner=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_18352_b200.runtime import gather_rows_to_root
    full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3)
    r0, r1 = _shard_rows(n, (rank, world), inner)
    got = gather_rows_to_root(full[r0:r1].clone(), n, (rank, world), root=world - 1, inner=inner)
    if rank == world - 1:
        out.put(got.numpy().tobytes())
    else:
        assert got is None
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world,inner", [(7, 2, 1), (1000, 3, 1), (2, 3, 1), (20, 3, 2), (130 * 10, 4, 130)])
def test_collect_rows_meet_on_the_writer_rank(n, world, inner):
    """The collect snapshots of a sharded region (uneven last block, a rank
    with no rows) reassemble in sweep order on the writer rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q, inner)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == np.arange(n * 3, dtype=np.float64).reshape(n, 3).tobytes()
