"""Row-slab sharding of the MiniWeather halo region, iterated in time.

SURVEY.md section 8(e): the C5 grid `state[V, NX, NZ]` is split into
contiguous blocks of interior rows, one per rank; every rank owns a slab
`[V, R + 2, NZ]` holding its R interior rows plus one halo row on each side.
A time step is

    exchange halo rows with ranks r - 1 and r + 1   (one grouped send/recv)
    ml(infer) region  state[1:R+1, 1:NZ-1] -> state_new[1:R+1, 1:NZ-1]
    swap state / state_new

which is exactly the reference's stencil time loop (bench/stencil.py:135-155
drives Runtime.invoke_region per step with the t/tnew swap) restricted to a
slab: the region reads each point's 3x3 neighbourhood of the pre-step state
(snapshot semantics, runtime.py:311-358) and never writes the global border
rows/columns, so a sharded run is bitwise equal to the unsharded one.

The exchange goes through `torch.distributed` point-to-point operations
(`batch_isend_irecv`: NCCL over NVLink between GPUs, gloo on CPU for the
tests); it is the only collective traffic and sits between region launches,
never on the data path inside one.  `LocalExchange` performs the same copies
between slabs that live in one process (one GPU, or tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from .bridge import ArrayBuffer
from .directives import parse_directive
from .runtime import BoundMap, RegionDescriptor, Runtime

__all__ = ["slab_rows", "HaloExchange", "LocalExchange", "Slab", "SlabStepper", "HALO_FUNCTOR", "PTS_FUNCTOR"]

HALO_FUNCTOR = "functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))"
PTS_FUNCTOR = "functor(pts: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j]))"


def slab_rows(nx: int, world: int, rank: int) -> tuple:
    """Global interior rows [g0, g1) of `rank` when rows 1 .. nx-2 are split
    into `world` contiguous blocks (the first nx-2 mod world blocks one row
    longer)."""
    n = nx - 2
    if n < world:
        raise ValueError(f"{n} interior rows cannot be split over {world} ranks")
    base, extra = divmod(n, world)
    g0 = 1 + rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


@dataclass
class Slab:
    """One rank's rows: `cur` / `nxt` are [V, R + 2, NZ] tensors whose row 0
    and row R + 1 are halos (or the fixed global border at the grid's edge)."""
    rank: int
    world: int
    g0: int
    g1: int
    cur: torch.Tensor
    nxt: torch.Tensor

    @property
    def rows(self) -> int:
        return self.g1 - self.g0

    def swap(self):
        self.cur, self.nxt = self.nxt, self.cur

    @staticmethod
    def from_global(state: np.ndarray, world: int, rank: int, device) -> "Slab":
        """Cut rank's slab (with its halo / border rows) out of a global field."""
        g0, g1 = slab_rows(state.shape[1], world, rank)
        part = np.array(state[:, g0 - 1:g1 + 1, :], copy=True)  # never alias the caller's field
        cur = torch.from_numpy(part).to(device)
        return Slab(rank, world, g0, g1, cur, cur.clone())


class HaloExchange:
    """+-1-row halo exchange with the neighbouring ranks of a process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self._buf = {}

    def _tmp(self, key, like):
        t = self._buf.get(key)
        if t is None or t.shape != like.shape or t.device != like.device or t.dtype != like.dtype:
            t = torch.empty_like(like)
            self._buf[key] = t
        return t

    def exchange(self, slab: Slab) -> None:
        dist = self.dist
        r, w, R = slab.rank, slab.world, slab.rows
        s = slab.cur
        ops, back = [], []
        if r > 0:
            snd = self._tmp("s_up", s[:, 1, :])
            snd.copy_(s[:, 1, :])
            rcv = self._tmp("r_up", s[:, 0, :])
            ops += [dist.P2POp(dist.isend, snd, r - 1, self.group), dist.P2POp(dist.irecv, rcv, r - 1, self.group)]
            back.append((s[:, 0, :], rcv))
        if r < w - 1:
            snd = self._tmp("s_dn", s[:, R, :])
            snd.copy_(s[:, R, :])
            rcv = self._tmp("r_dn", s[:, R + 1, :])
            ops += [dist.P2POp(dist.isend, snd, r + 1, self.group), dist.P2POp(dist.irecv, rcv, r + 1, self.group)]
            back.append((s[:, R + 1, :], rcv))
        if ops and dist.get_backend(self.group) == "gloo" and s.is_cuda:
            # gloo moves host tensors: stage the halo rows through the host
            host = [op.tensor.cpu() if op.op is dist.isend else torch.empty(op.tensor.shape, dtype=op.tensor.dtype)
                    for op in ops]
            ops = [dist.P2POp(op.op, h, op.peer, self.group) for op, h in zip(ops, host)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            recvd = [h for op, h in zip(ops, host) if op.op is dist.irecv]
            for (dst, _), h in zip(back, recvd):
                dst.copy_(h)
            return
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for dst, src in back:
            dst.copy_(src)


class LocalExchange:
    """The same halo copies between slabs held by one process."""

    def exchange_all(self, slabs: Sequence[Slab]) -> None:
        # read every boundary row before writing any halo (all from the pre-step state)
        ups = [s.cur[:, 1, :].clone() for s in slabs]
        dns = [s.cur[:, s.rows, :].clone() for s in slabs]
        for k, s in enumerate(slabs):
            if k > 0:
                s.cur[:, 0, :].copy_(dns[k - 1].to(s.cur.device))
            if k < len(slabs) - 1:
                s.cur[:, s.rows + 1, :].copy_(ups[k + 1].to(s.cur.device))


class SlabStepper:
    """Time-steps one slab with the ml(infer) region on the B200 runtime.

    Two region descriptors (cur -> nxt and nxt -> cur) are registered once
    (names `{name}{rank}_{0,1}`: unique per Runtime), so plans and the model
    stay cached across steps; `step()` = exchange + invoke + swap.  `region_fn(slab)` replaces the invoke for tests that step
    with the CPU oracle (no CUDA device)."""

    def __init__(self, slab: Slab, model_path: str, runtime: Optional[Runtime] = None,
                 exchange: Optional[HaloExchange] = None,
                 region_fn: Optional[Callable[[Slab], None]] = None, name: str = "mw_slab"):
        self.slab = slab
        self.exchange = exchange
        self.region_fn = region_fn
        self.rt = runtime
        self._handles: List[str] = []
        if region_fn is None:
            if runtime is None:
                raise ValueError("SlabStepper needs a Runtime (or a region_fn)")
            V, Rp2, NZ = slab.cur.shape
            env = {"R": slab.rows, "NZ": NZ}
            f_in, f_out = parse_directive(HALO_FUNCTOR), parse_directive(PTS_FUNCTOR)
            t_in = parse_directive("map(to: halo(state[1:R+1, 1:NZ-1]))", env).targets[0]
            t_out = parse_directive("map(from: pts(state_new[1:R+1, 1:NZ-1]))", env).targets[0]
            strides = (Rp2 * NZ, NZ, 1)
            bufs = [ArrayBuffer(t.reshape(-1), tuple(slab.cur.shape), strides) for t in (slab.cur, slab.nxt)]
            ml = parse_directive(f'ml(infer) in(state) out(state_new) model("{model_path}")')
            for k in range(2):
                desc = RegionDescriptor(
                    name=f"{name}{slab.rank}_{k}", accurate_fn=lambda: None, ml=ml,
                    in_maps=[BoundMap(f_in, t_in, bufs[k])], out_maps=[BoundMap(f_out, t_out, bufs[1 - k])],
                    env=env)
                self._handles.append(runtime.register_region(desc))
        self._parity = 0

    def step(self) -> None:
        if self.exchange is not None:
            self.exchange.exchange(self.slab)
        if self.region_fn is not None:
            self.region_fn(self.slab)
        else:
            self.rt.invoke_region(self._handles[self._parity])
        self.slab.swap()
        self._parity ^= 1

    def interior(self) -> np.ndarray:
        """This slab's interior rows of the current state, [V, R, NZ] (host)."""
        return self.slab.cur[:, 1:self.slab.rows + 1, :].cpu().numpy()
