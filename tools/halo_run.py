"""Iterated MiniWeather surrogate on a row-slab-sharded 4096 x 2048 grid with
NCCL halo exchange (paper_2407_18352_b200.halo), one process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/halo_run.py [--steps 20] [--nx 4096] [--nz 2048]

Prints per-step time (CUDA events, max over ranks) split into halo exchange
and region time, and a checksum of the final field (sum over ranks) that is
identical for every N (the sharded trajectory is bitwise the unsharded one).
"""
import argparse
import json
import os
import sys
import tempfile

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_18352_b200 as sm  # noqa: E402
from paper_2407_18352_b200 import halo, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--nx", type=int, default=4096)
    ap.add_argument("--nz", type=int, default=2048)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    field = np.stack([workloads._bumps(a.nx, a.nz, k) for k in range(4)])
    layers = workloads.init_weights([36, 8, 4])
    model = sm.Model(36, 4, [sm.DenseLayer(w, b, act) for w, b, act in layers])
    tmp = tempfile.mkdtemp(prefix="halo_run_")
    sm.save_model(model, tmp)
    slab = halo.Slab.from_global(field, world, rank, dev)
    with sm.Runtime(device=dev) as rt:
        st = halo.SlabStepper(slab, tmp, runtime=rt, exchange=halo.HaloExchange() if world > 1 else None)
        st.step()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t_ex = t_reg = 0.0
        for _ in range(a.steps):
            ev[0].record()
            if st.exchange is not None:
                st.exchange.exchange(slab)
            ev[1].record()
            rt.invoke_region(st._handles[st._parity])
            slab.swap()
            st._parity ^= 1
            ev[2].record()
            torch.cuda.synchronize()
            t_ex += ev[0].elapsed_time(ev[1])
            t_reg += ev[1].elapsed_time(ev[2])
        chk = torch.tensor([float(slab.cur[:, 1:slab.rows + 1].double().sum())], dtype=torch.float64, device=dev)
        tt = torch.tensor([t_ex / a.steps, t_reg / a.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(chk)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"world": world, "grid": [a.nx, a.nz], "steps": a.steps,
                          "exchange_ms": round(float(tt[0]), 4), "region_ms": round(float(tt[1]), 4),
                          "checksum": float(chk.item())}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
