"""Device-resident stencil driver: the reference's Fig. 2 application loop
(bench/stencil.py:101-175, `run_stencil`) with the state kept in HBM.

Every step invokes the annotated region through the public Runtime API with
the interleave schedule as the `if` clause (runtime.py:227-261,
`interleave_predicate` runtime.py:119): `if` true runs the ml(infer)
surrogate (the fused B200 kernel), false runs the application's accurate
Jacobi step -- here a device-side torch expression with the reference's
operation order (up, down, left, right, each scaled, summed left to right;
bench/stencil.py:62-76), so a `jacobi_model(0.25)` surrogate reproduces the
accurate trajectory bit for bit (criterion 3, tests/test_acceptance.py:89-110).
The t <- tnew copy and the per-step RMSE against the all-accurate trajectory
are computed on the device; the host reads the RMSE series once at the end.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from .bridge import ArrayBuffer
from .directives import parse_directive
from .runtime import BoundMap, RegionDescriptor, Runtime, interleave_predicate

__all__ = ["IN_FUNCTOR", "OUT_FUNCTOR", "jacobi_step_", "StencilRun", "run_stencil_device"]

# the reference's Fig. 2 directive set (bench/stencil.py:41-44)
IN_FUNCTOR = "functor(ifnctr: [i, j, 0:5] = (([i-1, j], [i+1, j], [i, j-1:j+2])))"
OUT_FUNCTOR = "functor(ofnctr: [i, j, 0:1] = ([i, j]))"
MAP_TO = "map(to: ifnctr(t[1:N-1, 1:M-1]))"
MAP_FROM = "map(from: ofnctr(tnew[1:N-1, 1:M-1]))"


def jacobi_step_(src: torch.Tensor, dst: torch.Tensor) -> None:
    """dst interior = 4-neighbour average of src, reference operation order;
    the boundary of dst is left as it is (fixed)."""
    c = torch.tensor(0.25, dtype=src.dtype, device=src.device)
    dst[1:-1, 1:-1] = src[:-2, 1:-1] * c + src[2:, 1:-1] * c + src[1:-1, :-2] * c + src[1:-1, 2:] * c


@dataclass
class StencilRun:
    per_step_rmse: List[float]
    surrogate_calls: int
    accurate_calls: int
    final: torch.Tensor


def run_stencil_device(field0: torch.Tensor, steps: int, model_path: str,
                       interleave: Tuple[int, int] = (0, 1), runtime: Optional[Runtime] = None) -> StencilRun:
    """`field0` [n, m] f32 on a CUDA device.  interleave = (n_accurate,
    n_surrogate) as in the reference's BenchConfig.interleave."""
    n, m = field0.shape
    dev = field0.device
    t = field0.clone().reshape(-1)
    tnew = field0.clone().reshape(-1)
    t2, tnew2 = t.view(n, m), tnew.view(n, m)
    # the all-accurate reference trajectory, on the device
    ref = field0.clone()
    ref_next = field0.clone()

    env = {"N": n, "M": m}
    tb = ArrayBuffer(t, (n, m), (m, 1))
    tnb = ArrayBuffer(tnew, (n, m), (m, 1))
    desc = RegionDescriptor(
        name="stencil", accurate_fn=lambda: jacobi_step_(t2, tnew2),
        ml=parse_directive(f'ml(infer) in(t) out(tnew) model("{model_path}") if(interleave_schedule)'),
        in_maps=[BoundMap(parse_directive(IN_FUNCTOR), parse_directive(MAP_TO, env).targets[0], tb)],
        out_maps=[BoundMap(parse_directive(OUT_FUNCTOR), parse_directive(MAP_FROM, env).targets[0], tnb)],
        env=env)
    own = runtime is None
    rt = runtime or Runtime(device=dev)
    try:
        h = rt.register_region(desc)
        n_acc, n_sur = interleave
        rmse = torch.empty(steps, dtype=torch.float64, device=dev)
        for step in range(steps):
            rt.invoke_region(h, if_value=interleave_predicate(step, n_acc, n_sur))
            t.copy_(tnew)
            jacobi_step_(ref, ref_next)
            ref, ref_next = ref_next, ref
            rmse[step] = torch.sqrt(torch.mean((t2.double() - ref.double()) ** 2))
        st = rt.stats(h)
        return StencilRun(rmse.tolist(), st.surrogate_calls, st.accurate_calls, t2.clone())
    finally:
        if own:
            rt.close()
