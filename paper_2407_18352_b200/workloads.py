"""The frozen benchmark configurations as runnable
regions: synthetic application arrays, the directive texts, and
random-init model weights.

Weights follow the survey's recipe: He (relu) / Glorot-style normal init from
`numpy.random.default_rng(seed=0)` drawn layer by layer (the distribution of
smlrt_train.mlp.init_mlp, trainer/src/smlrt_train/mlp.py:94-103), cast to
f32, biases N(0, 0.1) from `default_rng(1)`.  Data generators are seeded per
config.  `scale` shrinks the sweep for parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .bridge import ArrayBuffer
from .directives import parse_directive
from .models import Conv2dLayer, DenseLayer, MaxPool2dLayer, Model
from .runtime import BoundMap, RegionDescriptor

__all__ = ["CONFIGS", "Workload", "make", "init_weights"]

# (lo, hi) ranges of the Binomial Options records (bench/options.py:42-48)
_OPT_RANGES = ((50.0, 150.0), (50.0, 150.0), (0.2, 2.0), (0.01, 0.1), (0.1, 0.6))


@dataclass
class Spec:
    name: str
    elements: int
    dims: list
    precision: str
    in_functor: str
    out_functor: str
    map_to: str
    map_from: str
    bound: str          # roofline bound: "hbm" | "tensor" | "fp32"
    bytes_per_elem: int  # compulsory HBM bytes per element (section 8(d))
    notes: str = ""
    flops: int = 0        # override for non-MLP models

    @property
    def cnn(self) -> bool:
        return self.name.startswith("particlefilter")

    @property
    def flops_per_elem(self) -> int:
        return self.flops or 2 * sum(a * b for a, b in zip(self.dims, self.dims[1:]))


CONFIGS = {
    "options": Spec("options", 1_000_000, [5, 64, 32, 1], "fp32",
                    "functor(optin: [k, 0:5] = ([k, 0:5]))", "functor(optout: [k, 0:1] = ([k]))",
                    "map(to: optin(recs[0:N]))", "map(from: optout(price[0:N]))", "fp32", 24),
    # the same region at bf16: all three layers on warp-level tensor-core MMAs
    "options_bf16": Spec("options_bf16", 1_000_000, [5, 64, 32, 1], "bf16",
                         "functor(optin: [k, 0:5] = ([k, 0:5]))", "functor(optout: [k, 0:1] = ([k]))",
                         "map(to: optin(recs[0:N]))", "map(from: optout(price[0:N]))", "hbm", 24),
    "bonds": Spec("bonds", 16_777_216, [16, 256, 128, 1], "bf16",
                  "functor(bin: [k, 0:16] = ([k, 0:16]))", "functor(bout: [k, 0:1] = ([k]))",
                  "map(to: bin(bonds[0:N]))", "map(from: bout(val[0:N]))", "tensor", 68),
    "minibude": Spec("minibude", 67_108_864, [6, 1024, 512, 256, 1], "bf16",
                     "functor(pin: [p, 0:6] = ([0:6, p]))", "functor(pout: [p, 0:1] = ([p]))",
                     "map(to: pin(poses[0:N]))", "map(from: pout(energy[0:N]))", "tensor", 28),
    # conv 8x8/8 1->8 relu, maxpool 2, FC 512->128 relu, FC 128->2 (Table IV PF);
    # flops 2*(256*8*64 + 512*128 + 128*2) = 393,728; bytes 128*128*4 + 2*4
    "particlefilter": Spec("particlefilter", 16_384, [16384, 512, 128, 2], "fp32",
                           "functor(win: [k, 0:128, 0:128] = ([k, 16:144, 16:144]))",
                           "functor(loc: [k, 0:2] = ([k, 0], [k, 1]))",
                           "map(to: win(frames[0:N]))", "map(from: loc(locs[0:N]))", "hbm", 65_544,
                           flops=393_728),
    # the same CNN at bf16: exact conv front, dense tail on the tensor core
    "particlefilter_bf16": Spec("particlefilter_bf16", 16_384, [16384, 512, 128, 2], "bf16",
                                "functor(win: [k, 0:128, 0:128] = ([k, 16:144, 16:144]))",
                                "functor(loc: [k, 0:2] = ([k, 0], [k, 1]))",
                                "map(to: win(frames[0:N]))", "map(from: loc(locs[0:N]))", "hbm", 65_544,
                                flops=393_728),
    "miniweather": Spec("miniweather", 4094 * 2046, [36, 8, 4], "fp32",
                        "functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))",
                        "functor(pts: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j]))",
                        "map(to: halo(state[1:NX-1, 1:NZ-1]))",
                        "map(from: pts(state_new[1:NX-1, 1:NZ-1]))", "hbm", 32),
    # the same region at bf16: layer 1 on tcgen05 (stencil kernel), HBM-bound
    "miniweather_bf16": Spec("miniweather_bf16", 4094 * 2046, [36, 8, 4], "bf16",
                             "functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))",
                             "functor(pts: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j]))",
                             "map(to: halo(state[1:NX-1, 1:NZ-1]))",
                             "map(from: pts(state_new[1:NX-1, 1:NZ-1]))", "hbm", 32),
}


def init_weights(dims, act="relu", seed=0, bias_seed=1):
    rng = np.random.default_rng(seed)
    ws = []
    for fi, fo in zip(dims, dims[1:]):
        scale = np.sqrt(2.0 / fi) if act == "relu" else np.sqrt(1.0 / fi)
        ws.append(rng.normal(0.0, scale, size=(fo, fi)).astype(np.float32))
    brng = np.random.default_rng(bias_seed)
    bs = [brng.normal(0.0, 0.1, size=fo).astype(np.float32) for fo in dims[1:]]
    acts = [act] * (len(dims) - 2) + ["identity"]
    return list(zip(ws, bs, acts))


def _bumps(n, m, seed):
    """Smooth field: two seeded Gaussian bumps (bench/stencil.py:47-59 style)."""
    rng = np.random.default_rng(seed)
    rows = np.arange(n, dtype=np.float64)[:, None]
    cols = np.arange(m, dtype=np.float64)[None, :]
    f = np.zeros((n, m))
    for _ in range(2):
        r0, c0 = rng.uniform(0.2, 0.8) * (n - 1), rng.uniform(0.2, 0.8) * (m - 1)
        amp, w = rng.uniform(0.5, 1.0), rng.uniform(0.08, 0.2) * max(n, m)
        f += amp * np.exp(-((rows - r0) ** 2 + (cols - c0) ** 2) / (2 * w * w))
    return f.astype(np.float32)


@dataclass
class Workload:
    spec: Spec
    elements: int
    arrays: dict            # name -> host numpy array (logical shape)
    env: dict
    layers: list            # [(W, b, act)]
    model: Model = None
    buffers: dict = field(default_factory=dict)

    def functors(self):
        s = self.spec
        return (parse_directive(s.in_functor), parse_directive(s.out_functor),
                parse_directive(s.map_to, self.env).targets[0],
                parse_directive(s.map_from, self.env).targets[0])

    def to_device(self, device="cuda", pinned_host=False):
        """ArrayBuffers over device (or pinned host) copies of the arrays."""
        self.buffers = {}
        for k, a in self.arrays.items():
            t = torch.from_numpy(np.ascontiguousarray(a).reshape(-1))
            t = t.pin_memory() if pinned_host else t.to(device)
            strides = tuple(int(np.prod(a.shape[i + 1:])) for i in range(a.ndim))
            self.buffers[k] = ArrayBuffer(t, a.shape, strides)
        return self.buffers

    def descriptor(self, model_path, name=None):
        fi, fo, ti, to = self.functors()
        out_name = to.array
        return RegionDescriptor(
            name=name or self.spec.name, accurate_fn=lambda: None,
            ml=parse_directive(f'ml(infer) in({ti.array}) out({out_name}) model("{model_path}")'),
            in_maps=[BoundMap(fi, ti, self.buffers[ti.array])],
            out_maps=[BoundMap(fo, to, self.buffers[out_name])], env=self.env)


def cnn_layers(seed=0):
    """ParticleFilter CNN weights: conv as a 64->8 dense (He init), FC 512-128-2."""
    (cw, cb, _), _ = init_weights([64, 8, 8], seed=seed)
    fc = init_weights([512, 128, 2], seed=seed + 1)
    return [("conv2d", cw, cb, 8, "relu"), ("maxpool2d", 2)] + [("dense", w, b, a) for w, b, a in fc]


def make(name: str, elements: int | None = None, seed_offset: int = 0) -> Workload:
    s = CONFIGS[name]
    if s.cnn:
        layers = cnn_layers()
        model = Model(16384, 2, [Conv2dLayer(layers[0][1], layers[0][2], 8, 8, "relu"),
                                 MaxPool2dLayer(2)] + [DenseLayer(w, b, a) for _, w, b, a in layers[2:]],
                      precision=s.precision, input_shape=(1, 128, 128))
    else:
        layers = init_weights(s.dims)
        model = Model(s.dims[0], s.dims[-1], [DenseLayer(w, b, a) for w, b, a in layers],
                      precision=s.precision)
    if name.startswith("options"):
        n = elements or s.elements
        rng = np.random.default_rng(0 + seed_offset)
        recs = np.stack([rng.uniform(lo, hi, n) for lo, hi in _OPT_RANGES], 1).astype(np.float32)
        arrays, env = {"recs": recs, "price": np.zeros(n, np.float32)}, {"N": n}
    elif name == "bonds":
        n = elements or s.elements
        rng = np.random.default_rng(2 + seed_offset)
        arrays = {"bonds": rng.random((n, 16), dtype=np.float32), "val": np.zeros(n, np.float32)}
        env = {"N": n}
    elif name == "minibude":
        n = elements or s.elements
        rng = np.random.default_rng(3 + seed_offset)
        poses = (rng.random((6, n), dtype=np.float32) * 2 - 1).astype(np.float32)
        arrays, env = {"poses": poses, "energy": np.zeros(n, np.float32)}, {"N": n}
    elif s.cnn:
        n = elements or s.elements
        rng = np.random.default_rng(4 + seed_offset)
        arrays = {"frames": rng.random((n, 160, 160), dtype=np.float32), "locs": np.zeros((n, 2), np.float32)}
        env = {"N": n}
    elif name.startswith("miniweather"):
        nx, nz = (4096, 2048) if elements is None else _grid_for(elements)
        state = np.stack([_bumps(nx, nz, k + seed_offset) for k in range(4)])
        arrays = {"state": state, "state_new": np.zeros_like(state)}
        env = {"NX": nx, "NZ": nz}
        n = (nx - 2) * (nz - 2)
    else:
        raise KeyError(name)
    return Workload(s, n, arrays, env, layers, model)


def _grid_for(elements: int):
    nz = 2048 if elements >= 4096 * 64 else 132  # a 16-B multiple row pitch (TMA-able)
    nx = max(3, elements // (nz - 2) + 2)
    return nx, nz
