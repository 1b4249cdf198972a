"""Generate golden vectors from the REFERENCE implementation.

Run in the build container (it imports /root/reference read-only; nothing
here is used at run time on the GPU box, only the committed outputs):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json (case
metadata: directive texts, shapes, expected error classes).  Every value in
them is produced by calling the reference's own code: `concretize_to`,
`scatter_from`, `infer`, `Runtime.invoke_region`, the random case generators
of its test suite (tests/helpers.py:73-124) and its bench apps.
"""

from __future__ import annotations

import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests"), str(REF / "trainer" / "src")]

import smlrt  # noqa: E402
from helpers import random_bridge_case  # noqa: E402
from smlrt.bench.options import generate_options  # noqa: E402
from smlrt.bench.stencil import initial_field  # noqa: E402
from smlrt.bridge import ArrayBuffer, Tensor, concretize_to, scatter_from  # noqa: E402
from smlrt.directives import (MapTarget, ConcreteSlice, parse_directive,  # noqa: E402
                              parse_functor_decl, pretty_print)
from smlrt.models import DenseLayer, Model, infer, jacobi_model, save_model  # noqa: E402
from smlrt.runtime import BoundMap, RegionDescriptor, Runtime  # noqa: E402
from smlrt_train.mlp import init_mlp  # noqa: E402

OUT = Path(__file__).resolve().parent
arrays: dict[str, np.ndarray] = {}
meta: dict = {"source": "reference smlrt (/root/reference/pkg) via make_golden.py"}


def target_text(t: MapTarget) -> str:
    return str(t)


def put(name, a):
    arrays[name] = np.ascontiguousarray(a)


# 1. criterion-1 corpus: 200 random functor/array cases (test_acceptance.py:50-62)
cases = []
rng = random.Random(0xB21D6E)
for i in range(200):
    f, t, arr = random_bridge_case(rng)
    got = concretize_to(f, t, arr)
    cases.append({"functor": pretty_print(f), "target": target_text(t),
                  "shape": list(arr.shape), "strides": list(arr.strides), "dtype": arr.dtype})
    put(f"c1_{i}_data", arr.data)
    put(f"c1_{i}_out", got.data)
meta["c1"] = cases

# 2. scatter locality corpus (test_bridge.py:243-271): identity functor over
#    random sweeps, sentinel -7 arrays
scases = []
rng = random.Random(99)
for i in range(20):
    f, t, arr = random_bridge_case(rng)
    ident = parse_functor_decl("ident: [" + ", ".join(f.symbols) + ", 0:1] = (["
                               + ", ".join(f.symbols) + "])")
    dst = ArrayBuffer(np.full(arr.data.shape, -7.0, dtype=arr.data.dtype), arr.shape, arr.strides)
    sweep = tuple(s.count for s in t.slices)
    payload = np.arange(int(np.prod(sweep)), dtype=arr.data.dtype).reshape(sweep + (1,))
    scatter_from(ident, t, Tensor(payload), dst)
    scases.append({"functor": pretty_print(ident), "target": target_text(t),
                   "shape": list(arr.shape), "strides": list(arr.strides), "dtype": arr.dtype})
    put(f"sc_{i}_payload", payload)
    put(f"sc_{i}_after", dst.data)
meta["scatter"] = scases

# 3. error classes the bridge raises (bridge.py:202-454)
err_cases = [
    ("f: [i, 0:1] = ([i-1])", "a[0:4]", [4], "concretize"),
    ("f: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2])", "t[1:3]", [4, 4], "concretize"),
    ("f: [i, j, 0:4] = ([i-1, j], [i+1, j], [i, j-1:j+2])", "t[1:3, 1:3]", [4, 4], "concretize"),
    ("f: [i, 0:1] = ([i, 0])", "a[0:4]", [4], "concretize"),
    ("f: [i, j, 0:5] = ([i-1, j], [i+1, j], [i, j-1:j+2])", "t[1:3, 1:3]", [4, 4], "scatter"),
    ("f: [i, 0:2] = ([i], [i+1])", "a[1:4]", [8], "scatter"),
    ("f: [i, 0:2] = ([i])", "a[1:4]", [8], "scatter"),
    ("f: [i, 0:1] = ([i+5])", "a[0:4]", [8], "scatter"),
    ("f: [i, 0:1] = ([i])", "a[0:8:2]", [8], "scatter"),
    ("f: [i, j, 0:1] = ([i, 0])", "a[0:2, 0:3]", [4, 4], "scatter"),
]
errs = []
for ftxt, ttxt, shape, op in err_cases:
    f = parse_functor_decl(ftxt)
    t = parse_directive(f"map(to: f({ttxt}))").targets[0]
    arr = ArrayBuffer.from_numpy(np.arange(int(np.prod(shape)), dtype=np.float32).reshape(shape))
    try:
        if op == "concretize":
            concretize_to(f, t, arr)
        else:
            n = int(np.prod([s.count for s in t.slices]))
            payload = np.ones(tuple(s.count for s in t.slices) + f.feature_sizes, np.float32)
            scatter_from(f, t, Tensor(payload), arr)
        errs.append({"functor": ftxt, "target": ttxt, "shape": shape, "op": op, "error": None})
    except smlrt.errors.SmlrtError as e:
        errs.append({"functor": ftxt, "target": ttxt, "shape": shape, "op": op,
                     "error": type(e).__name__})
meta["errors"] = errs

# 4. infer goldens: reference forward passes (models.py:197-224)
def frozen(dims, act="relu", seed=0):
    m = init_mlp(dims, activation=act, seed=seed)
    brng = np.random.default_rng(1)
    layers = []
    for k, (w, _) in enumerate(zip(m.weights, m.biases)):
        b = brng.normal(0.0, 0.1, size=w.shape[0]).astype(np.float32)
        a = act if k < len(m.weights) - 1 else "identity"
        layers.append(DenseLayer(w.astype(np.float32), b, a))
    return Model(dims[0], dims[-1], layers)


inf = []
irng = np.random.default_rng(2024)
models = {
    "c1_options": (frozen([5, 64, 32, 1]), None),
    "c5_weather": (frozen([36, 8, 4]), None),
    "c2_bonds": (frozen([16, 256, 128, 1]), None),
    "tanh_5_12_1": (frozen([5, 12, 1], "tanh", 1), None),
    "relu_5_16_8_1": (frozen([5, 16, 8, 1], "relu", 0), None),
    "jacobi": (jacobi_model(0.25), None),
}
for name, (m, _) in models.items():
    x = irng.uniform(-2, 2, size=(257, m.input_features)).astype(np.float32)
    if name == "c1_options":
        x = generate_options(257, seed=0)
    y = infer(m, x)
    for k, L in enumerate(m.layers):
        put(f"inf_{name}_W{k}", L.weights)
        put(f"inf_{name}_b{k}", L.bias)
    put(f"inf_{name}_x", x)
    put(f"inf_{name}_y", y)
    inf.append({"name": name, "dims": [m.input_features] + [L.out_dim for L in m.layers],
                "acts": [L.activation for L in m.layers]})
meta["infer"] = inf

# 5. end-to-end regions through the reference Runtime
with tempfile.TemporaryDirectory() as td:
    # options: 4099 records (not a tile multiple), C1 model
    m = models["c1_options"][0]
    save_model(m, Path(td) / "c1")
    recs = generate_options(4099, seed=0)
    rbuf = ArrayBuffer.from_numpy(recs.copy())
    pbuf = ArrayBuffer.zeros((4099,), "f32")
    env = {"N": 4099}
    desc = RegionDescriptor(
        name="options", accurate_fn=lambda: None,
        ml=parse_directive(f'ml(infer) in(recs) out(price) model("{td}/c1")'),
        in_maps=[BoundMap(parse_directive("functor(optin: [k, 0:5] = ([k, 0:5]))"),
                          parse_directive("map(to: optin(recs[0:N]))", env).targets[0], rbuf)],
        out_maps=[BoundMap(parse_directive("functor(optout: [k, 0:1] = ([k]))"),
                           parse_directive("map(from: optout(price[0:N]))", env).targets[0], pbuf)],
        env=env)
    with Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    put("region_options_recs", recs)
    put("region_options_price", pbuf.data)

    # stencil: jacobi(0.25) surrogate, 32x32, 100 steps, seed 7 (criterion 3)
    save_model(jacobi_model(0.25), Path(td) / "jm")
    field0 = initial_field(32, 32, 7, "f32")
    tb = ArrayBuffer.from_numpy(field0.copy())
    nb = ArrayBuffer.from_numpy(field0.copy())
    env = {"N": 32, "M": 32}
    desc = RegionDescriptor(
        name="stencil", accurate_fn=lambda: None,
        ml=parse_directive(f'ml(infer) in(t) out(tnew) model("{td}/jm")'),
        in_maps=[BoundMap(parse_directive("functor(ifnctr: [i, j, 0:5] = (([i-1, j], [i+1, j], [i, j-1:j+2])))"),
                          parse_directive("map(to: ifnctr(t[1:N-1, 1:M-1]))", env).targets[0], tb)],
        out_maps=[BoundMap(parse_directive("functor(ofnctr: [i, j, 0:1] = ([i, j]))"),
                           parse_directive("map(from: ofnctr(tnew[1:N-1, 1:M-1]))", env).targets[0], nb)],
        env=env)
    with Runtime() as rt:
        h = rt.register_region(desc)
        for _ in range(100):
            rt.invoke_region(h)
            tb.to_numpy()[:, :] = nb.to_numpy()
    put("region_stencil_field0", field0)
    put("region_stencil_final", tb.data)

    # MiniWeather-style halo functor (C5 shape) on a small grid, 36-8-4 model
    m5 = models["c5_weather"][0]
    save_model(m5, Path(td) / "c5")
    rng5 = np.random.default_rng(5)
    state = rng5.uniform(-1, 1, size=(4, 20, 24)).astype(np.float32)
    sb = ArrayBuffer.from_numpy(state.copy())
    nb5 = ArrayBuffer.zeros((4, 20, 24), "f32")
    env = {"NX": 20, "NZ": 24}
    desc = RegionDescriptor(
        name="weather", accurate_fn=lambda: None,
        ml=parse_directive(f'ml(infer) in(state) out(state_new) model("{td}/c5")'),
        in_maps=[BoundMap(parse_directive("functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))"),
                          parse_directive("map(to: halo(state[1:NX-1, 1:NZ-1]))", env).targets[0], sb)],
        out_maps=[BoundMap(parse_directive("functor(pts: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j]))"),
                           parse_directive("map(from: pts(state_new[1:NX-1, 1:NZ-1]))", env).targets[0], nb5)],
        env=env)
    with Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    put("region_weather_state", state)
    put("region_weather_new", nb5.data)

# 6. on-disk formats written by the reference: model.json/weights.bin
#    (models.py:154-185) and an SRDB database (srdb.py:163-208)
from smlrt.srdb import open_db  # noqa: E402
with tempfile.TemporaryDirectory() as td:
    save_model(models["c1_options"][0], Path(td) / "m")
    meta["model_json"] = (Path(td) / "m" / "model.json").read_text()
    put("model_weights_bin", np.frombuffer((Path(td) / "m" / "weights.bin").read_bytes(), np.uint8))
    db = open_db(Path(td) / "db", "create")
    srng = np.random.default_rng(9)
    recs = []
    for k in range(3):
        x = srng.normal(size=(2, 3, 5)).astype(np.float32)
        y = srng.normal(size=(2, 3, 1)).astype(np.float32)
        put(f"srdb_x{k}", x)
        put(f"srdb_y{k}", y)
        db.append_record("stencil", Tensor(x), Tensor(y), 1000 + k)
    db.close()
    for which in ("inputs.bin", "outputs.bin", "times.bin"):
        put("srdb_" + which.replace(".", "_"),
            np.frombuffer((Path(td) / "db" / "regions" / "stencil" / which).read_bytes(), np.uint8))
    man = json.loads((Path(td) / "db" / "manifest.json").read_text())
    for r in man["regions"]:
        r["created_utc"] = "<nondeterministic>"
    meta["srdb_manifest"] = man

# 7. CNN (ParticleFilter shape) composed from reference pieces (SURVEY.md
#    section 8(c)): concretize_to with the 8x8 patch functor -> infer 64->8 relu
#    -> numpy 2x2 maxpool -> infer 512->128 relu -> 128->2
prng = np.random.default_rng(4)
frames = prng.random((3, 160, 160), dtype=np.float32)
m_conv = frozen([64, 8, 8])  # two layers; use the first (relu) as the conv
conv_w, conv_b = m_conv.layers[0].weights, m_conv.layers[0].bias
m_fc = frozen([512, 128, 2])
patch = parse_directive("functor(pf: [f, i, j, 0:8, 0:8] = ([f, i:i+8, j:j+8]))")
ptarget = parse_directive("map(to: pf(frames[0:3, 16:137:8, 16:137:8]))").targets[0]
pt = concretize_to(patch, ptarget, ArrayBuffer.from_numpy(frames))          # (3, 16, 16, 8, 8)
conv = infer(Model(64, 8, [DenseLayer(conv_w, conv_b, "relu")]), pt.data.reshape(-1, 64))
conv = conv.reshape(3, 16, 16, 8).transpose(0, 3, 1, 2)                   # (n, c, y, x)
pooled = conv.reshape(3, 8, 8, 2, 8, 2).max(axis=(3, 5)).reshape(3, 512)
y = infer(m_fc, pooled)
put("cnn_frames", frames)
put("cnn_conv_w", conv_w)
put("cnn_conv_b", conv_b)
for k, L in enumerate(m_fc.layers):
    put(f"cnn_fc_W{k}", L.weights)
    put(f"cnn_fc_b{k}", L.bias)
put("cnn_pooled", pooled)
put("cnn_y", y)
meta["cnn"] = {"window": "frames[k, 16:144, 16:144]", "conv": [1, 8, 8, 8], "pool": 2,
               "fc": [512, 128, 2], "acts": ["relu", "relu", "identity"]}

np.savez_compressed(OUT / "golden.npz", **arrays)
(OUT / "golden.json").write_text(json.dumps(meta, indent=1) + "\n")
print(f"wrote {len(arrays)} arrays, {len(meta['c1'])} c1 cases, {len(errs)} error cases")
