"""C4 ParticleFilter CNN: fused window-gather conv/pool front + exact dense
tail vs the reference-composed golden and the oracle (bitwise)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from goldens import arrays
from oracle import oracle
from paper_2407_18352_b200 import _native, workloads
from paper_2407_18352_b200.models import Conv2dLayer, DenseLayer, MaxPool2dLayer, Model

pytestmark = pytest.mark.gpu


def golden_model():
    a = arrays()
    return Model(16384, 2, [Conv2dLayer(a["cnn_conv_w"], a["cnn_conv_b"], 8, 8, "relu"), MaxPool2dLayer(2),
                            DenseLayer(a["cnn_fc_W0"], a["cnn_fc_b0"], "relu"),
                            DenseLayer(a["cnn_fc_W1"], a["cnn_fc_b1"], "identity")], input_shape=(1, 128, 128))


def run(wl, tmp_path, model=None, **kw):
    sm.save_model(model or wl.model, tmp_path / "pf")
    with sm.Runtime(**kw) as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "pf"))))
    return wl.buffers["locs"].to_numpy()


def test_cnn_region_golden(cuda, tmp_path):
    a = arrays()
    wl = workloads.make("particlefilter", 3)
    wl.arrays["frames"] = a["cnn_frames"]
    wl.to_device()
    m = golden_model()
    assert _native.model_path(sm.models.device_model(m, cuda)) == 4
    got = run(wl, tmp_path, m)
    assert got.tobytes() == a["cnn_y"].tobytes()


def test_cnn_infer_dense_batch(cuda):
    a = arrays()
    x = a["cnn_frames"][:, 16:144, 16:144].reshape(3, -1)
    y = sm.infer(golden_model(), x)
    assert y.tobytes() == a["cnn_y"].tobytes()


@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_cnn_region_matches_oracle(cuda, tmp_path, commit):
    wl = workloads.make("particlefilter", 700)
    wl.to_device()
    got = run(wl, tmp_path, commit=commit)
    x = wl.arrays["frames"][:, 16:144, 16:144].reshape(700, -1)
    want, finite = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    assert finite and got.tobytes() == want.tobytes()


def test_cnn_full_size_subsample(cuda, tmp_path):
    wl = workloads.make("particlefilter")
    wl.to_device()
    got = run(wl, tmp_path)
    idx = np.arange(0, wl.elements, 61)
    x = wl.arrays["frames"][idx, 16:144, 16:144].reshape(len(idx), -1)
    want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    assert got[idx].tobytes() == want.tobytes()


def test_cnn_region_chunks_bitwise(cuda, tmp_path):
    """More frames than one 16,384-row chunk: the region runs chunk by chunk,
    bitwise the oracle across the chunk boundary."""
    n = 16384 + 123
    wl = workloads.make("particlefilter", n)
    wl.to_device()
    got = run(wl, tmp_path)
    idx = np.r_[0:40, 16360:16400, n - 40:n]
    x = wl.arrays["frames"][idx, 16:144, 16:144].reshape(len(idx), -1)
    want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    assert got[idx].tobytes() == want.tobytes()


# --------------------------------------------------------------- bf16 CNN --
# precision "bf16": the exact conv/pool front writes bf16 features, the dense
# tail runs on the tcgen05 layer chain (model_path 7).  Tolerances as every
# bf16 path: vs the fp32 oracle max-abs <= 2e-2 max|ref| and
# RMSE/RMS <= 1e-2; vs a bf16 emulation of the same quantisation points
# (bf16 features and weights, f32 accumulation, bf16 hidden activations,
# f32 last layer) max-abs <= 2e-3 max|ref|.

def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def _emulate_cnn_bf16(layers, x, input_shape=(1, 128, 128)):
    feat, _ = oracle.cnn_forward(layers[:2], x, input_shape)  # exact conv + pool
    h = _bf16(feat.reshape(len(x), -1))
    dense = layers[2:]
    for i, (_, w, b, act) in enumerate(dense):
        h = h @ _bf16(w).T + b.astype(np.float64)
        if act == "relu":
            h = np.maximum(h, 0)
        if i + 1 < len(dense):
            h = _bf16(h)
    return h


def _tol(got, ref, bound):
    err = np.abs(got.astype(np.float64) - ref)
    scale = np.abs(ref).max()
    rmse = np.sqrt(np.mean(err ** 2)) / np.sqrt(np.mean(ref ** 2))
    assert err.max() <= bound * scale, (err.max(), scale)
    return err.max() / scale, rmse


@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_cnn_bf16_region(cuda, tmp_path, commit):
    n = 700  # not a multiple of the 128-row GEMM tile
    wl = workloads.make("particlefilter_bf16", n)
    wl.to_device()
    assert _native.model_path(sm.models.device_model(wl.model, cuda)) == 7
    got = run(wl, tmp_path, commit=commit)
    x = wl.arrays["frames"][:, 16:144, 16:144].reshape(n, -1)
    want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    _, rmse = _tol(got, want.astype(np.float64), 2e-2)
    assert rmse <= 1e-2
    _tol(got, _emulate_cnn_bf16(workloads.cnn_layers(), x), 2e-3)


def test_cnn_bf16_full_size_subsample(cuda, tmp_path):
    wl = workloads.make("particlefilter_bf16")
    wl.to_device()
    got = run(wl, tmp_path)
    idx = np.r_[0:64, 16384 - 64:16384, 5000:5100]
    x = wl.arrays["frames"][idx, 16:144, 16:144].reshape(len(idx), -1)
    want, _ = oracle.cnn_forward(workloads.cnn_layers(), x, (1, 128, 128))
    _, rmse = _tol(got[idx], want.astype(np.float64), 2e-2)
    assert rmse <= 1e-2
    _tol(got[idx], _emulate_cnn_bf16(workloads.cnn_layers(), x), 2e-3)


def test_cnn_bf16_padded_tail(cuda, tmp_path):
    """A front whose feature width is not a multiple of 64 (conv 8x8 over a
    96x96 window, pool 2: 8*6*6 = 288 features, K padded to 320) and a
    3-layer tail: the K padding must read as zero in every chunk."""
    rng = np.random.default_rng(9)
    cw = rng.normal(0, 0.125, (8, 64)).astype(np.float32)
    cb = rng.normal(0, 0.1, 8).astype(np.float32)
    fc = workloads.init_weights([288, 96, 40, 3], seed=4)
    layers = [("conv2d", cw, cb, 8, "relu"), ("maxpool2d", 2)] + [("dense", w, b, a) for w, b, a in fc]
    m = Model(96 * 96, 3, [Conv2dLayer(cw, cb, 8, 8, "relu"), MaxPool2dLayer(2)] +
              [DenseLayer(w, b, a) for w, b, a in fc], precision="bf16", input_shape=(1, 96, 96))
    n = 333
    frames = rng.random((n, 100, 100), dtype=np.float32)
    wl = workloads.make("particlefilter_bf16", n)
    wl.arrays = {"frames": frames, "locs": np.zeros((n, 3), np.float32)}
    wl.spec = type(wl.spec)(**{**wl.spec.__dict__,
                              "in_functor": "functor(win: [k, 0:96, 0:96] = ([k, 2:98, 2:98]))",
                              "out_functor": "functor(loc: [k, 0:3] = ([k, 0], [k, 1], [k, 2]))"})
    wl.model = m
    wl.to_device()
    assert _native.model_path(sm.models.device_model(m, cuda)) == 7
    got = run(wl, tmp_path)
    x = frames[:, 2:98, 2:98].reshape(n, -1)
    _tol(got, _emulate_cnn_bf16(layers, x, (1, 96, 96)), 2e-3)
