"""Pin the oracle (oracle/) against golden vectors the reference produced."""

import numpy as np
import pytest

from goldens import arrays, case, infer_layers, meta, functor, target
from oracle import c_oracle, oracle


def test_c1_corpus_gather_bitwise():
    a = arrays()
    for i in range(len(meta()["c1"])):
        f, t, c = case("c1", i)
        got = oracle.gather(f, t, a[f"c1_{i}_data"], c["shape"], c["strides"])
        want = a[f"c1_{i}_out"]
        assert got.dtype == want.dtype and got.tobytes() == want.tobytes(), i


def test_scatter_corpus_bitwise():
    a = arrays()
    for i in range(len(meta()["scatter"])):
        f, t, c = case("scatter", i)
        dt = np.float32 if c["dtype"] == "f32" else np.float64
        data = np.full(a[f"sc_{i}_after"].shape, -7.0, dtype=dt)
        oracle.scatter(f, t, a[f"sc_{i}_payload"], data, c["shape"], c["strides"])
        assert data.tobytes() == a[f"sc_{i}_after"].tobytes(), i


def test_error_cases_raise():
    for c in meta()["errors"]:
        f, t = functor(c["functor"]), target(c["target"])
        data = np.arange(int(np.prod(c["shape"])), dtype=np.float32)
        strides = [int(np.prod(c["shape"][k + 1:])) for k in range(len(c["shape"]))]

        def run():
            if c["op"] == "concretize":
                oracle.gather(f, t, data, c["shape"], strides)
            else:
                vals = np.ones((int(np.prod([s.count for s in t.slices])), f.feature_count), np.float32)
                if len(f.rhs) != f.feature_count:
                    raise ValueError("feature mismatch")
                oracle.scatter(f, t, vals, data, c["shape"], strides)

        if c["error"] is None:
            run()
        elif c["error"] in ("ArityMismatchError", "FeatureMismatchError") and c["op"] == "concretize":
            # feature/arity checks live in the bridge, not in the address oracle
            with pytest.raises(Exception):
                got = oracle.gather(f, t, data, c["shape"], strides)
                assert got.shape[-len(f.feature_sizes):] == f.feature_sizes
        else:
            with pytest.raises((IndexError, ValueError)):
                run()


@pytest.mark.parametrize("name", [m["name"] for m in meta()["infer"]])
def test_infer_goldens(name):
    layers, x, y = infer_layers(name)
    got, finite = oracle.infer(layers, x)
    assert finite
    if any(a == "tanh" for _, _, a in layers):
        assert np.max(np.abs(got - y)) <= 1e-6
    else:
        assert got.tobytes() == y.tobytes()


@pytest.mark.skipif(not c_oracle.available(), reason="oracle/build/liboracle.so not built")
@pytest.mark.parametrize("name", [m["name"] for m in meta()["infer"]])
def test_c_oracle_infer_goldens(name):
    layers, x, y = infer_layers(name)
    got, finite = c_oracle.mlp_f32(layers, x, threads=3)
    assert finite
    if any(a == "tanh" for _, _, a in layers):
        assert np.max(np.abs(got - y)) <= 1e-5
    else:
        assert got.tobytes() == y.tobytes()


def test_overflow_not_finite():
    layers = [(np.array([[2.0]], np.float32), np.zeros(1, np.float32), "identity")]
    _, finite = oracle.infer(layers, np.full((1, 1), 3e38, np.float32))
    assert not finite


def _options_maps(recs, price):
    n = recs.shape[0]
    fi = functor("functor(optin: [k, 0:5] = ([k, 0:5]))")
    fo = functor("functor(optout: [k, 0:1] = ([k]))")
    return ([(fi, target(f"recs[0:{n}]"), recs.reshape(-1), recs.shape, (5, 1))],
            [(fo, target(f"price[0:{n}]"), price, (n,), (1,))])


def test_region_options_golden():
    a = arrays()
    layers, _, _ = infer_layers("c1_options")
    recs = a["region_options_recs"]
    price = np.zeros(recs.shape[0], np.float32)
    ins, outs = _options_maps(recs, price)
    oracle.region(ins, outs, layers)
    assert price.tobytes() == a["region_options_price"].tobytes()


def test_region_stencil_trajectory_golden():
    a = arrays()
    jac = [(np.array([[0.25, 0.25, 0.25, 0.0, 0.25]], np.float32), np.zeros(1, np.float32), "identity")]
    t = a["region_stencil_field0"].copy()
    fi = functor("functor(ifnctr: [i, j, 0:5] = (([i-1, j], [i+1, j], [i, j-1:j+2])))")
    fo = functor("functor(ofnctr: [i, j, 0:1] = ([i, j]))")
    tg = target("t[1:31, 1:31]")
    for _ in range(100):
        tnew = t.copy().reshape(-1)
        oracle.region([(fi, tg, t.reshape(-1), (32, 32), (32, 1))],
                      [(fo, tg, tnew, (32, 32), (32, 1))], jac)
        t = tnew.reshape(32, 32)
    assert t.tobytes() == a["region_stencil_final"].tobytes()


def test_region_weather_golden():
    a = arrays()
    layers, _, _ = infer_layers("c5_weather")
    state = a["region_weather_state"]
    new = np.zeros(state.size, np.float32)
    fi = functor("functor(halo: [i, j, 0:4, 0:3, 0:3] = ([0:4, i-1:i+2, j-1:j+2]))")
    fo = functor("functor(pts: [i, j, 0:4] = ([0, i, j], [1, i, j], [2, i, j], [3, i, j]))")
    tg = target("state[1:19, 1:23]")
    oracle.region([(fi, tg, state.reshape(-1), (4, 20, 24), (480, 24, 1))],
                  [(fo, tg, new, (4, 20, 24), (480, 24, 1))], layers)
    assert new.tobytes() == a["region_weather_new"].tobytes()


def test_cnn_oracle_matches_reference_composition():
    a = arrays()
    layers = [("conv2d", a["cnn_conv_w"], a["cnn_conv_b"], 8, "relu"), ("maxpool2d", 2),
              ("dense", a["cnn_fc_W0"], a["cnn_fc_b0"], "relu"),
              ("dense", a["cnn_fc_W1"], a["cnn_fc_b1"], "identity")]
    x = a["cnn_frames"][:, 16:144, 16:144].reshape(3, -1)
    y, finite = oracle.cnn_forward(layers, x, (1, 128, 128))
    assert finite and y.tobytes() == a["cnn_y"].tobytes()
