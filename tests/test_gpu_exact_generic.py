"""Fused exact region with runtime dimensions (exact_generic.cu): any small
dense MLP without a templated instantiation runs gather -> layers -> scatter
in one kernel, bitwise equal to the reference's ordered f32 arithmetic
(models.py:188-194); models too large for shared memory take the unfused
exact path (also bitwise)."""

import numpy as np
import pytest

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def run_rows(tmp_path, dims, n, act="relu", dtype=np.float32, seed=0):
    layers = workloads.init_weights(dims, act)
    model = sm.Model(dims[0], dims[-1], [sm.DenseLayer(w, b, a) for w, b, a in layers])
    x = np.random.default_rng(seed).uniform(-2, 2, (n, dims[0])).astype(dtype)
    g = dims[-1]
    xb = sm.ArrayBuffer.from_numpy(x)
    yb = sm.ArrayBuffer.zeros((n, g), "f32" if dtype == np.float32 else "f64")
    env = {"N": n}
    fi = sm.parse_directive(f"functor(fi: [k, 0:{dims[0]}] = ([k, 0:{dims[0]}]))")
    pts = ", ".join(f"[k, {j}]" for j in range(g))
    fo = sm.parse_directive(f"functor(fo: [k, 0:{g}] = ({pts}))")
    sm.save_model(model, tmp_path / "m")
    desc = sm.RegionDescriptor(
        name="g", accurate_fn=lambda: None, ml=sm.parse_ml_clause(f'ml(infer) in(x) out(y) model("{tmp_path / "m"}")'),
        in_maps=[sm.BoundMap(fi, sm.parse_directive("map(to: fi(x[0:N]))", env).targets[0], xb)],
        out_maps=[sm.BoundMap(fo, sm.parse_directive("map(from: fo(y[0:N]))", env).targets[0], yb)], env=env)
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    ref, finite = c_oracle.mlp_f32(layers, x.astype(np.float32))
    return model, yb.to_numpy(), ref, finite


@pytest.mark.parametrize("dims", [[7, 48, 24, 3], [12, 100, 100, 1], [5, 32, 32, 32, 32, 2], [20, 256, 1],
                                  [3, 10], [64, 64, 64], [1, 9, 1]])
def test_generic_exact_bitwise(cuda, tmp_path, dims):
    model, got, ref, finite = run_rows(tmp_path, dims, 10_007)
    assert finite
    assert _native.model_path(sm.models.device_model(model, cuda)) == 6
    assert np.array_equal(got, ref)


def test_generic_exact_f64_arrays(cuda, tmp_path):
    _, got, ref, _ = run_rows(tmp_path, [7, 48, 24, 3], 3001, dtype=np.float64)
    assert np.array_equal(got, ref.astype(np.float64))


def test_generic_exact_tanh(cuda, tmp_path):
    _, got, ref, _ = run_rows(tmp_path, [6, 40, 20, 2], 4001, act="tanh")
    assert np.max(np.abs(got - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())


def test_large_model_unfused_bitwise(cuda, tmp_path):
    model, got, ref, _ = run_rows(tmp_path, [16, 512, 256, 1], 3000)
    assert _native.model_path(sm.models.device_model(model, cuda)) == 2
    assert np.array_equal(got, ref)


def test_frozen_shapes_keep_templates(cuda):
    for name in ("options", "miniweather"):
        wl = workloads.make(name, 5000)
        assert _native.model_path(sm.models.device_model(wl.model, cuda)) == 1
