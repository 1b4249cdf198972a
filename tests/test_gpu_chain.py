"""Generic bf16 tcgen05 layer chain (any dense model, any plans): every model
shape runs at bf16 -- the shape-specialised fused kernels are the fast path,
the chain the fallback (models.py:40-64 puts no restriction on widths or
depth).  Checked against the fp32 oracle with the survey's bf16 tolerance
(SURVEY.md section 8(d))."""

import numpy as np
import pytest

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def check_tol(got, ref):
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    rmse = np.sqrt(np.mean((got - ref) ** 2)) / np.sqrt(np.mean(ref ** 2))
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert rmse <= 1e-2, rmse
    return err.max() / scale, rmse


def run_rows(tmp_path, dims, n, act="relu", seed=0):
    """rows [n, F] f32 in an AoS array -> [n, G] f32 through a bf16 region."""
    layers = workloads.init_weights(dims, act)
    model = sm.Model(dims[0], dims[-1], [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, dims[0])).astype(np.float32)
    g = dims[-1]
    xb = sm.ArrayBuffer.from_numpy(x)
    yb = sm.ArrayBuffer.zeros((n, g), "f32")
    env = {"N": n}
    fi = sm.parse_directive(f"functor(fi: [k, 0:{dims[0]}] = ([k, 0:{dims[0]}]))")
    pts = ", ".join(f"[k, {j}]" for j in range(g))
    fo = sm.parse_directive(f"functor(fo: [k, 0:{g}] = ({pts}))")
    ti = sm.parse_directive("map(to: fi(x[0:N]))", env).targets[0]
    to = sm.parse_directive("map(from: fo(y[0:N]))", env).targets[0]
    sm.save_model(model, tmp_path / "m")
    desc = sm.RegionDescriptor(name="c", accurate_fn=lambda: None,
                               ml=sm.parse_ml_clause(f'ml(infer) in(x) out(y) model("{tmp_path / "m"}")'),
                               in_maps=[sm.BoundMap(fi, ti, xb)], out_maps=[sm.BoundMap(fo, to, yb)], env=env)
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    ref, finite = c_oracle.mlp_f32(layers, x)
    assert finite
    return model, yb.to_numpy().astype(np.float64), ref.astype(np.float64)


@pytest.mark.parametrize("dims", [[5, 64, 32, 1], [16, 512, 256, 1], [8, 128, 128, 128, 2], [7, 48, 24, 3],
                                  [100, 300, 5], [3, 2000, 7], [36, 8, 4], [12, 1]])
def test_chain_shapes(cuda, tmp_path, dims):
    model, got, ref = run_rows(tmp_path, dims, 20_011)
    assert _native.model_path(sm.models.device_model(model, cuda)) == 5
    check_tol(got, ref)


@pytest.mark.parametrize("act", ["tanh", "identity"])
def test_chain_activations(cuda, tmp_path, act):
    _, got, ref = run_rows(tmp_path, [9, 96, 40, 2], 5000, act)
    check_tol(got, ref)


def test_specialised_shapes_keep_fused_kernels(cuda):
    for name in ("bonds", "minibude"):
        wl = workloads.make(name, 1000)
        assert _native.model_path(sm.models.device_model(wl.model, cuda)) == 3


def test_wide_model_with_two_in_maps_falls_back_to_chain(cuda, tmp_path):
    """C3's model over two in-maps (a non-uniform plan the fused wide kernel
    does not take) runs through the chain."""
    n = 6007
    wl = workloads.make("minibude", n)
    poses = wl.arrays["poses"]
    a = np.ascontiguousarray(poses[:3]).astype(np.float32)
    b = np.ascontiguousarray(poses[3:]).astype(np.float64)
    ab, bb = sm.ArrayBuffer.from_numpy(a), sm.ArrayBuffer.from_numpy(b)
    eb = sm.ArrayBuffer.zeros((n,), "f32")
    env = {"N": n}
    fa = sm.parse_directive("functor(fa: [p, 0:3] = ([0:3, p]))")
    fb = sm.parse_directive("functor(fb: [p, 0:3] = ([0:3, p]))")
    fo = sm.parse_directive("functor(fo: [p, 0:1] = ([p]))")
    sm.save_model(wl.model, tmp_path / "m")
    desc = sm.RegionDescriptor(
        name="w2", accurate_fn=lambda: None,
        ml=sm.parse_ml_clause(f'ml(infer) in(a, b) out(e) model("{tmp_path / "m"}")'),
        in_maps=[sm.BoundMap(fa, sm.parse_directive("map(to: fa(a[0:N]))", env).targets[0], ab),
                 sm.BoundMap(fb, sm.parse_directive("map(to: fb(b[0:N]))", env).targets[0], bb)],
        out_maps=[sm.BoundMap(fo, sm.parse_directive("map(from: fo(e[0:N]))", env).targets[0], eb)], env=env)
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    ref, _ = c_oracle.mlp_f32(wl.layers, np.ascontiguousarray(poses.T))
    check_tol(eb.to_numpy().astype(np.float64), ref[:, 0].astype(np.float64))


def test_fp32_model_at_bf16_override(cuda, tmp_path):
    """Runtime(precision="bf16") on the C1 options model (an fp32 model file)."""
    wl = workloads.make("options", 30_000)
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime(precision="bf16") as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    check_tol(wl.buffers["price"].to_numpy().astype(np.float64), ref[:, 0].astype(np.float64))


def test_chain_nonfinite_raises(cuda, tmp_path):
    from paper_2407_18352_b200.errors import NonFiniteOutputError
    dims = [4, 64, 1]
    layers = workloads.init_weights(dims)
    layers[0][0][0, 0] = 3e38  # x * w overflows to inf in the first layer
    model = sm.Model(4, 1, [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    x = np.full((300, 4), 10.0, np.float32)
    xb, yb = sm.ArrayBuffer.from_numpy(x), sm.ArrayBuffer.zeros((300,), "f32")
    env = {"N": 300}
    fi = sm.parse_directive("functor(fi: [k, 0:4] = ([k, 0:4]))")
    fo = sm.parse_directive("functor(fo: [k, 0:1] = ([k]))")
    sm.save_model(model, tmp_path / "m")
    desc = sm.RegionDescriptor(
        name="nf", accurate_fn=lambda: None, ml=sm.parse_ml_clause(f'ml(infer) in(x) out(y) model("{tmp_path / "m"}")'),
        in_maps=[sm.BoundMap(fi, sm.parse_directive("map(to: fi(x[0:N]))", env).targets[0], xb)],
        out_maps=[sm.BoundMap(fo, sm.parse_directive("map(from: fo(y[0:N]))", env).targets[0], yb)], env=env)
    with sm.Runtime(commit="checked") as rt:
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(rt.register_region(desc))
    assert (yb.to_numpy() == 0).all()  # checked commit: nothing written


def test_chain_unfused_last_layer(cuda):
    """A last layer of <= 4 outputs runs in the previous GEMM's epilogue
    (EPI_DOTG: bf16 hidden activations dotted with the bf16 last-layer
    weights); SMLRT_CHAIN_FUSE_LAST=0 (read once per process) keeps it a
    GEMM of its own: the shape cases re-run in a subprocess with it off."""
    import os
    import subprocess
    import sys
    if os.environ.get("SMLRT_CHAIN_FUSE_LAST") == "0":
        pytest.skip("already the unfused run")
    env = dict(os.environ, SMLRT_CHAIN_FUSE_LAST="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k", "chain_shapes"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
