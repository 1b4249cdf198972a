"""tcgen05 bf16 path: descriptor self-test and the fused bonds region.

Tolerances: bf16 outputs within max-abs <= 2e-2*max|ref|
and RMSE/RMS <= 1e-2 of the fp32 reference; plus a tight check against a
bf16-emulated forward pass (same quantisation points, f64 accumulation)."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


@pytest.mark.parametrize("K,N", [(16, 256), (16, 128), (64, 128), (256, 128), (128, 256)])
def test_selftest_gemm(cuda, K, N):
    rng = np.random.default_rng(K * 1000 + N)
    A = rng.normal(size=(128, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    D = _native.tc_selftest(A, B)
    want = bf16(A) @ bf16(B).T
    assert np.max(np.abs(D - want)) <= 1e-4 * max(1.0, np.abs(want).max()), np.abs(D - want).max()


@pytest.mark.parametrize("K,N", [(64, 128), (256, 128), (128, 64), (64, 256)])
def test_selftest_gemm_tmem_a(cuda, K, N):
    rng = np.random.default_rng(K * 7 + N)
    A = rng.normal(size=(128, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    D = _native.tc_selftest(A, B, tmem_a=True)
    want = bf16(A) @ bf16(B).T
    assert np.max(np.abs(D - want)) <= 1e-4 * max(1.0, np.abs(want).max()), np.abs(D - want).max()


def emulate_bf16(layers, x):
    """bf16 operands, f32-ish accumulation, bf16 hidden re-quantisation of
    layer-1 output, f32 epilogue for the last two layers (as the kernel)."""
    (w1, b1, a1), (w2, b2, a2), (w3, b3, a3) = layers
    h = bf16(x) @ bf16(w1).T + b1
    h = np.maximum(h, 0) if a1 == "relu" else h
    h = bf16(h) @ bf16(w2).T + b2
    h = np.maximum(h, 0) if a2 == "relu" else h
    return h @ w3.T.astype(np.float64) + b3


def check_tol(got, ref):
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    rmse = np.sqrt(np.mean((got - ref) ** 2)) / np.sqrt(np.mean(ref ** 2))
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert rmse <= 1e-2, rmse
    return err.max(), err.max() / scale, rmse


@pytest.mark.parametrize("n", [128, 1000, 148 * 128 * 3 + 77, 300_000])
def test_bonds_region_tolerance(cuda, tmp_path, n):
    wl = workloads.make("bonds", n)
    wl.to_device()
    h = sm.models.device_model(wl.model, cuda)
    assert _native.model_path(h) == 3  # fused tcgen05 kernel
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    got = wl.buffers["val"].to_numpy().astype(np.float64)
    ref, finite = c_oracle.mlp_f32(wl.layers, wl.arrays["bonds"])
    assert finite
    check_tol(got, ref[:, 0].astype(np.float64))
    emu = emulate_bf16(wl.layers, wl.arrays["bonds"])[:, 0]
    assert np.max(np.abs(got - emu)) <= 2e-3 * max(1.0, np.abs(emu).max())


def test_bonds_generic_gather_and_f64(cuda, tmp_path):
    """Non-dense input rows (a strided 16-feature window of a wider f64 array)
    take the plan-driven gather; f64 output array."""
    n = 5000
    rng = np.random.default_rng(7)
    wide = rng.random((n, 20))
    layers = workloads.init_weights([16, 256, 128, 1])
    m = sm.Model(16, 1, [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    sm.save_model(m, tmp_path / "m")
    arr = sm.ArrayBuffer.from_numpy(wide)
    out = sm.ArrayBuffer.zeros((n,), "f64")
    fi = sm.parse_directive("functor(w: [k, 0:16] = ([k, 2:18]))")
    fo = sm.parse_directive("functor(o: [k, 0:1] = ([k]))")
    t = sm.parse_directive(f"map(to: w(wide[0:{n}]))").targets[0]
    to = sm.parse_directive(f"map(from: o(val[0:{n}]))").targets[0]
    desc = sm.RegionDescriptor(name="g", accurate_fn=lambda: None,
                               ml=sm.parse_ml_clause(f'ml(infer) in(wide) out(val) model("{tmp_path / "m"}")'),
                               in_maps=[sm.BoundMap(fi, t, arr)], out_maps=[sm.BoundMap(fo, to, out)])
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(desc))
    x = wide[:, 2:18].astype(np.float32)
    ref, _ = c_oracle.mlp_f32(layers, x)
    check_tol(out.to_numpy(), ref[:, 0].astype(np.float64))


def test_bonds_full_size_properties(cuda, tmp_path):
    """16.8M bonds: tolerance on a strided subsample, determinism, and shard
    independence (row blocks computed separately give identical bits)."""
    wl = workloads.make("bonds")
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        h = rt.register_region(wl.descriptor(str(tmp_path / "m")))
        rt.invoke_region(h)
        first = wl.buffers["val"].data.clone()
        rt.invoke_region(h)
        assert torch.equal(first, wl.buffers["val"].data)
    idx = np.arange(0, wl.elements, 997)
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["bonds"][idx])
    check_tol(first.cpu().numpy()[idx].astype(np.float64), ref[:, 0].astype(np.float64))
    wl.buffers["val"].data.zero_()
    for r in range(4):
        with sm.Runtime(shard=(r, 4)) as rt:
            rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    assert torch.equal(first, wl.buffers["val"].data)


def test_bf16_relu_propagates_nan(cuda, tmp_path):
    """np.maximum semantics: a NaN input must surface as NonFiniteOutputError
    through both bf16 relu epilogues (cvt.relu and max.NaN)."""
    from paper_2407_18352_b200.errors import NonFiniteOutputError
    wl = workloads.make("bonds", 4096)
    wl.arrays["bonds"][1234, 3] = np.nan
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    got = wl.buffers["val"].to_numpy()
    assert np.isnan(got[1234]) and np.isfinite(np.delete(got, 1234)).all()


@pytest.mark.parametrize("env", [{"SMLRT_TC_PAIR": "1"}])
def test_bonds_kernel_variants(cuda, env):
    """The opt-in bonds CTA-pair kernel meets the same
    tolerances; each runs in a subprocess because the switches are read once."""
    import os
    import subprocess
    import sys
    code = ("import sys, pathlib, tempfile, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import test_gpu_tc as t; import paper_2407_18352_b200 as sm;"
            "from paper_2407_18352_b200 import workloads; from oracle import c_oracle;"
            "wl = workloads.make('bonds', 148 * 128 * 3 + 77); wl.to_device();"
            "d = pathlib.Path(tempfile.mkdtemp()); sm.save_model(wl.model, d / 'm');"
            "rt = sm.Runtime(); rt.invoke_region(rt.register_region(wl.descriptor(str(d / 'm'))));"
            "got = wl.buffers['val'].to_numpy().astype(np.float64);"
            "ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays['bonds']); t.check_tol(got, ref[:, 0]);"
            "emu = t.emulate_bf16(wl.layers, wl.arrays['bonds'])[:, 0];"
            "assert np.max(np.abs(got - emu)) <= 2e-3 * max(1.0, np.abs(emu).max()); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
