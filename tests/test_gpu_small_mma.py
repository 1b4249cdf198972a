"""Small dense MLPs at bf16 on the warp-MMA region kernel (small_mma.cu): C1
options at precision "bf16" and other 3-layer shapes F <= 8 -> H1, H2 <= 64
-> G <= 8 -- layer 1 on tf32 MMAs from the gathered f32 features, layers 2-3
on bf16 MMAs with the activations in registers -- and, for packed rows with
F <= 6, the tcgen05 small-MLP kernel (small_tc.cu: layer 1 kind::tf32 with
the bias as two K columns, layer 2 kind::f16 with its A operand in TMEM,
layer 3 on the FP32 pipe) at the same quantisation points.  Against the fp32 oracle at
the bf16 tolerance of SURVEY.md 8(d) (max-abs <= 2e-2 max|ref|, RMSE/RMS <=
1e-2) and against an emulation of its quantisation points."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads
from paper_2407_18352_b200.errors import NonFiniteOutputError

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def _tf32_trunc(a):
    return (np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(
        np.float64)


def _tf32_rne(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000).astype(np.uint32).view(np.float32).astype(np.float64)


def _act(h, a):
    return np.maximum(h, 0) if a == "relu" else (np.tanh(h) if a == "tanh" else h)


def _emulate(layers, x):
    """the kernel's quantisation points: tf32 features (truncated by the MMA)
    and tf32 W1, bf16 hidden activations, bf16 W2 and W3, f32 biases (each
    is its accumulator's initial value), f32 accumulation"""
    (w1, b1, a1), (w2, b2, a2), (w3, b3, a3) = layers
    h = _act(_tf32_trunc(x) @ _tf32_rne(w1).T + b1, a1)
    h = _act(_bf16(h) @ _bf16(w2).T + b2, a2)
    return _act(_bf16(h) @ _bf16(w3).T + b3, a3)


def _region(dims, n, act, seed=3):
    wl = workloads.make("options_bf16", n)
    layers = workloads.init_weights(dims, act=act, seed=seed)
    wl.layers = layers
    wl.model = sm.Model(dims[0], dims[-1], [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    rng = np.random.default_rng(seed)
    wl.arrays = {"recs": rng.uniform(-2, 2, (n, dims[0])).astype(np.float32),
                 "price": np.zeros((n, dims[-1]), np.float32)}
    wl.spec = type(wl.spec)(**{**wl.spec.__dict__,
                              "in_functor": f"functor(optin: [k, 0:{dims[0]}] = ([k, 0:{dims[0]}]))",
                              "out_functor": "functor(optout: [k, 0:%d] = (%s))" % (
                                  dims[-1], ", ".join(f"[k, {j}]" for j in range(dims[-1])))})
    return wl


def _run(wl, tmp_path, **kw):
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    n0 = _native.launch_count()
    with sm.Runtime(**kw) as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    return wl.buffers["price"].to_numpy().reshape(wl.arrays["price"].shape), _native.launch_count() - n0


def _check(wl, got, emulate=True):
    x = wl.arrays["recs"]
    ref, _ = c_oracle.mlp_f32(wl.layers, x)
    ref = ref.astype(np.float64)
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert np.sqrt(np.mean(err ** 2)) <= 1e-2 * np.sqrt(np.mean(ref ** 2))
    if not emulate:
        return
    emu = _emulate(wl.layers, x)
    d = np.abs(got - emu)
    assert np.sqrt(np.mean(d ** 2)) <= 1e-4 * np.sqrt(np.mean(emu ** 2)) + 1e-7
    assert d.max() <= 1.5e-2 * np.abs(emu).max()


@pytest.mark.parametrize("dims,act,n", [([5, 64, 32, 1], "relu", 100_003), ([7, 16, 16, 8], "relu", 4097),
                                        ([8, 16, 16, 8], "relu", 3000), ([8, 64, 64, 8], "tanh", 70_001),
                                        ([3, 40, 24, 3], "relu", 999), ([7, 64, 64, 2], "tanh", 2000),
                                        ([2, 9, 17, 5], "identity", 77), ([5, 64, 32, 1], "relu", 1),
                                        ([6, 64, 64, 8], "tanh", 50_001), ([4, 32, 16, 2], "identity", 3333),
                                        ([1, 16, 64, 4], "relu", 129)])
@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_small_mma_matches_oracle(cuda, tmp_path, dims, act, n, commit):
    wl = _region(dims, n, act)
    got, launches = _run(wl, tmp_path, commit=commit)
    assert launches == (1 if commit == "fused" else 2)  # one fused kernel (+ the gated scatter)
    _check(wl, got)


def test_options_bf16_config(cuda, tmp_path):
    wl = workloads.make("options_bf16", 300_001)
    got, launches = _run(wl, tmp_path)
    assert launches == 1
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    err = np.abs(got.reshape(-1, 1) - ref)
    assert err.max() <= 2e-2 * np.abs(ref).max()


@pytest.mark.parametrize("commit", ["fused", "checked"])
def test_small_mma_nonfinite(cuda, tmp_path, commit):
    wl = _region([5, 64, 32, 1], 5000, "relu")
    wl.arrays["recs"][4321, 2] = np.nan
    wl.to_device()
    sm.save_model(wl.model, tmp_path / "m")
    wl.buffers["price"].data.fill_(3.0)
    with sm.Runtime(commit=commit) as rt:
        with pytest.raises(NonFiniteOutputError):
            rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    if commit == "checked":
        assert (wl.buffers["price"].to_numpy() == 3.0).all()


def test_nine_features_use_the_chain(cuda, tmp_path):
    """F = 9 does not fit layer 1's k8 MMA: the layer chain runs it."""
    wl = _region([9, 16, 16, 8], 3000, "relu")
    got, launches = _run(wl, tmp_path)
    assert launches == 5
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()


def test_mixed_activations_use_the_chain(cuda, tmp_path):
    wl = _region([5, 32, 32, 1], 3000, "relu")
    layers = wl.layers
    layers[1] = (layers[1][0], layers[1][1], "tanh")
    wl.layers = layers
    wl.model = sm.Model(5, 1, [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    got, launches = _run(wl, tmp_path)
    assert launches == 4  # the layer chain: gather, two GEMMs (the last 32->1 in the second's epilogue), scatter
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"])
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()


def test_f64_arrays_take_the_chain(cuda, tmp_path):
    """f64 application arrays (computed in f32, stored back as f64,
    models.py:211-223) fall back from the f32-only warp-MMA kernel to the
    layer chain, same tolerance."""
    wl = _region([5, 64, 32, 1], 2049, "relu")
    wl.arrays = {k: v.astype(np.float64) for k, v in wl.arrays.items()}
    got, launches = _run(wl, tmp_path)
    assert launches == 4 and got.dtype == np.float64
    ref, _ = c_oracle.mlp_f32(wl.layers, wl.arrays["recs"].astype(np.float32))
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()


@pytest.mark.parametrize("world", [3, 7])
def test_small_mma_shards_match_the_whole_call(cuda, tmp_path, world):
    """Sweep shards start at arbitrary rows, so the packed input rows of a
    shard start at any 4-B offset of a 16-B bulk-copy granule: every shard's
    rows are bitwise those of the unsharded call (ring chunks + per-lane
    tail)."""
    wl = _region([5, 64, 32, 1], 200_003, "relu")
    whole, _ = _run(wl, tmp_path)
    got = np.full_like(whole, np.nan)
    for r in range(world):
        wl.arrays["price"][:] = np.nan
        part, _ = _run(wl, tmp_path, shard=(r, world))
        done = ~np.isnan(part)
        got[done] = part[done]
    assert np.array_equal(got, whole)


def test_warp_mma_kernel_when_tcgen05_kernel_is_off(cuda):
    """Packed rows with F <= 6 take the tcgen05 small-MLP kernel
    (small_tc.cu); SMLRT_SMALL_TC=0 (read once per process) routes them to
    the warp-MMA kernel, which must meet the same checks: the C1 cases of
    this file re-run in a subprocess with the switch off."""
    import os
    import subprocess
    import sys
    if os.environ.get("SMLRT_SMALL_TC") == "0":
        pytest.skip("already the warp-MMA run")
    env = dict(os.environ, SMLRT_SMALL_TC="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k",
                        "matches_oracle or options_bf16_config or shards or nonfinite"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("in_soa,out_soa", [(True, False), (False, True), (True, True)])
def test_small_mlp_column_layouts(cuda, tmp_path, in_soa, out_soa):
    """Column-per-feature (SoA) arrays: strided input rows take the warp-MMA
    kernel's per-lane plan loads, packed input rows with SoA outputs take the
    tcgen05 kernel's generic output plan (row step 1, column offsets o * n);
    both against the oracle and the quantisation emulation."""
    dims, n = [5, 64, 32, 2], 20_011
    wl = _region(dims, n, "relu", seed=7)
    x = wl.arrays["recs"]
    fin = "functor(optin: [k, 0:5] = ([0:5, k]))" if in_soa else "functor(optin: [k, 0:5] = ([k, 0:5]))"
    fout = "functor(optout: [k, 0:2] = ([0, k], [1, k]))" if out_soa else "functor(optout: [k, 0:2] = ([k, 0], [k, 1]))"
    wl.arrays = {"recs": np.ascontiguousarray(x.T) if in_soa else x,
                 "price": np.zeros((2, n) if out_soa else (n, 2), np.float32)}
    wl.spec = type(wl.spec)(**{**wl.spec.__dict__, "in_functor": fin, "out_functor": fout})
    got, launches = _run(wl, tmp_path)
    assert launches == 1
    got = got.T if out_soa else got
    wl.arrays["recs"] = x  # the checks read row-major features
    _check(wl, np.ascontiguousarray(got).astype(np.float64))
