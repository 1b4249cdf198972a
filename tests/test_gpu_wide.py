"""C3 MiniBUDE (6-1024-512-256-1, bf16): TMA-fed tcgen05 GEMM chain vs the
fp32 oracle (SURVEY.md section 8(d) bf16 tolerance) and a bf16-emulated
forward pass."""

import numpy as np
import pytest
import torch

import paper_2407_18352_b200 as sm
from oracle import c_oracle
from paper_2407_18352_b200 import _native, workloads

pytestmark = pytest.mark.gpu


def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def emulate(layers, x):
    h = bf16(x)
    for i, (w, b, act) in enumerate(layers[:-1]):
        h = h @ bf16(w).T + b
        if act == "relu":
            h = np.maximum(h, 0)
        if i < len(layers) - 2:
            h = bf16(h)
    w, b, _ = layers[-1]
    return h @ w.T.astype(np.float64) + b


def check_tol(got, ref):
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    rmse = np.sqrt(np.mean((got - ref) ** 2)) / np.sqrt(np.mean(ref ** 2))
    assert err.max() <= 2e-2 * scale, (err.max(), scale)
    assert rmse <= 1e-2, rmse


def run(wl, tmp_path):
    sm.save_model(wl.model, tmp_path / "m")
    with sm.Runtime() as rt:
        rt.invoke_region(rt.register_region(wl.descriptor(str(tmp_path / "m"))))
    return wl.buffers["energy"].to_numpy().astype(np.float64)


@pytest.mark.parametrize("n", [100, 4096, 70_001])
def test_minibude_tolerance(cuda, tmp_path, n):
    wl = workloads.make("minibude", n)
    wl.to_device()
    assert _native.model_path(sm.models.device_model(wl.model, cuda)) == 3
    got = run(wl, tmp_path)
    x = np.ascontiguousarray(wl.arrays["poses"].T)  # SoA [6, N] -> rows
    ref, finite = c_oracle.mlp_f32(wl.layers, x)
    assert finite
    check_tol(got, ref[:, 0].astype(np.float64))
    emu = emulate(wl.layers, x)[:, 0]
    assert np.max(np.abs(got - emu)) <= 2e-3 * max(1.0, np.abs(emu).max())


def test_minibude_full_size_subsample(cuda, tmp_path):
    wl = workloads.make("minibude")
    wl.to_device()
    got = run(wl, tmp_path)
    idx = np.arange(0, wl.elements, 4099)
    x = np.ascontiguousarray(wl.arrays["poses"][:, idx].T)
    ref, _ = c_oracle.mlp_f32(wl.layers, x)
    check_tol(got[idx], ref[:, 0].astype(np.float64))


@pytest.mark.parametrize("env", [{"SMLRT_W4_PAIR": "0"}, {"SMLRT_WIDE_W4": "0"}])
def test_minibude_kernel_variants(cuda, tmp_path, env):
    """The single-CTA fused kernel (SMLRT_W4_PAIR=0) and round 1's two-kernel
    chain (SMLRT_WIDE_W4=0) meet the same tolerances (subprocesses: the
    switches are read once per process)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import test_gpu_wide as t, pathlib, tempfile;"
            "from paper_2407_18352_b200 import workloads; from oracle import c_oracle;"
            "wl = workloads.make('minibude', 70001); wl.to_device();"
            "got = t.run(wl, pathlib.Path(tempfile.mkdtemp()));"
            "x = np.ascontiguousarray(wl.arrays['poses'].T); ref, _ = c_oracle.mlp_f32(wl.layers, x);"
            "t.check_tol(got, ref[:, 0].astype(np.float64));"
            "emu = t.emulate(wl.layers, x)[:, 0];"
            "assert np.max(np.abs(got - emu)) <= 2e-3 * max(1.0, np.abs(emu).max()); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("act", ["tanh", "identity"])
def test_wide_fused_activations(cuda, tmp_path, act):
    """Same shape, other hidden activations (the fused kernel's tanh / identity
    instantiations) against the fp32 oracle."""
    n = 9000
    layers = workloads.init_weights([6, 1024, 512, 256, 1], act)
    model = sm.Model(6, 1, [sm.DenseLayer(w, b, a) for w, b, a in layers], precision="bf16")
    wl = workloads.make("minibude", n)
    wl.layers, wl.model = layers, model
    wl.to_device()
    got = run(wl, tmp_path)
    x = np.ascontiguousarray(wl.arrays["poses"].T)
    ref, _ = c_oracle.mlp_f32(layers, x)
    check_tol(got, ref[:, 0].astype(np.float64))
